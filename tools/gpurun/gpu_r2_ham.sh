# fused Hamming in k_count_frag; 32-warp F=4 variant
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "frag or cfg1 or rotated or full_blocks or ties or fallback or k100 or patience" > gpurun_out/t_ham.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/t_ham.log
timeout 600 python bench.py --mode 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b4_m1.json 2> gpurun_out/b4_m1.err; grep "mode 1" gpurun_out/b4_m1.err
CRISP_HAMMING_FUSED=0 timeout 600 python bench.py --mode 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b4_m1nf.json 2> gpurun_out/b4_m1nf.err; grep "mode 1" gpurun_out/b4_m1nf.err
CRISP_COUNT_F=4 timeout 600 python bench.py --mode 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b4_m1f4.json 2> gpurun_out/b4_m1f4.err; grep "mode 1" gpurun_out/b4_m1f4.err
timeout 600 python bench.py --cfg 5 --mode 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b5_m1.json 2> gpurun_out/b5_m1.err; grep "mode 1" gpurun_out/b5_m1.err
