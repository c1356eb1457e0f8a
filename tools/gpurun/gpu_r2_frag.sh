# k_count_frag v5 + ADSampling round 0 = 2k: parity subset, then timings
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "frag or wide or chunked or fallback or capacity or adsampling or ties" > gpurun_out/t_frag.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/t_frag.log
timeout 600 python bench.py --mode 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b4_m1.json 2> gpurun_out/b4_m1.err; grep "mode 1" gpurun_out/b4_m1.err
timeout 600 python bench.py --mode 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b4_m2.json 2> gpurun_out/b4_m2.err; grep "mode 2" gpurun_out/b4_m2.err
timeout 600 python bench.py --cfg 2 --mode 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b2_m2.json 2> gpurun_out/b2_m2.err; grep "mode 2" gpurun_out/b2_m2.err
timeout 600 python bench.py --cfg 3 --mode 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b3_frag.json 2> gpurun_out/b3_frag.err; grep "mode 1" gpurun_out/b3_frag.err
timeout 600 python tools/one_search.py 4 1 1 1000 > gpurun_out/p1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_count_frag" -s 1 -c 1 -o gpurun_out/r2_prof_frag4e python tools/one_search.py 4 1 1 1000 > gpurun_out/ncu1.log 2>&1; echo ncu1_rc=$?
