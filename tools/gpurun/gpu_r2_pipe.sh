timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "async_returns or cfg1_stagewise" > gpurun_out/t_pipe.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/t_pipe.log
for P in 1 2 4; do CRISP_PIPE=$P timeout 600 python bench.py --mode 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b4_p$P.json 2> gpurun_out/b4_p$P.err; echo pipe=$P; grep "mode 1" gpurun_out/b4_p$P.err | cut -c1-60; done
CRISP_PIPE=2 timeout 600 python bench.py --mode 0 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b4_p2m0.json 2> gpurun_out/b4_p2m0.err; grep "mode 0" gpurun_out/b4_p2m0.err | cut -c1-60
CRISP_PIPE=2 timeout 600 python bench.py --cfg 2 --mode 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b2_p2.json 2> gpurun_out/b2_p2.err; grep "mode 1" gpurun_out/b2_p2.err | cut -c1-60
