# global patience: emulation tests (rounds asserted) + bench N=2 on one GPU (gloo) vs N=1, + a timing of the protocol at cfg4 scale
timeout 1200 python -m pytest tests/test_gpu_global_patience.py tests/test_gpu_bench_multirank.py -x -q > gpurun_out/t_gp2.log 2>&1; echo rc=$?; tail -5 gpurun_out/t_gp2.log
