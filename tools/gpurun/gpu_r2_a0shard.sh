timeout 1500 python -m pytest tests/test_gpu_global_patience.py tests/test_gpu_bench_multirank.py -x -q > gpurun_out/t_a0shard.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/t_a0shard.log
timeout 1200 python tools/gp_scale_probe.py --G 2,4 --modes 1,0 > gpurun_out/gp_scale_a0.jsonl 2> gpurun_out/gp_scale_a0.err; echo rc=$?
timeout 900 python tools/gp_scale_probe.py --G 2,8 --modes 1,0 --Q 5000 > gpurun_out/gp_scale_a0_g8.jsonl 2> gpurun_out/gp_scale_a0_g8.err; echo rc8=$?
