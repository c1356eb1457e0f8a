# exact global patience over G shards (one-GPU emulation) + the filter tests + count parity
timeout 1200 python -m pytest tests/test_gpu_global_patience.py -x -q > gpurun_out/t_gp.log 2>&1; echo gp_rc=$?; tail -15 gpurun_out/t_gp.log
