# segment-major Hamming: parity (phi=1 paths) and cfg4/cfg2 timing vs the per-query kernel
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_filter.py tests/test_gpu_global_patience.py -x -q > gpurun_out/t_ham3.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/t_ham3.log
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1 --reps 5 --variants 'seg=;dense=CRISP_HAMMING_SEG=0;seg2=' > gpurun_out/probe_ham3.jsonl 2> gpurun_out/probe_ham3.err; echo rc=$?
timeout 900 python tools/stage_probe.py --cfg 2 --modes 1 --reps 10 --variants 'seg=;dense=CRISP_HAMMING_SEG=0' > gpurun_out/probe_ham3_2.jsonl 2> gpurun_out/probe_ham3_2.err; echo rc=$?
