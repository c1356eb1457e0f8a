# count kernel with the crossing checks one step late
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "frag or cfg1 or rotated or full_blocks or ties or fallback or k100 or chunked or capacity" > gpurun_out/t_cf4.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/t_cf4.log
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1 --reps 5 --variants 'base=' > gpurun_out/probe_cf4.jsonl 2> gpurun_out/probe_cf4.err; echo rc=$?
