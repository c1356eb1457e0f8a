# count kernel with static quad shares + sliding fragment window: parity (count variants, fullsize cfg4 index) and timing
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "frag or cfg1 or rotated or full_blocks or ties or fallback or k100 or chunked or capacity" > gpurun_out/t_cf3.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/t_cf3.log
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1,0 --reps 5 --variants 'base=' > gpurun_out/probe_cf3.jsonl 2> gpurun_out/probe_cf3.err; echo rc=$?
timeout 600 python tools/stage_probe.py --cfg 5 --modes 1 --reps 3 --variants 'base=' > gpurun_out/probe_cf3_5.jsonl 2> gpurun_out/probe_cf3_5.err; echo rc=$?
