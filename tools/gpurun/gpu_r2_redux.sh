timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "frag or wide or chunked or cfg1 or ragged" > gpurun_out/t_redux.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/t_redux.log
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1,0 --reps 3 --variants 'redux=' > gpurun_out/probe_redux4.jsonl 2> gpurun_out/probe_redux4.err; echo rc4=$?
timeout 600 python tools/stage_probe.py --cfg 3 --modes 1 --reps 2 --variants 'redux=' > gpurun_out/probe_redux3.jsonl 2> gpurun_out/probe_redux3.err; echo rc3=$?
timeout 600 python tools/stage_probe.py --cfg 5 --modes 1 --reps 2 --variants 'redux=' > gpurun_out/probe_redux5.jsonl 2> gpurun_out/probe_redux5.err; echo rc5=$?
