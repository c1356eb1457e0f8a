timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg1 or ragged or screen or ties or adaptive or k100 or wide" > gpurun_out/t_probered.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/t_probered.log
export PROBE_PF=20
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1 --reps 3 --variants 'redux=' > gpurun_out/probe_probered.jsonl 2> gpurun_out/probe_probered.err; echo rc4=$?
timeout 900 python tools/stage_probe.py --cfg 3 --modes 1 --reps 2 --variants 'redux=' > gpurun_out/probe_probered3.jsonl 2> gpurun_out/probe_probered3.err; echo rc3=$?
