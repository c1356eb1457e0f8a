timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "multiwindow or cfg1 or ragged or adsampling or k100 or ties" > gpurun_out/t_hsort.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/t_hsort.log
export PROBE_PF=20
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1 --reps 3 --variants 'hs=' > gpurun_out/probe_hsort4.jsonl 2> gpurun_out/probe_hsort4.err; echo rc4=$?
timeout 600 python tools/stage_probe.py --cfg 2 --modes 1 --reps 3 --variants 'hs=' > gpurun_out/probe_hsort2.jsonl 2> gpurun_out/probe_hsort2.err; echo rc2=$?
timeout 600 python tools/stage_probe.py --cfg 5 --modes 1 --reps 2 --variants 'hs=' > gpurun_out/probe_hsort5.jsonl 2> gpurun_out/probe_hsort5.err; echo rc5=$?
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -k "cfg4" > gpurun_out/t_hsort_full.log 2>&1; echo full_rc=$?; tail -2 gpurun_out/t_hsort_full.log
