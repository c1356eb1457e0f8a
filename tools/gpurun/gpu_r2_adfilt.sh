timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_filter.py -x -q -k "adsampling or filter" > gpurun_out/t_adfilt.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/t_adfilt.log
export PROBE_PF=20
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1 --reps 3 --variants 'exact=;ad=PROBE_AD=1' > gpurun_out/probe_adfilt.jsonl 2> gpurun_out/probe_adfilt.err; echo rc=$?
