# session 4: the count with two quads in flight per lane (CRISP_COUNT_DEPTH=2): parity (every count test
# with the variant forced, plus the new stagewise variant), then the cfg4 phi=1 stage probe
CRISP_COUNT_DEPTH=2 timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "stagewise or chunked or wide or tie or fullsize" > gpurun_out/s4e_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/s4e_tests.log
export PROBE_PF=20
timeout 1200 python tools/stage_probe.py --cfg 4 --modes 1 --reps 3 --variants 'base=;d2=CRISP_COUNT_DEPTH=2;base2=;d2b=CRISP_COUNT_DEPTH=2' > gpurun_out/s4e_probe.jsonl 2> gpurun_out/s4e_probe.err; echo rc=$?
