# session 4: the staging prefix by a 32-bit scan + ballot:
# the whole GPU suite, then the cfg4 phi=1 stage probe
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s4i_gpu_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/s4i_gpu_tests.log
export PROBE_PF=20
timeout 1200 python tools/stage_probe.py --cfg 4 --modes 1 --reps 3 --variants 'scan32=;scan32b=' > gpurun_out/s4i_probe.jsonl 2> gpurun_out/s4i_probe.err; echo rc=$?
