# session 4: the 89-instruction step (funnel shift, block-relative word address):
# the whole GPU suite, then the cfg4 phi=1 stage probe
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s4j_gpu_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/s4j_gpu_tests.log
export PROBE_PF=20
timeout 1200 python tools/stage_probe.py --cfg 4 --modes 1 --reps 3 --variants 'step89=;step89b=' > gpurun_out/s4j_probe.jsonl 2> gpurun_out/s4j_probe.err; echo rc=$?
