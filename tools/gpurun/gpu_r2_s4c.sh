# session 4: count ids prefetch at staging (CRISP_COUNT_PREFETCH 1 = L2, 2 = L1), cfg4 phi=1 stage probe
export PROBE_PF=20
timeout 1200 python tools/stage_probe.py --cfg 4 --modes 1 --reps 3 --variants 'base=;pfL2=CRISP_COUNT_PREFETCH=1;pfL1=CRISP_COUNT_PREFETCH=2;base2=' > gpurun_out/s4c_probe.jsonl 2> gpurun_out/s4c_probe.err; echo rc=$?
