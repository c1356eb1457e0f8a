export PROBE_PF=20
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1 --reps 3 --variants 'base=;list=CRISP_HSORT_LIST_MAX=16384' > gpurun_out/probe_hslist.jsonl 2> gpurun_out/probe_hslist.err; echo rc=$?
