export PROBE_PF=20
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1 --reps 3 --variants 'base=;sp1k=CRISP_LB_SPAN=1024;sp1.5k=CRISP_LB_SPAN=1536;f192=CRISP_LB_FIRST=192;f128=CRISP_LB_FIRST=128;r4=CRISP_LB_ROUNDS=4;rs3=CRISP_ROUND_SPLITS=3;nofilt=CRISP_FILTER_ROUNDS=0' > gpurun_out/probe_pf20.jsonl 2> gpurun_out/probe_pf20.err; echo rc=$?
