# gap check: stage sums vs event time with the filter rounds, variants in alternating order
timeout 600 python tools/stage_probe.py --cfg 2 --modes 1 --reps 10 --variants 'on=;off=CRISP_FILTER_ROUNDS=0;on2=;off2=CRISP_FILTER_ROUNDS=0;f256=CRISP_LB_FIRST=256' > gpurun_out/probe_gap2.jsonl 2> gpurun_out/probe_gap2.err; echo rc=$?
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1 --reps 6 --variants 'f256=CRISP_LB_FIRST=256;off=CRISP_FILTER_ROUNDS=0;on=;f256b=CRISP_LB_FIRST=256;f384=CRISP_LB_FIRST=384' > gpurun_out/probe_gap4.jsonl 2> gpurun_out/probe_gap4.err; echo rc=$?
CRISP_LB_FIRST=256 timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/b_filt.json 2> gpurun_out/b_filt.err; echo bench_rc=$?; grep "mode" gpurun_out/b_filt.err
