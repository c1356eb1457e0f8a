# filtered verification: deferred exact queue, lane-parallel bounds; CTA/SM and split variants
timeout 900 python -m pytest tests/test_gpu_filter.py -x -q > gpurun_out/t_filt2.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/t_filt2.log
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1,0 --reps 5 --variants 'base=;c4=CRISP_LB_CTAS=4;s2=CRISP_ROUND_SPLITS=2;s6=CRISP_ROUND_SPLITS=6;c4s6=CRISP_LB_CTAS=4,CRISP_ROUND_SPLITS=6' > gpurun_out/probe_lb2.jsonl 2> gpurun_out/probe_lb2.err; echo rc=$?
