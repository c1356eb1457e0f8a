# verification filter (R17): its tests, cfg4/cfg2 stage timings on/off and knob variants, then the parity suite
timeout 900 python -m pytest tests/test_gpu_filter.py -x -q > gpurun_out/t_filt.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/t_filt.log
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1,0 --reps 3 --variants 'off=CRISP_FILTER_ROUNDS=0,CRISP_FILTER_RERANK=0;on=;f256=CRISP_LB_FIRST=256;f128=CRISP_LB_FIRST=128;s1024=CRISP_LB_SPAN=1024;s4096=CRISP_LB_SPAN=4096' > gpurun_out/probe_filt4.jsonl 2> gpurun_out/probe_filt4.err; echo probe4_rc=$?
timeout 600 python tools/stage_probe.py --cfg 2 --modes 1,0 --reps 3 --variants 'off=CRISP_FILTER_ROUNDS=0,CRISP_FILTER_RERANK=0;on=;f128=CRISP_LB_FIRST=128' > gpurun_out/probe_filt2.jsonl 2> gpurun_out/probe_filt2.err; echo probe2_rc=$?
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t_par.log 2>&1; echo par_rc=$?; tail -3 gpurun_out/t_par.log
