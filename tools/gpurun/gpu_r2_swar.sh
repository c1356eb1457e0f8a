# k_count_frag with reductions + final SWAR scan: parity variants, then cfg4/cfg3/cfg5 stage timings
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "swar or wide or chunked" > gpurun_out/t_swar.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/t_swar.log
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1,0 --reps 3 --variants 'base=;swar=CRISP_COUNT_SWAR=1;swar_f4=CRISP_COUNT_SWAR=1,CRISP_COUNT_F=4;f4=CRISP_COUNT_F=4' > gpurun_out/probe_swar4.jsonl 2> gpurun_out/probe_swar4.err; echo rc4=$?
timeout 600 python tools/stage_probe.py --cfg 3 --modes 1 --reps 2 --variants 'base=;swar=CRISP_COUNT_SWAR=1' > gpurun_out/probe_swar3.jsonl 2> gpurun_out/probe_swar3.err; echo rc3=$?
timeout 600 python tools/stage_probe.py --cfg 5 --modes 1 --reps 2 --variants 'base=;swar=CRISP_COUNT_SWAR=1' > gpurun_out/probe_swar5.jsonl 2> gpurun_out/probe_swar5.err; echo rc5=$?
