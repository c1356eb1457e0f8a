# count variants: F=1 with 8-warp CTAs (4 per SM), F=1 16 warps, default (non-clobber atomics)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "frag_f1 or chunked" > gpurun_out/t_cf5.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/t_cf5.log
CRISP_COUNT_F=1 CRISP_COUNT_W8=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "frag and not fused and not group" > gpurun_out/t_cf5b.log 2>&1; echo tests_w8_rc=$?; tail -2 gpurun_out/t_cf5b.log
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1 --reps 5 --variants 'base=;f1=CRISP_COUNT_F=1;f1w8=CRISP_COUNT_F=1,CRISP_COUNT_W8=1;base2=' > gpurun_out/probe_cf5.jsonl 2> gpurun_out/probe_cf5.err; echo rc=$?
