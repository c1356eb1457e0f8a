# block-major filtered rounds: parity + timing vs the per-query kernel
timeout 1500 python -m pytest tests/test_gpu_filter.py tests/test_gpu_global_patience.py -x -q > gpurun_out/t_lbblk.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/t_lbblk.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "k100 or patience or ties or frag" > gpurun_out/t_lbblk2.log 2>&1; echo tests2_rc=$?; tail -2 gpurun_out/t_lbblk2.log
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1 --reps 5 --variants 'blk=;old=CRISP_LB_BLOCKS=0;b13=CRISP_LB_BSH=13;b15=CRISP_LB_BSH=15' > gpurun_out/probe_lbblk.jsonl 2> gpurun_out/probe_lbblk.err; echo rc=$?
timeout 900 python tools/stage_probe.py --cfg 5 --modes 1 --reps 3 --variants 'blk=;old=CRISP_LB_BLOCKS=0' > gpurun_out/probe_lbblk5.jsonl 2> gpurun_out/probe_lbblk5.err; echo rc=$?
