# block-major filtered rounds with 64 queries per CTA; then DRAM/L2 of the block kernel vs the per-query kernel
timeout 1500 python -m pytest tests/test_gpu_filter.py -x -q > gpurun_out/t_lbblk3.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/t_lbblk3.log
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1 --reps 5 --variants 'q64=;q8=CRISP_LB_QPC=8;old=CRISP_LB_BLOCKS=0;q64b15=CRISP_LB_BSH=15' > gpurun_out/probe_lbblk2.jsonl 2> gpurun_out/probe_lbblk2.err; echo rc=$?
timeout 600 python tools/one_search.py 4 1 1 > gpurun_out/p1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k "regex:k_verify_lb_blk|k_span_bucket" -c 40 --csv --log-file gpurun_out/r2_lbblk_traffic.csv python tools/one_search.py 4 1 1 > gpurun_out/ncu_lbblk.log 2>&1; echo ncu_rc=$?
