# round-2 closing bundle on the HEAD tree (89-instruction count step): GPU suite, the driver's bench command,
# reference arm, smoke, and the ncu launch list (traffic) of one cfg4 phi=1 search
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/head_gpu_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/head_gpu_tests.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/head_bench.json 2> gpurun_out/head_bench.err; echo bench_rc=$?; cat gpurun_out/head_bench.json
timeout 900 python bench.py --impl reference --gpus 1 --steps 5 --warmup 3 > gpurun_out/head_bench_ref.json 2> gpurun_out/head_bench_ref.err; echo ref_rc=$?; cat gpurun_out/head_bench_ref.json
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
KRE='regex:k_(prep_queries|slice_rows|rot_tc|recompute|screen_tc|probe|query_key|act_rows|count_frag|count_warp|fallback|hamming|hsort|verify_rows|patience|rerank_exact|merge_lists|q8_prep|lb_bounds|lb_threshold)'
timeout 600 python tools/one_search.py 4 1 1 > gpurun_out/head_p1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k "$KRE" -c 400 --csv --log-file gpurun_out/head_traffic_m1.csv python tools/one_search.py 4 1 1 > gpurun_out/head_ncu_m1.log 2>&1; echo ncu_m1_rc=$?
