# round-2 bundle with the verification filter: full GPU tests, the driver's bench command, reference arm,
# smoke, ncu launch lists (traffic) of one cfg4 search per mode
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests_d.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r2_gpu_tests_d.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_f.json 2> gpurun_out/r2_bench_f.err; echo bench_rc=$?; grep mode gpurun_out/r2_bench_f.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 5 --warmup 3 > gpurun_out/r2_bench_ref_f.json 2> gpurun_out/r2_bench_ref_f.err; echo ref_rc=$?
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
KRE='regex:k_(prep_queries|slice_rows|rot_tc|recompute|screen_tc|probe|query_key|act_rows|count_frag|count_warp|fallback|hamming|hsort|verify_rows|patience|rerank_exact|merge_lists|q8_prep|lb_bounds|lb_threshold)'
for m in 1 0; do
timeout 600 python tools/one_search.py 4 $m 1 > gpurun_out/p$m.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k "$KRE" -c 400 --csv --log-file gpurun_out/r2_traffic_filt_m$m.csv python tools/one_search.py 4 $m 1 > gpurun_out/ncu_m$m.log 2>&1; echo ncu_m${m}_rc=$?
done
