# full GPU test suite + per-kernel traffic of one cfg4 search step (both modes) + cfg2/3/5 lines
timeout 2000 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests_b.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/r2_gpu_tests_b.log
KRE='regex:k_(prep_queries|slice_rows|rot_tc|recompute|probe|query_key|act_rows|count_frag|count_warp|fallback|hamming|hsort|verify_rows|patience|rerank_exact|merge_lists)'
for MODE in 1 0; do
timeout 600 python tools/one_search.py 4 $MODE 1 > gpurun_out/p_$MODE.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k "$KRE" -c 400 --csv --log-file gpurun_out/r2_traffic_cfg4_m$MODE.csv python tools/one_search.py 4 $MODE 1 > gpurun_out/ncu_$MODE.log 2>&1; echo ncu_rc=$?
done
for C in 2 3 5; do timeout 900 python bench.py --cfg $C --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b$C.json 2> gpurun_out/b$C.err; echo cfg$C=$?; grep "^mode" gpurun_out/b$C.err; done
