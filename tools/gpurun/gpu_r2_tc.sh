# base-256 digits (7 slices, 28 pairs): tests, timings, peaks (L2 via ld.cg), per-kernel DRAM traffic of a cfg4 step
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "certified_rotation or rotated or k100 or build" > gpurun_out/t_tc.log 2>&1; echo tc_tests_rc=$?; tail -3 gpurun_out/t_tc.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
timeout 600 python bench.py --mode 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b4_m1.json 2> gpurun_out/b4_m1.err; grep "mode 1" gpurun_out/b4_m1.err
CRISP_ROTATE_GEMM=cublaslt timeout 600 python bench.py --mode 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b4_m1lt.json 2> gpurun_out/b4_m1lt.err; grep "mode 1" gpurun_out/b4_m1lt.err
timeout 300 python tools/measure_peaks.py r02_peaks; echo peaks_rc=$?
KRE='regex:k_(prep_queries|slice_rows|rot_tc|recompute|probe|query_key|act_rows|count_frag|count_warp|fallback|hamming|hsort|verify_rows|patience|rerank_exact|merge_lists)'
timeout 600 python tools/one_search.py 4 1 1 > gpurun_out/p1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k "$KRE" -s 130 -c 40 --csv --log-file gpurun_out/r2_traffic_cfg4_m1.csv python tools/one_search.py 4 1 1 > gpurun_out/ncu1.log 2>&1; echo ncu1_rc=$?
