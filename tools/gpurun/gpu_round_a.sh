# Round profiling bundle (run under gpurun): GPU test suite, bench line, ncu
# launch list of the bench command (library kernels only), one --set full
# capture of the hot kernels of each mode.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench_rc=$?
KRE='regex:k_(prep_queries|rotate_f64|slice_rows|certify|recompute|probe|query_key|count_warp|count_select|fallback|hamming|hsort|verify_rows|patience|rerank_exact|merge_lists|stats)|gemm_s8'
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
python tools/one_search.py 2 1 1 > gpurun_out/plain3.log 2>&1 && python tools/one_search.py 2 0 1 > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_(count_warp|verify_rows|hsort_cta|probe|patience|hamming_dense)" -s 11 -c 11 -o gpurun_out/prof_m1 python tools/one_search.py 2 1 1 > gpurun_out/ncu_m1.log 2>&1; echo ncu2_rc=$?
# the certified a0 of the second search (the build runs the same kernels on 31 tiles first)
ncu --set full --clock-control none --import-source on -k "regex:k_(slice_rows|certify|recompute)" -s 96 -c 3 -o gpurun_out/prof_a0 python tools/one_search.py 2 1 1 > gpurun_out/ncu_a0.log 2>&1; echo ncu2b_rc=$?
ncu --set full --clock-control none --import-source on -k "regex:k_(rerank_exact|count_warp)" -s 2 -c 2 -o gpurun_out/prof_m0 python tools/one_search.py 2 0 1 > gpurun_out/ncu_m0.log 2>&1; echo ncu3_rc=$?
