nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_b0.json 2> gpurun_out/r2_b0.err; echo bench_rc=$?
KRE='regex:k_(prep_queries|rotate_f64|slice_rows|certify|recompute|probe|query_key|count_warp|count_select|fallback|hamming|hsort|verify_rows|patience|rerank_exact|merge_lists|stats)|gemm_s8'
timeout 600 python tools/one_search.py 4 1 1 > gpurun_out/p0.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" -c 3000 --csv --log-file gpurun_out/r2_launches_cfg4.csv python tools/one_search.py 4 1 1 > gpurun_out/ncu0.log 2>&1; echo ncu0_rc=$?
timeout 600 python tools/one_search.py 4 1 1 1000 > gpurun_out/p1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_count_select" -s 1 -c 1 -o gpurun_out/r2_prof_count4 python tools/one_search.py 4 1 1 1000 > gpurun_out/ncu1.log 2>&1; echo ncu1_rc=$?
