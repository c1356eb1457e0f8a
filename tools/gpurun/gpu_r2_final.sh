# round-2 bundle: full GPU tests, the driver's bench command, reference arm, smoke, ncu launch list + full capture
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests_c.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r2_gpu_tests_c.log
start=$(date +%s); timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench_rc=$? wall_s=$(( $(date +%s) - start ))
timeout 900 python bench.py --impl reference --gpus 1 --steps 5 --warmup 3 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err; echo ref_rc=$?
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
KRE='regex:k_(prep_queries|slice_rows|rot_tc|recompute|screen_tc|probe|query_key|act_rows|count_frag|count_warp|fallback|hamming|hsort|verify_rows|patience|rerank_exact|merge_lists)'
timeout 600 python tools/one_search.py 4 1 1 > gpurun_out/p1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k "$KRE" -c 400 --csv --log-file gpurun_out/r2_traffic_final_m1.csv python tools/one_search.py 4 1 1 > gpurun_out/ncu1.log 2>&1; echo ncu1_rc=$?
ncu --set full --clock-control none --import-source on -k "regex:k_(verify_rows|count_frag|hamming_dense|rot_tc|screen_tc|probe|hsort_cta|recompute)" -s 72 -c 10 -o gpurun_out/r2_ncu_full_final python tools/one_search.py 4 1 1 > gpurun_out/ncu2.log 2>&1; echo ncu2_rc=$?
