# session-4 bundle on the restored tree (after hsort listing B, H2D parts, phi=0 point): GPU tests, the driver's bench command, reference arm, smoke,
# a launch list of one cfg4 phi=1 search (search kernels only), one ncu --set full of the verification rounds
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s4a_gpu_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/s4a_gpu_tests.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s4a_bench.json 2> gpurun_out/s4a_bench.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference --gpus 1 --steps 5 --warmup 3 > gpurun_out/s4a_bench_ref.json 2> gpurun_out/s4a_bench_ref.err; echo ref_rc=$?
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
export PROBE_PF=20
KRE='regex:k_(prep_queries|slice_rows|rot_tc|recompute|screen_tc|probe|query_key|act_rows|count_frag|count_warp|fallback|qcodes|hamming|hhist|hsort|verify_rows|q8_prep|patience|rerank_exact|merge_lists|lb_bounds|lb_threshold)'
timeout 600 python tools/one_search.py 4 1 1 > gpurun_out/p1s4a.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k "$KRE" -c 600 --csv --log-file gpurun_out/s4a_launches_m1.csv python tools/one_search.py 4 1 1 > gpurun_out/ncu_m1s4a.log 2>&1; echo ncu_m1_rc=$?
