# session-3 baseline on the latest commits: full GPU tests, the driver's bench command, reference arm, smoke,
# launch list of the bench's cfg4 phi=1 search, one ncu --set full capture of the collision count
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s3_gpu_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/s3_gpu_tests.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference --gpus 1 --steps 5 --warmup 3 > gpurun_out/s3_bench_ref.json 2> gpurun_out/s3_bench_ref.err; echo ref_rc=$?
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
KRE='regex:k_'
timeout 600 python tools/one_search.py 4 1 1 > gpurun_out/p1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k "$KRE" -c 400 --csv --log-file gpurun_out/s3_launches_m1.csv python tools/one_search.py 4 1 1 > gpurun_out/ncu_m1.log 2>&1; echo ncu_m1_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_count_frag -s 1 -c 1 -o gpurun_out/s3_count_full python tools/one_search.py 4 1 1 > gpurun_out/ncu_full.log 2>&1; echo ncu_full_rc=$?
