# bench line with the updated traffic file; ncu --set full of the first k_verify_rows_lb launch and of k_count_frag
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s3c_bench.json 2> gpurun_out/s3c_bench.err; echo bench_rc=$?
export PROBE_PF=20
timeout 600 python tools/one_search.py 4 1 1 > gpurun_out/p1c.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_verify_rows_lb -s 0 -c 1 -o gpurun_out/s3c_verify_full python tools/one_search.py 4 1 1 > gpurun_out/ncu_vfull_c.log 2>&1; echo ncu_v_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_count_frag -s 0 -c 1 -o gpurun_out/s3c_count_full python tools/one_search.py 4 1 1 > gpurun_out/ncu_cfull_c.log 2>&1; echo ncu_c_rc=$?
