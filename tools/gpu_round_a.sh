# Round profiling bundle (run under gpurun): bench line, ncu launch list of the
# same command, one --set full capture of the hot kernels, the GPU test suite.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench_rc=$?
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
python tools/one_search.py 2 1 1 > gpurun_out/plain3.log 2>&1 && python tools/one_search.py 2 0 1 > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_count_warp|k_verify_rows|k_hsort_cta|k_probe|k_rotate|k_patience" -s 9 -c 9 -o gpurun_out/prof_m1 python tools/one_search.py 2 1 1 > gpurun_out/ncu_m1.log 2>&1; echo ncu2_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_rerank_exact|k_count_warp" -s 2 -c 2 -o gpurun_out/prof_m0 python tools/one_search.py 2 0 1 > gpurun_out/ncu_m0.log 2>&1; echo ncu3_rc=$?
