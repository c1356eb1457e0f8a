# long-patience configs with filtered spans of P/2
for c in 3 5; do
timeout 1500 python bench.py --cfg $c --mode 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_cfg${c}_f2.json 2> gpurun_out/r2_bench_cfg${c}_f2.err; echo cfg${c}_rc=$?; grep "mode" gpurun_out/r2_bench_cfg${c}_f2.err
done
timeout 900 python -m pytest tests/test_gpu_filter.py -x -q 2>&1 | tail -2
