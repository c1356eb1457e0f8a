# bench lines of the other configs with the verification filter (stage breakdown in the .err)
for c in 2 3 5; do
timeout 1500 python bench.py --cfg $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_cfg${c}_f.json 2> gpurun_out/r2_bench_cfg${c}_f.err; echo cfg${c}_rc=$?; grep "mode" gpurun_out/r2_bench_cfg${c}_f.err
done
