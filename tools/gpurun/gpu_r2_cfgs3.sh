# other configs' bench lines on the final code (parity-test configs, not the driver's N=1 line)
for c in 2 3 5; do
timeout 1500 python bench.py --cfg $c --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3_bench_cfg$c.json 2> gpurun_out/s3_bench_cfg$c.err; echo cfg${c}_rc=$?
done
