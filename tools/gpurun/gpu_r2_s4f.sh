# session 4 final: the driver's bench command (bench.py now reports the count's update_frac), the reference arm, smoke
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s4f_bench.json 2> gpurun_out/s4f_bench.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference --gpus 1 --steps 5 --warmup 3 > gpurun_out/s4f_bench_ref.json 2> gpurun_out/s4f_bench_ref.err; echo ref_rc=$?
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
