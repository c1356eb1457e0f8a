# the driver's bench command + the model-build / multirank tests
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
start=$(date +%s); timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench_rc=$? wall_s=$(( $(date +%s) - start )); tail -4 gpurun_out/r2_bench.err
timeout 1200 python -m pytest tests -m gpu -x -q -k "model_from or multirank" > gpurun_out/t_model.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/t_model.log
