# count with shared reductions + SWAR scan; grouped phi=0 re-rank
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "frag or group or fallback or cfg1 or rotated or full_blocks or wide or chunked or capacity or ties" > gpurun_out/t_next.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/t_next.log
timeout 600 python bench.py --mode 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b4_m1.json 2> gpurun_out/b4_m1.err; grep "mode 1" gpurun_out/b4_m1.err
for G in 1 0; do
CRISP_RERANK_GROUP=$G timeout 900 python bench.py --cfg 3 --mode 0 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b3_g$G.json 2> gpurun_out/b3_g$G.err; grep "mode 0" gpurun_out/b3_g$G.err
CRISP_RERANK_GROUP=$G timeout 900 python bench.py --cfg 5 --mode 0 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b5_g$G.json 2> gpurun_out/b5_g$G.err; grep "mode 0" gpurun_out/b5_g$G.err
done
