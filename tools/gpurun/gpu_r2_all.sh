timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "screen or cfg1_stagewise" > gpurun_out/t_all.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/t_all.log
CRISP_IMMA_STATS=1 timeout 600 python tools/one_search.py 4 1 1 2>&1 | grep -E "crisp imma" | tail -3
for C in 4 2 3 5; do timeout 900 python bench.py --cfg $C --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b$C.json 2> gpurun_out/b$C.err; echo cfg$C=$?; grep "^mode" gpurun_out/b$C.err | cut -c1-330; done
