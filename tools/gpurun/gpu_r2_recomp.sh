timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "rotat or adversar or imma or a0 or cfg1 or blockwise or k100" > gpurun_out/t_recomp.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/t_recomp.log
CRISP_IMMA_STATS=1 PROBE_PF=20 timeout 600 python tools/one_search.py 4 1 1 2>&1 | grep imma | tail -2
export PROBE_PF=20
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1 --reps 3 --variants 'rows=' > gpurun_out/probe_recomp.jsonl 2> gpurun_out/probe_recomp.err; echo rc4=$?
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -k "cfg4_index or index_bit_exact" > gpurun_out/t_recomp_full.log 2>&1; echo full_rc=$?; tail -2 gpurun_out/t_recomp_full.log
