timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "frag or multiwindow or ties or k100 or adaptive" > gpurun_out/t_hamtma.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/t_hamtma.log
export PROBE_PF=20
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1 --reps 3 --variants 'tma=;seg=CRISP_HAMMING_TMA=0' > gpurun_out/probe_hamtma.jsonl 2> gpurun_out/probe_hamtma.err; echo rc4=$?
timeout 900 python tools/stage_probe.py --cfg 5 --modes 1 --reps 2 --variants 'tma=;seg=CRISP_HAMMING_TMA=0' > gpurun_out/probe_hamtma5.jsonl 2> gpurun_out/probe_hamtma5.err; echo rc5=$?
