# segment-major Hamming with precomputed query codes; HT 2 vs 4
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "frag or k100 or ties or fallback or patience" > gpurun_out/t_ham4.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/t_ham4.log
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1 --reps 5 --variants 'seg=;ht4=CRISP_HAMMING_SEG_HT=4;dense=CRISP_HAMMING_SEG=0' > gpurun_out/probe_ham4.jsonl 2> gpurun_out/probe_ham4.err; echo rc=$?
timeout 600 python tools/stage_probe.py --cfg 5 --modes 1 --reps 3 --variants 'seg=;dense=CRISP_HAMMING_SEG=0' > gpurun_out/probe_ham4_5.jsonl 2> gpurun_out/probe_ham4_5.err; echo rc=$?
