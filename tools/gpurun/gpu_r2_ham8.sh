timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "frag or multiwindow or ties or k100" > gpurun_out/t_ham8.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/t_ham8.log
export PROBE_PF=20
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1 --reps 3 --variants 'seg8=;seg4=CRISP_HAMMING_SEG8=0' > gpurun_out/probe_ham8.jsonl 2> gpurun_out/probe_ham8.err; echo rc4=$?
timeout 900 python tools/stage_probe.py --cfg 5 --modes 1 --reps 2 --variants 'seg8=;seg4=CRISP_HAMMING_SEG8=0' > gpurun_out/probe_ham8_5.jsonl 2> gpurun_out/probe_ham8_5.err; echo rc5=$?
timeout 900 python tools/stage_probe.py --cfg 3 --modes 1 --reps 2 --variants 'seg8=;seg4=CRISP_HAMMING_SEG8=0' > gpurun_out/probe_ham8_3.jsonl 2> gpurun_out/probe_ham8_3.err; echo rc3=$?
