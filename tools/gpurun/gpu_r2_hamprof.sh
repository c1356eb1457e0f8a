export PROBE_PF=20
timeout 600 python tools/one_search.py 4 1 1 > gpurun_out/p1h.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hamming_seg -s 0 -c 1 -o gpurun_out/s3_ham_full python tools/one_search.py 4 1 1 > gpurun_out/ncu_ham.log 2>&1; echo ncu_rc=$?
