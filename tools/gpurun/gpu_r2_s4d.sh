# session 4: host-buffer crisp_search at cfg4 (H2D part schedules), the bench line's e2e gap
timeout 1200 python tools/e2e_probe.py 4 1,t3,t4,4,8 > gpurun_out/s4d_e2e.log 2>&1; echo rc=$?
tail -20 gpurun_out/s4d_e2e.log
