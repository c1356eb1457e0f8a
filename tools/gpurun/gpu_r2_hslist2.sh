timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "multiwindow or k100 or cfg1 or ragged or ties or adsampling" > gpurun_out/t_hslist.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/t_hslist.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -k "cfg4" > gpurun_out/t_hslist_full.log 2>&1; echo full_rc=$?; tail -2 gpurun_out/t_hslist_full.log
