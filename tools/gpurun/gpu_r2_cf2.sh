# one full ncu capture of the cfg4 count kernel (second search), a finer phi=1 op-point grid
timeout 600 python tools/one_search.py 4 1 1 > gpurun_out/p1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_count_frag -s 1 -c 1 -o gpurun_out/r2_prof_count_final python tools/one_search.py 4 1 1 > gpurun_out/ncu_cf.log 2>&1; echo ncu_rc=$?
timeout 1800 python bench.py --sweep --cfg 4 --sweep-M 32 --sweep-beta 0.008,0.009,0.01,0.011 --sweep-alpha 0.28,0.3,0.33 --sweep-modes 1 > gpurun_out/sweep4_fine.jsonl 2> gpurun_out/sweep4_fine.err; echo rc=$?
