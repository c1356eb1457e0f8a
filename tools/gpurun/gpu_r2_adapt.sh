# f4 adaptive subspaces: the new parity tests, then the screen/build/f4 neighbours and smoke
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "adaptive or blockwise or build_matches or screen" > gpurun_out/t_adapt.log 2>&1; echo tests_rc=$?; tail -30 gpurun_out/t_adapt.log | grep -v "^$" | tail -25
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
