# a1 screen on the tensor cores: parity (screen paths + the stagewise suite), smoke, timings, ncu of the screen
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "screen or cfg1 or rotated or ties or wide or k100 or fallback or model_from" > gpurun_out/t_a1.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/t_a1.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
timeout 600 python bench.py --mode 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b4_m1.json 2> gpurun_out/b4_m1.err; grep "mode 1" gpurun_out/b4_m1.err
python -c "import json;d=json.load(open('gpurun_out/b4_m1.json'));print(d['counters_per_step'])"
CRISP_PROBE_SCREEN=0 timeout 600 python bench.py --mode 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b4_m1n.json 2> gpurun_out/b4_m1n.err; grep "mode 1" gpurun_out/b4_m1n.err
timeout 600 python tools/one_search.py 4 1 1 > gpurun_out/p1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_screen_tc|k_probe" -s 2 -c 2 -o gpurun_out/r2_prof_a1 python tools/one_search.py 4 1 1 > gpurun_out/ncu1.log 2>&1; echo ncu1_rc=$?
