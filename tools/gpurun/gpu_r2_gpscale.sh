# projected multi-GPU steps at cfg4 (G ranks' kernels on one GPU, collectives modelled); Q shrinks with G (memory)
timeout 1200 python tools/gp_scale_probe.py --G 4 --Q 5000 --modes 1,0 > gpurun_out/gp_scale_cfg4_g4.jsonl 2> gpurun_out/gp_scale_cfg4_g4.err; echo rc4=$?; tail -2 gpurun_out/gp_scale_cfg4_g4.err
timeout 1200 python tools/gp_scale_probe.py --G 8 --Q 2500 --modes 1,0 > gpurun_out/gp_scale_cfg4_g8.jsonl 2> gpurun_out/gp_scale_cfg4_g8.err; echo rc8=$?; tail -2 gpurun_out/gp_scale_cfg4_g8.err
timeout 1200 python tools/gp_scale_probe.py --G 2 --Q 10000 --modes 0 > gpurun_out/gp_scale_cfg4_g2m0.jsonl 2> gpurun_out/gp_scale_cfg4_g2m0.err; echo rc2=$?; tail -2 gpurun_out/gp_scale_cfg4_g2m0.err
