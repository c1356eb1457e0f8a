# op-point sweep at cfg4 with the verification filter (phi=1 and phi=0), M=32
timeout 2400 python bench.py --sweep --cfg 4 --sweep-M 32 --sweep-beta 0.006,0.008,0.01,0.0125 --sweep-alpha 0.25,0.3,0.35,0.4 --sweep-modes 1 > gpurun_out/sweep4_filt_m1.jsonl 2> gpurun_out/sweep4_filt_m1.err; echo rc1=$?
timeout 2400 python bench.py --sweep --cfg 4 --sweep-M 32 --sweep-beta 0.01,0.015,0.02 --sweep-alpha 0.15,0.2,0.25 --sweep-modes 0 > gpurun_out/sweep4_filt_m0.jsonl 2> gpurun_out/sweep4_filt_m0.err; echo rc0=$?
