export PROBE_PF=20
timeout 900 python tools/stage_probe.py --cfg 4 --modes 1 --reps 3 --variants 'base=;ctas4=CRISP_LB_CTAS=4;rs1=CRISP_ROUND_SPLITS=1;rs3=CRISP_ROUND_SPLITS=3;rr64=CRISP_ROUND_ROWS=64;rr256=CRISP_ROUND_ROWS=256;rsp2=CRISP_RERANK_SPLITS=2;rsp8=CRISP_RERANK_SPLITS=8' > gpurun_out/probe_vocc.jsonl 2> gpurun_out/probe_vocc.err; echo rc=$?
