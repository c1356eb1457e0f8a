# session 4: the shared-memory update ceiling (tools/peaks/smem_red_peak.cu, the count's launch shape),
# and one ncu --set full source-level capture of the cfg4 collision count (k_count_frag)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/smem_red_peak tools/peaks/smem_red_peak.cu && \
for i in 1 2; do /tmp/smem_red_peak; done > gpurun_out/s4b_smem_peak.jsonl; echo peak_rc=$?
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv,noheader >> gpurun_out/s4b_smem_peak.jsonl
export PROBE_PF=20
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_count_frag -s 1 -c 1 -o gpurun_out/s4b_count python tools/one_search.py 4 1 1 > gpurun_out/s4b_ncu.log 2>&1; echo ncu_rc=$?
ncu -i gpurun_out/s4b_count.ncu-rep --page source --csv --print-source sass > gpurun_out/s4b_count_src.csv 2>/dev/null; echo src_rc=$?
ncu -i gpurun_out/s4b_count.ncu-rep --page raw --csv > gpurun_out/s4b_count_raw.csv 2>/dev/null; echo raw_rc=$?
