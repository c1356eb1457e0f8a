"""Build and run tools/peaks/l2_hbm_peak.cu on the GPU box: the L2 -> SM read
bandwidth (the ceiling of the L2-resident hot kernels) and the HBM read
bandwidth, measured in-repo; writes profiles/<name>.json (with the clocks seen)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = os.path.join(ROOT, "tools", "peaks", "l2_hbm_peak.cu")
exe = "/tmp/l2_hbm_peak"
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-o", exe, src])
out = json.loads(subprocess.check_output([exe], text=True).strip().splitlines()[-1])
q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
out["nvidia_smi_after"] = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader"], capture_output=True,
                                         text=True).stdout.strip()
name = sys.argv[1] if len(sys.argv) > 1 else "r02_peaks"
for d in ("profiles", "gpurun_out"):
    os.makedirs(os.path.join(ROOT, d), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", name + ".json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))
