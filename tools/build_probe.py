"""Build throughput: wall time of crisp_build on a config's
base set (data resident on the GPU), repeated; run under ncu for the kernel split."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as ge  # noqa: E402
import bench  # noqa: E402
import synth  # noqa: E402

ge.build()
import paper_2603_05180_b200 as crisp  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
c = synth.CONFIGS[cfg]
op = bench.load_op(cfg)
w = synth.Workload(cfg, device="cuda")
X = w.base(c["N"])
torch.cuda.synchronize()
for r in range(reps):
    t0 = time.perf_counter()
    ix = crisp.Index.build(X, op["M"], K=50, seed=op.get("seed", 1))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print({"cfg": cfg, "N": c["N"], "D": c["D"], "M": op["M"], "rotated": ix.info()["rotated"], "build_s": round(dt, 3),
           "points_per_s": round(c["N"] / dt)})
    ix.free()
