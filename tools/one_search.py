"""One cfg search (for ncu): build, warm up once, run `reps` searches of the given mode."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as ge  # noqa: E402
import synth  # noqa: E402
import bench  # noqa: E402

cfg, mode, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 1
Qn = int(sys.argv[4]) if len(sys.argv) > 4 else None
ge.build()
import paper_2603_05180_b200 as crisp  # noqa: E402

c = synth.CONFIGS[cfg]
op = bench.load_op(cfg)
dev = torch.device("cuda", 0)
w = synth.Workload(cfg, device=dev)
X, Qd = w.base(c["N"]), w.queries(Qn or c["Q"])
index = crisp.Index.build(X, op["M"], K=50, seed=op.get("seed", 1))
mp = op["modes"][mode]
index.set_search_params(beta=mp["beta"], alpha=mp["alpha"], patience_factor=mp.get("patience_factor", 40))
index.set_adsampling(mode == 1 and os.environ.get("PROBE_AD", "0") == "1")
k = c["k"]
ids = torch.empty((Qd.shape[0], k), dtype=torch.int64, device=dev)
dd = torch.empty((Qd.shape[0], k), dtype=torch.float32, device=dev)
for _ in range(reps + 1):
    index.search_async(Qd, k, mode, ids, dd, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok", ids[0].tolist())
