"""Host-API (crisp_search with pinned host buffers) timing on cfg2 against the
device-pointer call: where the end-to-end overhead goes."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as ge  # noqa: E402
import bench  # noqa: E402
import synth  # noqa: E402

ge.build()
import paper_2603_05180_b200 as crisp  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = synth.CONFIGS[cfg]
op = bench.load_op(cfg)
w = synth.Workload(cfg, device="cuda")
X, Qd = w.base(c["N"]), w.queries(c["Q"])
Q, D, k = Qd.shape[0], Qd.shape[1], c["k"]
ix = crisp.Index.build(X, op["M"], K=50, seed=op.get("seed", 1))
mp = op["modes"][1]
ix.set_search_params(beta=mp["beta"], alpha=mp["alpha"], patience_factor=mp.get("patience_factor", 40))
qh = torch.empty((Q, D), dtype=torch.float32).pin_memory()
qh.copy_(Qd.cpu())
qn = qh.numpy()
ih = torch.empty((Q, k), dtype=torch.int64).pin_memory().numpy()
dh = torch.empty((Q, k), dtype=torch.float32).pin_memory().numpy()
ids = torch.empty((Q, k), dtype=torch.int64, device="cuda")
dd = torch.empty((Q, k), dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    ix.search_async(Qd, k, 1, ids, dd, s)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    ix.search_async(Qd, k, 1, ids, dd, s)
torch.cuda.synchronize()
t_dev = (time.perf_counter() - t0) / 10
parts_ms = {}
for parts in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["4"]):
    tri = parts.startswith("t")
    os.environ["CRISP_H2D_TRI"] = "1" if tri else "0"
    os.environ["CRISP_H2D_PARTS"] = parts.lstrip("t")
    for _ in range(3):
        crisp._check(crisp.lib().crisp_search(ix._h, crisp._ptr(qn), Q, k, 1, crisp._ptr(ih), crisp._ptr(dh)))
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        crisp._check(crisp.lib().crisp_search(ix._h, crisp._ptr(qn), Q, k, 1, crisp._ptr(ih), crisp._ptr(dh)))
        ts.append(time.perf_counter() - t0)
    parts_ms[parts] = round(float(np.median(ts)) * 1e3, 3)
    print("per-call ms", parts, [round(t * 1e3, 2) for t in ts], flush=True)
torch.cuda.synchronize()
hd = torch.empty((Q, D), dtype=torch.float32, device="cuda")
t0 = time.perf_counter()
for _ in range(10):
    hd.copy_(qh, non_blocking=True)
torch.cuda.synchronize()
t_h2d = (time.perf_counter() - t0) / 10
print({"device_ms": t_dev * 1e3, "host_ms_median_by_parts": parts_ms, "h2d_ms": t_h2d * 1e3,
       "same": bool(np.array_equal(ih, ids.cpu().numpy()))})
