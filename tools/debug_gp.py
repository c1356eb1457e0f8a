"""Round-by-round trace of the global-patience emulation (debugging aid)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import __graft_entry__ as ge  # noqa: E402

ge.build()
import paper_2603_05180_b200 as crisp  # noqa: E402
from paper_2603_05180_b200 import dist  # noqa: E402
from test_gpu_parity import build_gpu, make_case  # noqa: E402
from test_gpu_global_patience import shard_indexes  # noqa: E402

os.environ.update(CRISP_GP_MIN="32", CRISP_GP_MAX="64", CRISP_PATIENCE_FIRST="32")
X, Qv, ox = make_case(cfg=4, N=24000, D=128, Q=40, M=8, K=16, seed=5, rotation=1)
G = 2
shards, bases = shard_indexes(crisp, X, ox, G)
for s in shards:
    s.set_verify_filter(False)
    s.set_search_params(budget=2500, tau=2, patience_factor=30)
dev = torch.device("cuda", 0)
q = torch.from_numpy(Qv).to(dev)
engines = []
for s in shards:
    e = dist.CudaEngine(crisp, dev)
    e.index = s
    engines.append(e)
k = 10
counts = [e.begin(q, k, 1) for e in engines]
gc = torch.stack(counts).sum(0).to(torch.int32)
print("global |C|", gc[:8].tolist())
hists = torch.stack([e.hist(gc) for e in engines])
hh = torch.stack([e.gp_order(gc, hists, G, r) for r, e in enumerate(engines)])
print("hh sums", hh.sum(2)[:, :8].tolist())
for r, e in enumerate(engines):
    e.gp_prepare(hh, G, r, bases)
for rnd in range(30):
    ns = [e.gp_round() for e in engines]
    stride = max(1, max(ns))
    got = [e.gp_fetch(stride) for e in engines]
    all_ent = torch.stack([g_[0] for g_ in got])
    all_cnt = torch.stack([g_[1] for g_ in got])
    running = [e.gp_replay(all_cnt, all_ent, stride, G) for e in engines]
    print("round", rnd, "entries", ns, "counts q0..3", all_cnt[:, :4].tolist(), "running", running)
    if running[0] == 0:
        break
