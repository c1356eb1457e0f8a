"""Projected multi-GPU step of the point-sharded search at cfg4 (Optimized Mode
with exact global patience, Guaranteed Mode with the exact global fallback),
measured by running the G ranks' kernels one after another on ONE GPU.

Every engine call of every rank is bracketed by CUDA events; a rank's compute
time is the sum of its calls.  The projected step at G GPUs is the slowest
rank's compute plus the collectives, modelled from their measured sizes as
latency + bytes / bandwidth (one all-reduce, then all-gathers; --bw GB/s per
rank, --lat us per collective).  Results must equal the single index (checked).
usage: python tools/gp_scale_probe.py --G 2,4,8 [--modes 1,0] [--Q 10000]"""
import argparse
import json
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

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=4)
ap.add_argument("--G", default="2,4,8")
ap.add_argument("--modes", default="1,0")
ap.add_argument("--Q", type=int, default=None)
ap.add_argument("--bw", type=float, default=400.0, help="all-gather bandwidth per rank, GB/s (model)")
ap.add_argument("--lat", type=float, default=30.0, help="latency per collective, us (model)")
ap.add_argument("--sharded-a0", type=int, default=1, help="a0 sharded by query + all-gather of q' (dist N9)")
args = ap.parse_args()
ge.build()
import paper_2603_05180_b200 as crisp  # noqa: E402
from paper_2603_05180_b200 import dist  # noqa: E402

c = synth.CONFIGS[args.cfg]
op = bench.load_op(args.cfg)
M = op["M"]
dev = torch.device("cuda", 0)
w = synth.Workload(args.cfg, device=dev)
N, k = c["N"], c["k"]
X, Qd = w.base(N), w.queries(args.Q or c["Q"])
Q = Qd.shape[0]
# the model (R, codebooks) of a build over all rows, from the counter-based samples (crisp_build_model)
seed = op.get("seed", 1)
cev_ids, km_ids = crisp.model_samples(N, seed, 100000)
R, cb, _ = crisp.build_model(X[torch.from_numpy(cev_ids.astype(np.int64)).to(dev)].cpu().numpy(),
                             X[torch.from_numpy(km_ids.astype(np.int64)).to(dev)].cpu().numpy(), M, K=50, seed=seed)
full = crisp.Index.build(X, M, R=R, codebooks=cb, K=50, seed=seed)
stream = torch.cuda.current_stream().cuda_stream


def timed(fn, *a):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn(*a)
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)


def coll(nbytes_per_rank, G):
    """ms of one all-gather of nbytes_per_rank from each of G ranks (model)."""
    return args.lat * 1e-3 + nbytes_per_rank * (G - 1) / (args.bw * 1e9) * 1e3


modes = [int(m) for m in args.modes.split(",")]
single = {}
for mode in modes:  # the single index first (then freed: the G shard sessions need the memory)
    mp = op["modes"][mode]
    full.set_search_params(beta=mp["beta"], alpha=mp["alpha"], patience_factor=mp.get("patience_factor", 40))
    ids1 = torch.empty((Q, k), dtype=torch.int64, device=dev)
    dd1 = torch.empty((Q, k), dtype=torch.float32, device=dev)
    for _ in range(3):  # warm-up (the first searches of a process are slower)
        full.search_async(Qd, k, mode, ids1, dd1, stream)
    torch.cuda.synchronize()
    t1 = min(timed(full.search_async, Qd, k, mode, ids1, dd1, stream)[1] for _ in range(3))
    single[mode] = (ids1, t1)
full.free()
torch.cuda.empty_cache()
rows = []
for mode in modes:
    mp = op["modes"][mode]
    ids1, t1 = single[mode]
    for G in [int(g) for g in args.G.split(",")]:
        shards, bases = [], []
        for r in range(G):
            lo, hi = dist.shard_range(N, r, G)
            shards.append(crisp.Index.build(X[lo:hi], M, R=R, codebooks=cb, K=50, gid_base=lo,
                                            workspace_bytes=150 * 2**30 // G))
            bases.append(lo)
        sizes = sum(s.local_cell_sizes() for s in shards)
        engines = []
        for s in shards:
            s.set_global_cell_sizes(sizes)
            s.set_search_params(beta=mp["beta"], alpha=mp["alpha"], patience_factor=mp.get("patience_factor", 40))
            e = dist.CudaEngine(crisp, dev)
            e.index = s
            engines.append(e)
        for rep in range(2):  # the second repetition is timed
            t = np.zeros(G)
            comm = 0.0
            counts = []
            if args.sharded_a0:  # N9: each rank transforms its slice, one all-gather of q'
                per = (Q + G - 1) // G
                parts = []
                for r, e in enumerate(engines):
                    qr, ms = timed(e.transform, Qd[min(Q, r * per):min(Q, (r + 1) * per)])
                    parts.append(qr)
                    t[r] += ms
                qrot = torch.cat(parts).contiguous()
                comm += coll(per * qrot.shape[1] * 4, G)
                for r, e in enumerate(engines):
                    cnt, ms = timed(e.begin_transformed, qrot, k, mode)
                    counts.append(cnt)
                    t[r] += ms
            else:
                for r, e in enumerate(engines):
                    cnt, ms = timed(e.begin, Qd, k, mode)
                    counts.append(cnt)
                    t[r] += ms
            gc = torch.stack(counts).sum(0).to(torch.int32)
            comm += coll(4 * Q, G)  # all-reduce of |C_q| (counted as one all-gather)
            hs = []
            for r, e in enumerate(engines):
                h, ms = timed(e.hist, gc)
                hs.append(h)
                t[r] += ms
            hists = torch.stack(hs)
            comm += coll(hists[0].numel() * 4, G)
            n_rounds = 0
            if mode == 1:
                hh = []
                for r, e in enumerate(engines):
                    x, ms = timed(e.gp_order, gc, hists, G, r)
                    hh.append(x)
                    t[r] += ms
                hh = torch.stack(hh)
                comm += coll(hh[0].numel() * 4, G)
                for r, e in enumerate(engines):
                    _, ms = timed(e.gp_prepare, hh, G, r, bases)
                    t[r] += ms
                while True:
                    ns = []
                    for r, e in enumerate(engines):
                        n, ms = timed(e.gp_round)
                        ns.append(n)
                        t[r] += ms
                    stride = max(1, max(ns))
                    got = [e.gp_fetch(stride) for e in engines]
                    all_ent = torch.stack([g_[0] for g_ in got])
                    all_cnt = torch.stack([g_[1] for g_ in got])
                    comm += coll(8, G) + coll(4 * Q, G) + coll(16 * stride, G)
                    run = []
                    for r, e in enumerate(engines):
                        x, ms = timed(e.gp_replay, all_cnt, all_ent, stride, G)
                        run.append(x)
                        t[r] += ms
                    n_rounds += 1
                    if run[0] == 0:
                        break
                res = []
                for r, e in enumerate(engines):
                    x, ms = timed(e.gp_result)
                    res.append(x)
                    t[r] += ms
                ids_g = res[0][0]
            else:
                outs = []
                for r, e in enumerate(engines):
                    x, ms = timed(e.finish, gc, hists, G, r)
                    outs.append(x)
                    t[r] += ms
                comm += coll(16 * Q * k, G)
                ids_g, _ = engines[0].merge(torch.stack([o[1] for o in outs]), torch.stack([o[0] for o in outs]))
                t[0] += 0.0
        same = bool(torch.equal(ids_g, ids1))
        step = float(t.max()) + comm
        row = dict(cfg=args.cfg, mode=mode, G=G, Q=Q, single_ms=t1, rank_ms=[round(x, 3) for x in t],
                   comm_model_ms=round(comm, 3), projected_step_ms=round(step, 3),
                   projected_qps=Q / step * 1e3, speedup=t1 / step, rounds=n_rounds, equal_to_single=same,
                   model=f"all-gather {args.bw} GB/s per rank, {args.lat} us per collective",
                   sharded_a0=bool(args.sharded_a0))
        print(json.dumps(row), flush=True)
        rows.append(row)
        for s in shards:
            s.free()
        torch.cuda.empty_cache()
