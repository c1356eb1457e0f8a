"""Stage timings of one config under environment variants (perf experiments).
usage: python tools/stage_probe.py --cfg 2 --variants 'A=CRISP_COUNT_EMODE=0;B=CRISP_COUNT_EMODE=1'
A variant may set CRISP_BLOCK_IDS (forces a rebuild)."""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as ge  # noqa: E402
import synth  # noqa: E402
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=2)
ap.add_argument("--modes", default="0,1")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--variants", default="base=")
args = ap.parse_args()
ge.build()
import paper_2603_05180_b200 as crisp  # noqa: E402

c = synth.CONFIGS[args.cfg]
op = bench.load_op(args.cfg)
dev = torch.device("cuda", 0)
w = synth.Workload(args.cfg, device=dev)
X, Qd = w.base(c["N"]), w.queries(c["Q"])
k = c["k"]
ids = torch.empty((c["Q"], k), dtype=torch.int64, device=dev)
dd = torch.empty((c["Q"], k), dtype=torch.float32, device=dev)
stream = torch.cuda.current_stream().cuda_stream
index, index_bs = None, None
for var in args.variants.split(";"):
    name, _, assigns = var.partition("=")
    env = dict(a.split("=", 1) for a in assigns.split(",") if a)
    saved = {kk: os.environ.get(kk) for kk in env}
    os.environ.update(env)
    bs = os.environ.get("CRISP_BLOCK_IDS", "")
    if index is None or bs != index_bs:
        if index is not None:
            index.free()
        index = crisp.Index.build(X, op["M"], K=50, seed=op.get("seed", 1))
        index_bs = bs
    for mode in [int(m) for m in args.modes.split(",")]:
        if mode not in op["modes"]:
            continue
        mp = op["modes"][mode]
        index.set_search_params(beta=mp["beta"], alpha=mp["alpha"], patience_factor=int(os.environ.get("PROBE_PF", "40")))
        if mode == 1:
            index.set_adsampling(os.environ.get("PROBE_AD", "0") == "1")
        index.search_async(Qd, k, mode, ids, dd, stream)
        torch.cuda.synchronize()
        crisp.stage_times(reset=True)
        crisp.search_counters(reset=True)
        crisp.set_stage_timing(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            index.search_async(Qd, k, mode, ids, dd, stream)
        e1.record()
        torch.cuda.synchronize()
        st = crisp.stage_times(reset=True)
        cnt = crisp.search_counters(reset=True)
        crisp.set_stage_timing(False)
        ms = e0.elapsed_time(e1) / args.reps
        print(json.dumps({"variant": name, "env": env, "mode": mode, "ms": ms, "qps": c["Q"] / ms * 1e3,
                          "stages": {kk: v / args.reps for kk, v in st.items()},
                          "counters": {kk: v / args.reps for kk, v in cnt.items()}}), flush=True)
    for kk, v in saved.items():
        if v is None:
            os.environ.pop(kk, None)
        else:
            os.environ[kk] = v
