"""Is the synthetic data and the GPU build deterministic run to run?
usage: python tools/determinism.py CFG [N]"""
import hashlib
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as ge  # noqa: E402
import synth  # noqa: E402
import bench  # noqa: E402

cfg = int(sys.argv[1])
c = synth.CONFIGS[cfg]
N = int(sys.argv[2]) if len(sys.argv) > 2 else c["N"]
ge.build()
import paper_2603_05180_b200 as crisp  # noqa: E402


def h(t):
    a = t.cpu().numpy() if torch.is_tensor(t) else np.asarray(t)
    return hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()[:12]


op = bench.load_op(cfg)
hs = []
for rep in range(2):
    w = synth.Workload(cfg, device=torch.device("cuda", 0))
    X = w.base(N)
    ix = crisp.Index.build(X, op["M"], K=50, seed=op.get("seed", 1))
    e = ix.export()
    row = {"X": h(X), "cb": h(e["codebooks"]), "cells": h(e["cells"]), "ids": h(e["ids"]),
           "offsets": h(e["offsets"]), "Xrot": h(e["X"]), "info": ix.info()["cev"]}
    print(rep, row, flush=True)
    hs.append(row)
    ix.free()
    del X, e
    torch.cuda.empty_cache()
print("identical" if hs[0] == hs[1] else "DIFFERENT")
