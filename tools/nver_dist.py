import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import __graft_entry__ as ge, synth, bench
ge.build()
import paper_2603_05180_b200 as crisp
c = synth.CONFIGS[2]; op = bench.load_op(2)
w = synth.Workload(2, device="cuda")
X, Qd = w.base(c["N"]), w.queries(2000)
ix = crisp.Index.build(X, op["M"], K=50, seed=op.get("seed", 1))
mp = op["modes"][1]
ix.set_search_params(beta=mp["beta"], alpha=mp["alpha"], patience_factor=40)
_, _, t = ix.trace(Qd.cpu().numpy(), 10, 1)
nv = t["n_verified"]; cn = t["cand_n"]
print("nver quantiles", np.percentile(nv, [0, 10, 25, 50, 75, 90, 95, 99, 100]).tolist(), "mean", nv.mean())
print("cand quantiles", np.percentile(cn, [0, 10, 50, 90, 100]).tolist())
for S in (256, 384, 512, 640, 768, 1024):
    print(S, "frac>S", float((nv > S).mean()), "rows if round0=S then exact:", float(np.minimum(nv, 10**9).mean()), "round0 waste", float(np.maximum(0, np.minimum(cn, S) - nv).mean()))
