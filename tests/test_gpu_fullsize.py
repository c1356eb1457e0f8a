"""Parity at BASELINE.json's full size, in the launch configuration bench.py
times (cfg2: N=1M, D=960, Q=10k, k=10, M=16, both modes at the operating
point), on sampled outputs the oracle computes one by one.  The oracle builds
the index itself (its R, its codebooks, its X' = XR); the GPU index is built
with crisp_build_with from the oracle's R and codebooks, so X', cells and CSR
must come out bit-identical, and the sampled queries' results must match."""
import json
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def setup():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build()
    import paper_2603_05180_b200 as crisp

    op = json.load(open(os.path.join(ROOT, "configs", "operating_points.json")))["2"]
    c = synth.CONFIGS[2]
    w = synth.Workload(2, device="cuda")
    Xd, Qd = w.base(c["N"]), w.queries(c["Q"])
    X, Qh = Xd.cpu().numpy(), Qd.cpu().numpy()
    ox = oracle.build(X, op["M"], K=50, kmeans_iters=20, kmeans_sample=100000, seed=op["seed"])
    assert ox["rotated"]
    ix = crisp.Index.build(Xd, op["M"], R=ox["R"], codebooks=ox["cb"], K=50, seed=op["seed"])
    return crisp, ix, ox, Xd, Qd, Qh, op, c


def test_fullsize_index_bit_exact(setup):
    crisp, ix, ox, *_ = setup
    e = ix.export()
    for name, ref in (("X", ox["X"]), ("cells", ox["cells"]), ("offsets", ox["off"]), ("ids", ox["ids"]),
                      ("codes", ox["codes"])):
        assert np.array_equal(e[name], ref), name


@pytest.mark.parametrize("mode", [0, 1])
def test_fullsize_sampled_queries(setup, mode):
    import torch

    crisp, ix, ox, Xd, Qd, Qh, op, c = setup
    mp = op["modes"][str(mode)]
    ix.set_search_params(beta=mp["beta"], alpha=mp["alpha"], patience_factor=40)
    k = c["k"]
    ids = torch.empty((c["Q"], k), dtype=torch.int64, device="cuda")
    dd = torch.empty((c["Q"], k), dtype=torch.float32, device="cuda")
    ix.search_async(Qd, k, mode, ids, dd, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    sample = np.random.default_rng(mode).choice(c["Q"], 40, replace=False)
    B, tau = oracle.budget_ids(mp["beta"], c["N"]), oracle.tau_int(mp["alpha"], op["M"])
    r_ids, r_d, _ = oracle.search(ox, Qh[sample], k, mode, B, tau, patience_factor=40)
    g_ids, g_d = ids.cpu().numpy()[sample], dd.cpu().numpy()[sample]
    assert np.array_equal(g_ids, r_ids)
    assert np.all(np.abs(g_d - r_d) <= 1e-5 * np.abs(r_d))
