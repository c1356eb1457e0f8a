"""The verification filter (DESIGN R17, crisp_set_verify_filter): a certified
lower bound of ||q' - x|| from the index's int8 copy (rows centred on the
column means, quantised per row) decides that a candidate cannot enter the
current top-k, so its fp32 row is not read.  The outputs
must not change: ids, distances and the patience stop with the filter on equal
those with it off and the oracle's (exact re-rank; patience,
P:L458), on inputs built to stress the bound (values at 2^-40 and 2^40 with
query components 2^-105 below them, a large common mean, near-duplicate rows
closer than the int8 resolution, exact integer ties)."""
import numpy as np
import pytest

import oracle
from test_gpu_parity import assert_topk_parity, build_gpu, compare_trace, make_case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def crisp():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build()
    import paper_2603_05180_b200 as c

    return c


def run_both(crisp, ix, Qv, k, mode):
    """(ids, d, trace, counters) with the filter on, then the same search with it off."""
    import torch

    out = []
    for on in (True, False):
        ix.set_verify_filter(on)
        crisp.set_stage_timing(True)
        crisp.search_counters(reset=True)
        ids, d, t = ix.trace(Qv, k, mode)
        ids2, d2 = ix.search(Qv, k, mode)
        cnt = crisp.search_counters(reset=True)
        crisp.set_stage_timing(False)
        torch.cuda.synchronize()
        assert np.array_equal(ids2, ids) and np.array_equal(d2, d), "untraced search"
        out.append((ids, d, t, cnt))
    ix.set_verify_filter(True)
    (i1, d1, t1, c1), (i0, d0, t0, c0) = out
    assert np.array_equal(i1, i0), "ids with and without the filter"
    assert np.array_equal(d1, d0), "distances with and without the filter"
    if mode == 1:
        assert np.array_equal(t1["n_verified"], t0["n_verified"]), "patience stop"
    assert c0["filter_rows"] == 0
    return i1, d1, t1, c1


@pytest.mark.parametrize("first,span", [(64, 2048), (64, 64), (128, 256), (512, 2048)])
@pytest.mark.parametrize("mode", [0, 1])
def test_filter_equals_exact(crisp, monkeypatch, mode, first, span):
    """Text-like data (the cfg4 stand-in at D = 256), k = 10 and 40: rounds of
    the filtered verification after a short exact round 0 (phi = 1), the
    two-pass re-rank (phi = 0); both against the oracle, trace included."""
    monkeypatch.setenv("CRISP_FILTER_ROUNDS", "2")  # also where P < 4 F (off by default there)
    monkeypatch.setenv("CRISP_LB_FIRST", str(first))
    monkeypatch.setenv("CRISP_LB_SPAN", str(span))
    monkeypatch.setenv("CRISP_ROUND_MIN", "32")
    X, Qv, ox = make_case(cfg=4, N=30000, D=256, Q=48, M=8, K=20, seed=3, rotation=1)
    ix = build_gpu(crisp, X, ox, block_ids=8192)
    for k, B, tau, P in ((10, 3000, 2, 40), (40, 6000, 1, 20)):
        ix.set_search_params(budget=B, tau=tau, patience_factor=P)
        ids, d, t, cnt = run_both(crisp, ix, Qv, k, mode)
        r_ids, r_d, ot = oracle.search(ox, Qv, k, mode, B, tau, patience_factor=P, trace=True)
        compare_trace(t, ot, mode, X.shape[0])
        assert_topk_parity(ids, d, r_ids, r_d, f"filter mode={mode} k={k}")
        assert cnt["filter_rows"] > 0, "the filter must engage"
        assert cnt["filter_exact"] < cnt["filter_rows"], "the filter must exclude rows"


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("scale_exp", [-40, 0, 40])
def test_filter_extreme_scales(crisp, monkeypatch, mode, scale_exp):
    """Data and queries scaled by 2^-40 / 2^40 (per-row power-of-two scales of
    the codes, fp64 digits of the query); at 2^40 two queries carry components
    far below the data's scale; a third variant adds a large common mean (the
    centring on the column means keeps the bound useful)."""
    monkeypatch.setenv("CRISP_FILTER_ROUNDS", "2")
    monkeypatch.setenv("CRISP_LB_FIRST", "64")
    monkeypatch.setenv("CRISP_LB_SPAN", "256")
    X, Qv, _ = make_case(cfg=1, N=12000, D=64, Q=32, M=4, K=12, seed=5)
    f = np.float32(2.0 ** scale_exp)
    X = X * f
    Qv = Qv * f
    if scale_exp > 0:
        Qv[:2, ::3] = np.float32(1.2345 * 2.0 ** (scale_exp - 145))
    if scale_exp == 0:
        X = X + np.float32(1000.0)
        Qv = Qv + np.float32(1000.0)
    ox = oracle.build(X, 4, K=12, rotation_mode=0, kmeans_iters=10, kmeans_sample=12000, seed=5)
    ix = build_gpu(crisp, X, ox, block_ids=4096)
    B, tau, k, P = 2500, 1, 10, 30
    ix.set_search_params(budget=B, tau=tau, patience_factor=P)
    ids, d, t, cnt = run_both(crisp, ix, Qv, k, mode)
    r_ids, r_d, ot = oracle.search(ox, Qv, k, mode, B, tau, patience_factor=P, trace=True)
    compare_trace(t, ot, mode, X.shape[0])
    assert_topk_parity(ids, d, r_ids, r_d, f"scale 2^{scale_exp}")
    assert cnt["filter_rows"] > 0


@pytest.mark.parametrize("mode", [0, 1])
def test_filter_near_duplicates_and_ties(crisp, monkeypatch, mode):
    """Rows that differ from the query, and from one another, by less than the
    int8 resolution (the bound cannot separate them: the exact rows decide),
    plus exact integer ties broken by id (d, id)."""
    monkeypatch.setenv("CRISP_FILTER_ROUNDS", "2")
    monkeypatch.setenv("CRISP_LB_FIRST", "64")
    monkeypatch.setenv("CRISP_LB_SPAN", "128")
    r = np.random.default_rng(11)
    N, D, M, K = 8000, 48, 4, 8
    X = r.integers(0, 3, (N, D)).astype(np.float32)
    base = r.standard_normal(D).astype(np.float32)
    X[:400] = base + (r.standard_normal((400, D)) * 1e-5).astype(np.float32)  # within int8 resolution
    X[400:800] = X[:400]  # exact duplicates: ties broken by id
    Qv = np.vstack([base[None, :] + (r.standard_normal((6, D)) * 1e-6).astype(np.float32),
                    r.integers(0, 3, (14, D)).astype(np.float32)]).astype(np.float32)
    ox = oracle.build(X, M, K=K, rotation_mode=0, kmeans_iters=8, kmeans_sample=N, seed=2)
    ix = crisp.Index.build(X, M, codebooks=ox["cb"], K=K)
    for B, tau, k, P in ((2000, 1, 20, 10), (N, 2, 50, 5)):
        ix.set_search_params(budget=B, tau=tau, patience_factor=P)
        ids, d, t, _ = run_both(crisp, ix, Qv, k, mode)
        r_ids, r_d, ot = oracle.search(ox, Qv, k, mode, B, tau, patience_factor=P, trace=True)
        compare_trace(t, ot, mode, N)
        assert np.array_equal(ids, r_ids), f"(d, id) order B={B}"


def test_filter_toggle_and_memory(crisp):
    """crisp_set_verify_filter frees and rebuilds the int8 copy (hbm_bytes
    follows: codes, 16 B of row terms, the column means), and an index built
    with CRISP_VERIFY_FILTER=0 has none."""
    import os

    X, Qv, ox = make_case(cfg=1, N=5000, D=64, Q=8, M=4, K=8, seed=1)
    ix = build_gpu(crisp, X, ox)
    h_on = ix.info()["hbm_bytes"]
    ix.set_verify_filter(False)
    h_off = ix.info()["hbm_bytes"]
    assert h_on - h_off == 5000 * 64 + 5000 * 16 + 64 * 4
    ix.set_verify_filter(True)
    assert ix.info()["hbm_bytes"] == h_on
    os.environ["CRISP_VERIFY_FILTER"] = "0"
    try:
        ix2 = build_gpu(crisp, X, ox)
    finally:
        os.environ.pop("CRISP_VERIFY_FILTER")
    assert ix2.info()["hbm_bytes"] == h_off
