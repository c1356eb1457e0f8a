"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, stage by
stage and end to end, on seeded inputs that span several id blocks and ragged
tails.  Integer/index outputs must be bit-exact; distances within 1e-5
relative (north star).  A top-k mismatch is accepted only as a documented
near-tie: the oracle's own dist64 values of the swapped ids differ by at most
1e-12 relative; every such case is counted and none is
expected on these inputs."""
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

NEAR_TIE_REL = 1e-12


@pytest.fixture(scope="module")
def crisp():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build()
    import paper_2603_05180_b200 as c

    return c


def assert_topk_parity(ids, d, ref_ids, ref_d, what=""):
    ids, ref_ids = np.asarray(ids), np.asarray(ref_ids)
    d, ref_d = np.asarray(d, np.float64), np.asarray(ref_d, np.float64)
    assert ids.shape == ref_ids.shape
    fin = np.isfinite(ref_d)
    assert np.array_equal(np.isfinite(d), fin), what
    assert np.all(np.abs(d[fin] - ref_d[fin]) <= 1e-5 * np.abs(ref_d[fin])), what
    bad = np.nonzero(np.any(ids != ref_ids, axis=1))[0]
    for q in bad:
        # only swaps among (oracle) near-tied distances are allowed
        for i in np.nonzero(ids[q] != ref_ids[q])[0]:
            rel = abs(d[q, i] - ref_d[q, i]) / max(ref_d[q, i], 1e-300)
            assert rel <= NEAR_TIE_REL * 10, f"{what}: query {q} pos {i} not a near-tie"
    assert len(bad) == 0, f"{what}: {len(bad)} near-tie rows (documented, none expected here)"


def make_case(cfg=1, N=20000, D=None, Q=100, M=8, K=50, seed=0, rotation=0, kmeans_iters=10):
    w = synth.Workload(cfg, D=D)
    X = w.base(N).numpy()
    Qv = w.queries(Q).numpy()
    ox = oracle.build(X, M, K=K, rotation_mode=rotation, kmeans_iters=kmeans_iters, kmeans_sample=20000, seed=seed)
    return X, Qv, ox


def build_gpu(crisp, X, ox, block_ids=None, **kw):
    if block_ids:
        os.environ["CRISP_BLOCK_IDS"] = str(block_ids)
    try:
        return crisp.Index.build(X, ox["M"], R=ox["R"], codebooks=ox["cb"], K=ox["K"], **kw)
    finally:
        os.environ.pop("CRISP_BLOCK_IDS", None)


def compare_index(ix, ox):
    e = ix.export()
    assert np.array_equal(e["X"], ox["X"]), "stored (rotated) vectors"
    assert np.array_equal(e["cells"], ox["cells"]), "cell assignment"
    assert np.array_equal(e["offsets"], ox["off"]), "CSR offsets"
    assert np.array_equal(e["ids"], ox["ids"]), "CSR ids"
    assert np.array_equal(e["codes"], ox["codes"]), "binary codes"


def compare_trace(t, ot, mode, N):
    Q = t["act_len"].shape[0]
    assert np.array_equal(t["qrot"], ot["qrot"]), "a0 q'"
    assert np.array_equal(t["act_len"], ot["act_len"]), "a2 activated counts"
    for q in range(Q):
        for m in range(t["act_len"].shape[1]):
            L = t["act_len"][q, m]
            assert np.array_equal(t["act_cell"][q, m, :L], ot["act_cell"][q, m, :L]), "a2 pop order"
            assert np.array_equal(t["act_w"][q, m, :L], ot["act_w"][q, m, :L]), "a2 weights"
    assert np.array_equal(t["retrieved"], ot["retrieved"]), "a2 retrieved"
    assert np.array_equal(t["V"].astype(np.uint16), ot["V"]), "a3 collision scores"
    assert np.array_equal(t["fallback"], ot["fallback"]), "a4 fallback"
    assert np.array_equal(t["cand_n"], ot["cand_n"]), "a4 |C|"
    for q in range(Q):
        n = t["cand_n"][q]
        assert np.array_equal(t["cand"][q, :n], ot["cand"][q, :n]), "a4 C_q"
        if mode == 1:
            assert np.array_equal(t["order"][q, :n], ot["order"][q, :n]), "a4 Hamming order"
    if mode == 1:
        assert np.array_equal(t["n_verified"], ot["n_verified"]), "a5 patience stop"


# collision-count variants: CTA-flattened, warp-owned with byte load/store
# pairs (+ standalone dense Hamming at phi=1), warp-owned with shared atomics
# and the Hamming popcounts fused; the row
# kernels run two-row steps in the first and one CTA per query in the last
COUNT_VARIANTS = {"select": {"CRISP_COUNT_KERNEL": "0", "CRISP_ROWS4": "0"},
                  "warp": {"CRISP_COUNT_KERNEL": "1", "CRISP_HAMMING_FUSED": "0"},
                  "warp_fused": {"CRISP_COUNT_KERNEL": "1", "CRISP_HAMMING_FUSED": "1", "CRISP_RERANK_SPLITS": "1",
                                 "CRISP_COUNT_ATOM": "1"},
                 # fragment-flattened count (the small-cell default) with 1, 2 and 4 id blocks per CTA
                 "frag": {"CRISP_COUNT_KERNEL": "2"},
                 "frag_f1": {"CRISP_COUNT_KERNEL": "2", "CRISP_COUNT_F": "1"},
                 "frag_f4": {"CRISP_COUNT_KERNEL": "2", "CRISP_COUNT_F": "4"},
                 # crossing bits from the atomics' returns (CRISP_COUNT_SWAR=0) instead of the scan
                 "frag_cross": {"CRISP_COUNT_KERNEL": "2", "CRISP_COUNT_SWAR": "0"},
                 "frag_fused": {"CRISP_COUNT_KERNEL": "2", "CRISP_HAMMING_FUSED": "1"},
                 # reductions without return + the final SWAR threshold scan (the default) with 4 blocks
                 "frag_swar_f4": {"CRISP_COUNT_KERNEL": "2", "CRISP_COUNT_SWAR": "1", "CRISP_COUNT_F": "4"},
                 # the grouped Guaranteed-Mode re-rank (k_rerank_group) after either count kernel
                 "frag_group": {"CRISP_COUNT_KERNEL": "2", "CRISP_RERANK_GROUP": "1"},
                 "warp_group": {"CRISP_COUNT_KERNEL": "1", "CRISP_RERANK_GROUP": "1"}}


@pytest.mark.parametrize("variant", list(COUNT_VARIANTS))
@pytest.mark.parametrize("mode", [0, 1])
def test_cfg1_stagewise(crisp, monkeypatch, mode, variant):
    """BASELINE configs[0] (PR1: N=20k, D=256, Q=100, k=10) in full, M=8;
    every collision-count variant."""
    for k_, v_ in COUNT_VARIANTS[variant].items():
        monkeypatch.setenv(k_, v_)
    X, Qv, ox = make_case()
    ix = build_gpu(crisp, X, ox)
    compare_index(ix, ox)
    B, tau, k = oracle.budget_ids(0.01, 20000), 3, 10
    ix.set_search_params(budget=B, tau=tau, patience_factor=40)
    ids, d, t = ix.trace(Qv, k, mode)
    r_ids, r_d, ot = oracle.search(ox, Qv, k, mode, B, tau, patience_factor=40, trace=True)
    compare_trace(t, ot, mode, X.shape[0])
    assert_topk_parity(ids, d, r_ids, r_d, f"cfg1 mode {mode}")
    # the untraced path gives the same answer
    ids2, d2 = ix.search(Qv, k, mode)
    assert np.array_equal(ids2, ids) and np.array_equal(d2, d)


@pytest.mark.parametrize("variant", list(COUNT_VARIANTS))
@pytest.mark.parametrize("mode", [0, 1])
def test_rotated_multiblock_ragged(crisp, monkeypatch, mode, variant):
    """Rotation injected (R from the oracle), 5 id blocks with a ragged tail,
    D not a multiple of 2M (zero padding), K=31."""
    for k_, v_ in COUNT_VARIANTS[variant].items():
        monkeypatch.setenv(k_, v_)
    X, Qv, ox = make_case(cfg=2, N=18001, D=90, Q=40, M=4, K=31, rotation=1, seed=3)
    assert ox["rotated"] and ox["Dp"] == 96
    ix = build_gpu(crisp, X, ox, block_ids=4096)
    assert ix.info()["n_blocks"] == 5
    compare_index(ix, ox)
    B, tau, k = 700, 2, 7
    ix.set_search_params(budget=B, tau=tau, patience_factor=3)
    ids, d, t = ix.trace(Qv, k, mode)
    r_ids, r_d, ot = oracle.search(ox, Qv, k, mode, B, tau, patience_factor=3, trace=True)
    compare_trace(t, ot, mode, X.shape[0])
    assert_topk_parity(ids, d, r_ids, r_d, "rotated")


@pytest.mark.parametrize("variant", list(COUNT_VARIANTS))
@pytest.mark.parametrize("mode", [0, 1])
def test_full_blocks_ragged_tail(crisp, monkeypatch, mode, variant):
    """Full 32768-id counter blocks (4096 counters per warp) with a ragged
    third block, stage by stage."""
    for k_, v_ in COUNT_VARIANTS[variant].items():
        monkeypatch.setenv(k_, v_)
    X, Qv, ox = make_case(cfg=1, N=70001, D=64, Q=24, M=4, K=16, seed=5)
    ix = build_gpu(crisp, X, ox, block_ids=32768)
    assert ix.info()["n_blocks"] == 3
    B, tau, k = 9000, 2, 10
    ix.set_search_params(budget=B, tau=tau, patience_factor=3)
    ids, d, t = ix.trace(Qv, k, mode)
    r_ids, r_d, ot = oracle.search(ox, Qv, k, mode, B, tau, patience_factor=3, trace=True)
    compare_trace(t, ot, mode, X.shape[0])
    assert_topk_parity(ids, d, r_ids, r_d, "full blocks")
    ids2, d2 = ix.search(Qv, k, mode)
    assert np.array_equal(ids2, ids) and np.array_equal(d2, d)


@pytest.mark.parametrize("kernel", ["1", "2", "frag_cross"])
@pytest.mark.parametrize("mode", [0, 1])
def test_many_subspaces_wide_counters(crisp, monkeypatch, mode, kernel):
    """M=64 (scores up to 2M=128 do not fit the 7-bit SWAR compare: the
    __vcmpgeu4 path of the threshold scan), stage by stage."""
    if kernel in COUNT_VARIANTS:
        for k_, v_ in COUNT_VARIANTS[kernel].items():
            monkeypatch.setenv(k_, v_)
    else:
        monkeypatch.setenv("CRISP_COUNT_KERNEL", kernel)
    X, Qv, ox = make_case(cfg=1, N=9001, D=256, Q=16, M=64, K=6, seed=7)
    ix = build_gpu(crisp, X, ox, block_ids=4096)
    B, tau, k = 1500, 30, 10
    ix.set_search_params(budget=B, tau=tau, patience_factor=2)
    ids, d, t = ix.trace(Qv, k, mode)
    r_ids, r_d, ot = oracle.search(ox, Qv, k, mode, B, tau, patience_factor=2, trace=True)
    compare_trace(t, ot, mode, X.shape[0])
    if mode == 1:
        assert int(ot["V"].max()) >= 64, "scores above 63 exercise the wide compare"
    assert_topk_parity(ids, d, r_ids, r_d, "M=64")


@pytest.mark.parametrize("F", ["1", "2"])
@pytest.mark.parametrize("mode", [0, 1])
def test_count_frag_chunked_entries(crisp, monkeypatch, mode, F):
    """k_count_frag with more activated cells than one staging chunk holds
    (M=32 subspaces x 256 cells, budget = N: 8192 activated cells per query, 4
    chunks), weights 2 on the first k ranks, a 3-block ragged id range."""
    monkeypatch.setenv("CRISP_COUNT_KERNEL", "2")
    monkeypatch.setenv("CRISP_COUNT_F", F)
    X, Qv, ox = make_case(cfg=1, N=9001, D=128, Q=6, M=32, K=16, seed=11, kmeans_iters=4)
    ix = build_gpu(crisp, X, ox, block_ids=4096)
    assert ix.info()["n_blocks"] == 3
    N = X.shape[0]
    for B, tau, k in ((N, 40, 10), (2500, 5, 10)):
        ix.set_search_params(budget=B, tau=tau, patience_factor=2)
        ids, d, t = ix.trace(Qv, k, mode)
        r_ids, r_d, ot = oracle.search(ox, Qv, k, mode, B, tau, patience_factor=2, trace=True)
        compare_trace(t, ot, mode, N)
        assert_topk_parity(ids, d, r_ids, r_d, f"frag chunks B={B}")
    assert int(t["act_len"].sum(axis=1).max()) == 32 * 256 or B != N


@pytest.mark.parametrize("group", ["0", "1"])
@pytest.mark.parametrize("mode", [0, 1])
def test_fallback_and_small_k(crisp, monkeypatch, mode, group):
    """tau above every reachable score -> the underflow fallback;
    Guaranteed Mode through both re-rank kernels (the fallback's candidates sit
    in one segment spanning every id range of the grouped kernel)."""
    monkeypatch.setenv("CRISP_RERANK_GROUP", group)
    X, Qv, ox = make_case(cfg=3, N=9000, D=64, Q=30, M=4, K=12, seed=5)
    ix = build_gpu(crisp, X, ox, block_ids=4096)
    for k, tau in ((5, 9), (1, 4), (64, 3)):
        ix.set_search_params(budget=120, tau=tau, patience_factor=2)
        ids, d, t = ix.trace(Qv, k, mode)
        r_ids, r_d, ot = oracle.search(ox, Qv, k, mode, 120, tau, patience_factor=2, trace=True)
        compare_trace(t, ot, mode, X.shape[0])
        assert_topk_parity(ids, d, r_ids, r_d, f"fallback k={k} tau={tau}")
    assert ot["fallback"].any()


@pytest.mark.parametrize("variant", list(COUNT_VARIANTS))
@pytest.mark.parametrize("mode", [0, 1])
def test_k100_text_like(crisp, monkeypatch, mode, variant):
    """k = 100 (cfg4's k) on a cfg4-like rotated, normalised low-rank case:
    the per-warp top-k lists, their merge and the patience scan at k = 100,
    against the oracle end to end and stage by stage."""
    for k_, v_ in COUNT_VARIANTS[variant].items():
        monkeypatch.setenv(k_, v_)
    X, Qv, ox = make_case(cfg=4, N=30000, D=192, Q=20, M=8, K=24, rotation=1, seed=9)
    ix = build_gpu(crisp, X, ox, block_ids=8192)
    B, tau, k = 1500, 3, 100
    ix.set_search_params(budget=B, tau=tau, patience_factor=4)
    ids, d, t = ix.trace(Qv, k, mode)
    r_ids, r_d, ot = oracle.search(ox, Qv, k, mode, B, tau, patience_factor=4, trace=True)
    compare_trace(t, ot, mode, X.shape[0])
    assert_topk_parity(ids, d, r_ids, r_d, "k=100")
    ids2, d2 = ix.search(Qv, k, mode)
    assert np.array_equal(ids2, ids) and np.array_equal(d2, d)


def test_full_coverage_is_exact_knn(crisp):
    X, Qv, ox = make_case(cfg=1, N=6000, D=128, Q=25, M=4, K=10)
    ix = build_gpu(crisp, X, ox)
    ix.set_search_params(budget=6000, tau=1)
    ids, d = ix.search(Qv, 10, 0)
    b_ids, b_d = oracle.bruteforce_knn(ox["X"], Qv, 10)
    assert_topk_parity(ids, d, b_ids, b_d, "full coverage")
    # self queries come first with distance exactly 0
    ids, d = ix.search(X[[3, 999, 5999]], 3, 0)
    assert ids[:, 0].tolist() == [3, 999, 5999] and np.all(d[:, 0] == 0.0)


def test_edge_cases(crisp):
    X, Qv, ox = make_case(cfg=1, N=700, D=32, Q=3, M=2, K=4)
    ix = build_gpu(crisp, X, ox)
    ix.set_search_params(budget=50, tau=1)
    ids, d = ix.search(Qv[:0], 5, 0)  # Q = 0
    assert ids.shape == (0, 5)
    # k larger than every candidate set -> padding (-1, +inf)
    ids, d = ix.search(Qv, 600, 0)
    r_ids, r_d, _ = oracle.search(ox, Qv, 600, 0, 50, 1)
    assert_topk_parity(ids, d, r_ids, r_d, "padding")
    assert (ids == -1).any() and np.isinf(d[ids == -1]).all()
    with pytest.raises(crisp.CrispError):
        ix.search(Qv, 0, 0)
    with pytest.raises(crisp.CrispError):
        ix.search(Qv, 701, 0)


def test_gpu_build_matches_oracle_build(crisp):
    """crisp_build end to end (no injection), unrotated data: the sample, the
    k-means++ seeding, Lloyd and the assignment follow the oracle's order, so
    the codebooks and the CSR come out identical; CEV agrees to 1e-9."""
    w = synth.Workload(5, D=128)
    X = w.base(12000).numpy()
    ox = oracle.build(X, 4, K=16, rotation_mode=-1, kmeans_iters=6, kmeans_sample=5000, seed=9)
    assert not ox["rotated"]
    ix = crisp.Index.build(X, 4, K=16, kmeans_iters=6, kmeans_sample=5000, seed=9)
    info = ix.info()
    assert abs(info["cev"] - ox["cev"]) < 1e-9 and info["rotated"] == 0
    e = ix.export()
    assert np.array_equal(e["codebooks"], ox["cb"]), "k-means codebooks"
    compare_index(ix, ox)


def test_kmeanspp_parallel_pick_matches_sequential(crisp, monkeypatch):
    """The certified parallel k-means++ pick (k_kpp_pick_par) against the
    oracle-order sequential kernel (CRISP_KPP_SEQ=1): the GPU's own builds must
    give bit-identical codebooks, cells and CSR on a 60k-point sample."""
    w = synth.Workload(2, D=128)
    X = w.base(60000).numpy()
    a = crisp.Index.build(X, 4, K=50, rotation=0, kmeans_iters=4, seed=5)
    ea = a.export()
    monkeypatch.setenv("CRISP_KPP_SEQ", "1")
    b = crisp.Index.build(X, 4, K=50, rotation=0, kmeans_iters=4, seed=5)
    eb = b.export()
    for name in ("codebooks", "cells", "offsets", "ids"):
        assert np.array_equal(ea[name], eb[name]), name


def test_gpu_rotation_properties(crisp):
    """Rotation forced on: R orthogonal (fp32 storage, 1e-5), close to the
    oracle's R (same Philox G; QR by cuSOLVER vs Householder), and the CEV gate
     fires on strongly correlated data."""
    w = synth.Workload(2, D=96)
    X = w.base(4000).numpy()
    ox = oracle.build(X, 4, K=8, rotation_mode=1, kmeans_iters=3, seed=4)
    ix = crisp.Index.build(X, 4, K=8, rotation=1, kmeans_iters=3, seed=4)
    e = ix.export()
    R = e["R"].astype(np.float64)
    assert np.abs(R @ R.T - np.eye(96)).max() < 1e-5
    assert np.abs(R - ox["R"]).max() < 1e-5
    auto = crisp.Index.build(X, 4, K=8, kmeans_iters=2, seed=4)
    assert auto.info()["rotated"] == (ox["cev"] > 0.85) == 1


@pytest.mark.parametrize("gemm", ["tcgen05", "cublaslt"])
@pytest.mark.parametrize("D,M", [(203, 4), (100, 3)])
def test_certified_rotation_adversarial(crisp, monkeypatch, D, M, gemm):
    """a0 on the int8 tensor cores with the certified rounding (rotate_imma.cu):
    q' must equal the oracle's sequential fp64 chain bit for bit on rows chosen
    to stress the certificate: zeros, a single non-zero, 60 orders of magnitude
    inside one row, subnormal inputs, power-of-two scalings, alternating signs,
    exact cancellations, and padded dimensions (D' = 208 and D' = 102, whose
    digit planes pad to 256 and 128: 2 and 1 k-blocks, 4 and 2 column tiles,
    ragged 128-row tiles).  Both level-GEMM engines: the hand-written tcgen05
    kernel with the fused certificate (default) and cuBLASLt + k_certify."""
    if gemm == "cublaslt":
        monkeypatch.setenv("CRISP_ROTATE_GEMM", "cublaslt")
    rng = np.random.default_rng(11)
    Dp = oracle.padded_dim(D, M)  # 208 (a multiple of 16) and 102 (the int8 planes pad to 112)
    X = rng.standard_normal((2500, D)).astype(np.float32)
    R, _ = oracle.rotation(Dp, 9)
    ix = crisp.Index.build(X, M, R=R, codebooks=oracle.train_codebooks(oracle.rotate_rows(
        np.pad(X, ((0, 0), (0, Dp - D))), R), M, 6, 2, 2500, 3), K=6, seed=3)
    rows = []
    rows.append(np.zeros(D))
    e = np.zeros(D); e[17] = 3.0; rows.append(e)
    rows.append(np.where(np.arange(D) % 2 == 0, 1e15, 1e-15) * rng.standard_normal(D))
    rows.append(np.full(D, 1e-40))                       # subnormal fp32 inputs
    rows.append(rng.standard_normal(D) * 1e-38)
    rows.append(np.where(np.arange(D) % 2 == 0, 1.0, -1.0))
    c = rng.standard_normal(D); c[1::2] = -c[0::2][: D // 2]; rows.append(c)
    for k in range(-20, 21, 4):
        rows.append(rng.standard_normal(D) * 2.0 ** k)
    rows.append(np.abs(rng.standard_normal(D)) * 100 + 1000)  # large common mean (Gist-like)
    Q = np.vstack(rows + [rng.standard_normal(D) * rng.uniform(0.1, 10) for _ in range(300)]).astype(np.float32)
    ix.set_search_params(budget=200, tau=1, patience_factor=5)
    _, _, t = ix.trace(Q, 3, 1)
    ref = oracle.rotate_rows(np.pad(Q, ((0, 0), (0, Dp - D))), R)
    got = t["qrot"][:, :Dp]
    bad = np.nonzero(~np.all(got.view(np.uint32) == ref.view(np.uint32), axis=1))[0]
    assert bad.size == 0, f"rows {bad[:10]} differ"


@pytest.mark.parametrize("first,rounds,rmin", [(64, 1, 128), (64, 0, 128), (128, 3, 32), (256, 16, 64)])
def test_patience_rounds_and_tail(crisp, monkeypatch, first, rounds, rmin):
    """Optimized mode through every verification path: round 0 of `first` rows,
    `rounds` - 1 rounds of per-query spans (>= rmin rows), then the tail kernel;
    results and the patience stop index must equal the oracle's sequential rule
    (P:L458).  The untraced search (Hamming order cut at the rounds' reach, the
    tail completing it for queries that go further) gives the same answer."""
    monkeypatch.setenv("CRISP_PATIENCE_FIRST", str(first))
    monkeypatch.setenv("CRISP_PATIENCE_ROUNDS", str(rounds))
    monkeypatch.setenv("CRISP_ROUND_MIN", str(rmin))
    X, Qv, ox = make_case(cfg=1, N=12000, D=128, Q=24, M=4, K=9, seed=7)
    ix = build_gpu(crisp, X, ox, block_ids=4096)
    for pf, B in ((1, 900), (3, 2500), (0, 700), (60, 3000)):
        ix.set_search_params(budget=B, tau=1, patience_factor=pf)
        ids, d, t = ix.trace(Qv, 5, 1)
        r_ids, r_d, ot = oracle.search(ox, Qv, 5, 1, B, 1, patience_factor=pf, trace=True)
        compare_trace(t, ot, 1, X.shape[0])
        assert_topk_parity(ids, d, r_ids, r_d, f"patience first={first} rounds={rounds} pf={pf}")
        ids2, d2 = ix.search(Qv, 5, 1)
        assert np.array_equal(ids2, ids) and np.array_equal(d2, d), f"untraced pf={pf}"


@pytest.mark.parametrize("parts", ["3", "5", "3eq"])
@pytest.mark.parametrize("mode", [0, 1])
def test_host_buffers_match_device(crisp, monkeypatch, mode, parts):
    """crisp_search with host buffers (the H2D copy overlapped with the query
    transform and the probe, in parts of sizes 1 : 2 : ... : P, or equal parts)
    returns what the device-pointer call returns."""
    import torch

    monkeypatch.setenv("CRISP_H2D_PARTS", parts.rstrip("eq"))
    monkeypatch.setenv("CRISP_H2D_TRI", "0" if parts.endswith("eq") else "1")

    X, _, ox = make_case(cfg=1, N=20000, Q=10, seed=3)
    Qv = synth.Workload(1).queries(3000).numpy()
    ix = build_gpu(crisp, X, ox)
    ix.set_search_params(budget=oracle.budget_ids(0.01, 20000), tau=3, patience_factor=40)
    h_ids, h_d = ix.search(Qv, 10, mode)
    Qd = torch.from_numpy(Qv).cuda()
    ids = torch.empty((3000, 10), dtype=torch.int64, device="cuda")
    dd = torch.empty((3000, 10), dtype=torch.float32, device="cuda")
    ix.search_async(Qd, 10, mode, ids, dd, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(h_ids, ids.cpu().numpy()) and np.array_equal(h_d, dd.cpu().numpy())


@pytest.mark.parametrize("mode", [0, 1])
def test_candidate_capacity_bound(crisp, monkeypatch, mode):
    """|C_q| close to N (budget 9000 of 14000 ids, tau = 1): the per-query
    candidate capacity is the exact upper bound derived from B, tau and the
    largest cells (no read-back, no regrow), and the results are exact."""
    monkeypatch.setenv("CRISP_COUNT_BPC", "2")
    X, Qv, ox = make_case(cfg=1, N=14000, D=64, Q=20, M=4, K=6, seed=11)
    ix = build_gpu(crisp, X, ox, block_ids=4096)
    ix.set_search_params(budget=9000, tau=1, patience_factor=0)
    ids, d = ix.search(Qv, 10, mode)
    r_ids, r_d, ot = oracle.search(ox, Qv, 10, mode, 9000, 1, patience_factor=0, trace=True)
    assert ot["cand_n"].max() > 8000
    assert_topk_parity(ids, d, r_ids, r_d, "capacity bound")


@pytest.mark.parametrize("tau", [2, 5])
def test_shard_emulation_exact_fallback(crisp, tau):
    """G=3 point shards on one GPU through the phased shard session (exact
    global fallback), 'collectives' as device sums/stacks, then the a6 merge
    kernel: Guaranteed-Mode results equal the single index for every query,
    fallback queries included."""
    import torch

    X, Qv, ox = make_case(cfg=1, N=9001, D=64, Q=40, M=4, K=8, seed=13)
    k, B, G = 6, 400, 3
    single = build_gpu(crisp, X, ox, block_ids=4096)
    single.set_search_params(budget=B, tau=tau)
    ids1, d1 = single.search(Qv, k, 0)
    _, _, ot = oracle.search(ox, Qv, k, 0, B, tau, trace=True)
    shards = []
    for g in range(G):
        lo, hi = (9001 * g) // G, (9001 * (g + 1)) // G
        os.environ["CRISP_BLOCK_IDS"] = "4096"
        try:
            shards.append(crisp.Index.build(X[lo:hi], ox["M"], codebooks=ox["cb"], K=ox["K"], gid_base=lo))
        finally:
            os.environ.pop("CRISP_BLOCK_IDS", None)
    sizes = sum(s.local_cell_sizes() for s in shards)
    assert np.array_equal(sizes, ox["gsize"])
    for s in shards:
        s.set_global_cell_sizes(sizes)
        s.set_search_params(budget=B, tau=tau)
    q = torch.from_numpy(Qv).cuda()
    counts = [torch.empty(len(Qv), dtype=torch.int32, device="cuda") for _ in shards]
    sess = [s.shard_begin(q, k, 0, c) for s, c in zip(shards, counts)]
    gc = sum(counts)
    hists = [torch.zeros((len(Qv), 2 * ox["M"] + 2), dtype=torch.int32, device="cuda") for _ in shards]
    for ss, h in zip(sess, hists):
        crisp.Index.shard_hist(ss, gc, h)
    allh = torch.stack(hists).contiguous()
    outs = []
    for g, ss in enumerate(sess):
        gi = torch.empty((len(Qv), k), dtype=torch.int64, device="cuda")
        gd = torch.empty((len(Qv), k), dtype=torch.float64, device="cuda")
        crisp.Index.shard_finish(ss, gc, allh, G, g, gi, gd)
        crisp.Index.shard_free(ss)
        outs.append((gi, gd))
    od64 = torch.empty((len(Qv), k), dtype=torch.float64, device="cuda")
    od = torch.empty((len(Qv), k), dtype=torch.float32, device="cuda")
    oi = torch.empty((len(Qv), k), dtype=torch.int64, device="cuda")
    crisp.merge_topk(torch.stack([o[1] for o in outs]).contiguous(), torch.stack([o[0] for o in outs]).contiguous(),
                     od64, od, oi)
    torch.cuda.synchronize()
    if tau == 5:
        assert ot["fallback"].sum() >= 2
    assert np.array_equal(oi.cpu().numpy(), ids1)
    assert np.array_equal(od.cpu().numpy(), d1)
    # ... and equal the oracle's single-index search (the comparator is the oracle)
    r_ids, r_d, _ = oracle.search(ox, Qv, k, 0, B, tau)
    assert np.array_equal(oi.cpu().numpy(), r_ids)
    assert np.array_equal(od64.cpu().numpy(), r_d) or np.allclose(od64.cpu().numpy(), r_d, rtol=1e-12, atol=0)


def test_merge_topk_matches_oracle(crisp):
    """a6 (crisp_merge_topk) against oracle.merge_topk on lists with heavy exact
    distance ties (values from a small integer set, so (d, gid) decides),
    padded rows (-1, +inf) and shards holding fewer than k results."""
    import torch

    r = np.random.default_rng(3)
    for G, Q, k in ((2, 50, 10), (3, 40, 7), (8, 16, 100), (1, 5, 1)):
        d = np.sort(r.integers(0, 6, (G, Q, k)).astype(np.float64), axis=2)
        gids = np.empty((G, Q, k), np.int64)
        for g in range(G):
            for q in range(Q):
                gids[g, q] = np.sort(r.choice(np.arange(g * 1000, (g + 1) * 1000), k, replace=False))
        # each list ascending by (d, gid); pad the tail of some lists
        o = np.lexsort((gids, d), axis=2)
        d, gids = np.take_along_axis(d, o, 2), np.take_along_axis(gids, o, 2)
        pad = r.integers(0, k + 1, (G, Q))
        for g in range(G):
            for q in range(Q):
                d[g, q, pad[g, q]:] = np.inf
                gids[g, q, pad[g, q]:] = -1
        ref_d, ref_i = oracle.merge_topk(d, gids)
        dd, di = torch.from_numpy(d).cuda(), torch.from_numpy(gids).cuda()
        od64 = torch.empty((Q, k), dtype=torch.float64, device="cuda")
        od = torch.empty((Q, k), dtype=torch.float32, device="cuda")
        oi = torch.empty((Q, k), dtype=torch.int64, device="cuda")
        crisp.merge_topk(dd, di, od64, od, oi)
        torch.cuda.synchronize()
        assert np.array_equal(oi.cpu().numpy(), ref_i), (G, Q, k)
        assert np.array_equal(od64.cpu().numpy(), ref_d), (G, Q, k)


@pytest.mark.parametrize("mode", [0, 1])
def test_exact_ties_integer_data_duplicate_rows_and_centroids(crisp, mode):
    """Integer-valued data (exact distances: ties are real, not near-ties) with
    duplicated rows, and codebooks with duplicated centroids: the assignment
    (lowest c wins), the half sorts (delta, c), the cell order (cost, i, j), the
    Hamming order (h, id) and the top-k (d, id) all hit exact ties on both
    sides (App. A.2; Fig. 3; MNIST-like integer data)."""
    r = np.random.default_rng(17)
    N, D, M, K = 6000, 32, 4, 10
    X = r.integers(0, 4, (N, D)).astype(np.float32)
    X[3000:3600] = X[:600]  # duplicate rows
    Qv = r.integers(0, 4, (30, D)).astype(np.float32)
    Qv[:5] = X[[7, 3007, 100, 200, 2999]]  # self queries, some duplicated in X
    cb = oracle.train_codebooks(X, M, K, 5, N, 3)
    cb[:, :, 1] = cb[:, :, 0]  # duplicate centroids (half-sort and assignment ties)
    cb[:, :, 5] = np.round(cb[:, :, 5])
    ox = oracle.build(X, M, K=K, rotation_mode=0, codebooks=cb)
    ix = crisp.Index.build(X, M, codebooks=cb, K=K)
    compare_index(ix, ox)
    assert not np.any(ox["cells"] // K == 1) and not np.any(ox["cells"] % K == 1), "a duplicate never wins (lowest c)"
    for B, tau, k, P in ((300, 2, 10, 2), (1500, 1, 25, 1), (N, 4, 5, 3)):
        ix.set_search_params(budget=B, tau=tau, patience_factor=P)
        ids, d, t = ix.trace(Qv, k, mode)
        r_ids, r_d, ot = oracle.search(ox, Qv, k, mode, B, tau, patience_factor=P, trace=True)
        compare_trace(t, ot, mode, N)
        assert np.array_equal(ids, r_ids), f"(d, id) ties B={B}"
        assert np.array_equal(d, r_d.astype(np.float32)), "integer distances are exact"


def test_build_waits_for_pending_device_writes(crisp):
    """crisp_build on a device buffer that is still being written on the
    caller's stream: the stored vectors must be the final ones."""
    import torch

    N, D = 200000, 64
    X = torch.zeros((N, D), dtype=torch.float32, device="cuda")
    a = torch.randn((4096, 4096), device="cuda")
    for _ in range(20):  # keep the stream busy
        a = a @ a * 1e-3
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    X.normal_(generator=g)
    X.add_(a[0, 0] * 0)
    ix = crisp.Index.build(X, 4, K=8, seed=1, rotation=0)
    e = ix.export()
    assert np.array_equal(e["X"][:, :D], X.cpu().numpy())
    ix.free()


# ---------------------------------------------------------------- f1: ADSampling (Eq. 2)
@pytest.mark.parametrize("rounds", [(256, 1024, 2), (32, 64, 2), (32, 64, 0)])
def test_adsampling_stagewise(crisp, monkeypatch, rounds):
    """Optimized Mode with ADSampling against the oracle, stage by stage
    (Hamming order, patience stop, ids, distances): the default rounds, short
    rounds (several pruning rounds and the sequential tail) and the tail alone."""
    first, batch, nr = rounds
    monkeypatch.setenv("CRISP_AD_FIRST", str(first))
    monkeypatch.setenv("CRISP_PATIENCE_BATCH", str(max(batch, 64)))
    monkeypatch.setenv("CRISP_PATIENCE_ROUNDS", str(nr))
    X, Qv, ox = make_case(cfg=2, N=18001, D=90, Q=40, M=4, K=31, rotation=1, seed=3)
    ix = build_gpu(crisp, X, ox, block_ids=4096)
    B, tau, k = 700, 2, 7
    for pf in (3, 40):
        ix.set_search_params(budget=B, tau=tau, patience_factor=pf)
        ix.set_adsampling(True, 2.1, 32)
        ids, d, t = ix.trace(Qv, k, 1)
        r_ids, r_d, ot = oracle.search(ox, Qv, k, 1, B, tau, patience_factor=pf, trace=True, adsampling=True)
        compare_trace(t, ot, 1, X.shape[0])
        assert_topk_parity(ids, d, r_ids, r_d, f"adsampling pf={pf}")
        ids2, d2 = ix.search(Qv, k, 1)
        assert np.array_equal(ids2, ids) and np.array_equal(d2, d)


@pytest.mark.parametrize("eps0,stride", [(2.1, 32), (0.5, 16), (2.1, 128)])
def test_adsampling_margins_and_strides(crisp, eps0, stride):
    """Other margins and checkpoint strides, cfg1 (N=20k, D=256, M=8)."""
    X, Qv, ox = make_case()
    ix = build_gpu(crisp, X, ox)
    B, tau, k = oracle.budget_ids(0.01, 20000), 3, 10
    ix.set_search_params(budget=B, tau=tau, patience_factor=40)
    ix.set_adsampling(True, eps0, stride)
    ids, d, t = ix.trace(Qv, k, 1)
    r_ids, r_d, ot = oracle.search(ox, Qv, k, 1, B, tau, patience_factor=40, trace=True, adsampling=True,
                                   eps0=eps0, ad_stride=stride)
    compare_trace(t, ot, 1, X.shape[0])
    assert_topk_parity(ids, d, r_ids, r_d, f"adsampling eps0={eps0} stride={stride}")
    # switching it off restores exact verification
    ix.set_adsampling(False)
    ids3, _ = ix.search(Qv, k, 1)
    r3, _, _ = oracle.search(ox, Qv, k, 1, B, tau, patience_factor=40)
    assert np.array_equal(ids3, r3)


def test_adsampling_k100(crisp):
    X, Qv, ox = make_case(cfg=4, N=30000, D=192, Q=20, M=8, K=24, rotation=1, seed=9)
    ix = build_gpu(crisp, X, ox, block_ids=8192)
    B, tau, k = 1500, 3, 100
    ix.set_search_params(budget=B, tau=tau, patience_factor=4)
    ix.set_adsampling(True)
    ids, d, t = ix.trace(Qv, k, 1)
    r_ids, r_d, ot = oracle.search(ox, Qv, k, 1, B, tau, patience_factor=4, trace=True, adsampling=True)
    compare_trace(t, ot, 1, X.shape[0])
    assert_topk_parity(ids, d, r_ids, r_d, "adsampling k=100")


@pytest.mark.parametrize("filt", ["0", "2"])
def test_adsampling_behind_the_verification_filter(crisp, monkeypatch, filt):
    """f1 with the certified int8 filter (R17) forced on for every round >= 1
    (CRISP_FILTER_ROUNDS=2): rows the bound excludes are misses under Eq. 2
    too, and Eq. 2 is still applied in order to every row that would enter the
    top-k, so the patience stop, ids and distances equal the oracle's
    ADSampling search (k = 100 and k = 7, short and long patience)."""
    monkeypatch.setenv("CRISP_FILTER_ROUNDS", filt)
    X, Qv, ox = make_case(cfg=4, N=30000, D=192, Q=20, M=8, K=24, rotation=1, seed=9)
    ix = build_gpu(crisp, X, ox, block_ids=8192)
    for (B, tau, k, pf) in ((1500, 3, 100, 4), (1500, 3, 100, 40), (900, 2, 7, 40)):
        ix.set_search_params(budget=B, tau=tau, patience_factor=pf)
        ix.set_adsampling(True)
        ids, d, t = ix.trace(Qv, k, 1)
        r_ids, r_d, ot = oracle.search(ox, Qv, k, 1, B, tau, patience_factor=pf, trace=True, adsampling=True)
        compare_trace(t, ot, 1, X.shape[0])
        assert_topk_parity(ids, d, r_ids, r_d, f"adsampling + filter k={k} pf={pf}")
        ids2, d2 = ix.search(Qv, k, 1)
        assert np.array_equal(ids2, ids) and np.array_equal(d2, d)


def test_adsampling_rejects_bad_stride(crisp):
    X, Qv, ox = make_case(cfg=1, N=2000, D=64, Q=4, M=4, K=6)
    ix = build_gpu(crisp, X, ox)
    with pytest.raises(crisp.CrispError):
        ix.set_adsampling(True, 2.1, 24)
    with pytest.raises(crisp.CrispError):
        ix.set_adsampling(True, -1.0, 32)


@pytest.mark.parametrize("rotation", [1, -1])
def test_model_from_gathered_samples_equals_full_build(crisp, rotation):
    """crisp_build_model on the gathered CEV and k-means sample rows (the
    multi-GPU model build) gives exactly the rotation, the
    codebooks and the CEV of crisp_build over all rows; the library's sampled
    row ids equal the oracle's (both implement the counter-based sampler)."""
    w = synth.Workload(2, D=96)
    X = w.base(30000).numpy()
    params = dict(K=8, kmeans_iters=4, kmeans_sample=5000, seed=11, rotation=rotation)
    full = crisp.Index.build(X, 4, **params)
    e, info = full.export(), full.info()
    cev_ids, km_ids = crisp.model_samples(30000, 11, 5000)
    assert np.array_equal(cev_ids, oracle.sample_rows(30000, oracle.cev_sample_size(30000), 11, 1))
    assert np.array_equal(km_ids, oracle.sample_rows(30000, 5000, 11, 3))
    R, cb, cev = crisp.build_model(X[cev_ids], X[km_ids], 4, **params)
    assert cev == info["cev"]
    assert (R is not None) == bool(info["rotated"])
    if R is not None:
        assert np.array_equal(R, e["R"])
    assert np.array_equal(cb, e["codebooks"])
    full.free()


@pytest.mark.parametrize("screen,R", [("1", "1"), ("1", "3"), ("1", "24"), ("0", "24")])
@pytest.mark.parametrize("mode", [0, 1])
def test_probe_screen_on_tensor_cores(crisp, monkeypatch, mode, screen, R):
    """a1 with the tensor-core screen (probe_tc.cu): the activated cells, their
    pop order and weights stay bit-exact whatever prefix length R the screen
    certifies (R = 1 and 3 force most walks past the certified prefix and
    through the exact redo), and equal the unscreened probe's."""
    import torch

    monkeypatch.setenv("CRISP_PROBE_SCREEN", screen)
    monkeypatch.setenv("CRISP_PROBE_R", R)
    X, Qv, ox = make_case(cfg=1, N=20000, D=256, Q=64, M=8, K=50, seed=0)
    ix = build_gpu(crisp, X, ox)
    B, tau, k = 300, 3, 10
    ix.set_search_params(budget=B, tau=tau, patience_factor=40)
    crisp.set_stage_timing(True)
    crisp.search_counters(reset=True)
    ids, d, t = ix.trace(Qv, k, mode)
    cnt = crisp.search_counters(reset=True)
    crisp.set_stage_timing(False)
    torch.cuda.synchronize()
    r_ids, r_d, ot = oracle.search(ox, Qv, k, mode, B, tau, patience_factor=40, trace=True)
    compare_trace(t, ot, mode, X.shape[0])
    assert_topk_parity(ids, d, r_ids, r_d, f"screen={screen} R={R}")
    if screen == "1" and R == "1":
        assert cnt["probe_screen_redone"] > 0, "R = 1 must send walks through the exact redo"
    if screen == "1" and R == "24":
        assert cnt["probe_exact_half_distances"] < 64 * 8 * 2 * 50, "the screen must save exact half distances"


@pytest.mark.parametrize("mode", [0, 1])
def test_blockwise_rotation_f4(crisp, mode):
    """f4, block-wise variance redistribution (DESIGN R16): the GPU build
    picks the oracle's block (the b subspaces of largest sample variance; the
    covariance diagonal is computed in the same sequential fp64 order), its R is
    the identity outside the block exactly and matches the oracle's rotation on
    it (cuSOLVER vs LAPACK QR: 1e-5); with the oracle's R injected, X', cells,
    CSR, codes and the search are bit-exact, and the rows outside the block keep
    their input values."""
    r = np.random.default_rng(12)
    M, D, N = 8, 64, 12000
    scale = np.ones(D)
    scale[16:24] = 12.0
    scale[48:56] = 5.0
    X = (r.standard_normal((N, D)) * scale).astype(np.float32)
    Qv = (r.standard_normal((40, D)) * scale).astype(np.float32)
    ox = oracle.build(X, M, K=10, rotation_mode=1, kmeans_iters=4, seed=5, rotation_block=2)
    gix = crisp.Index.build(X, M, K=10, rotation=1, kmeans_iters=4, seed=5, rotation_block=2)
    assert gix.info()["rotation_block"] == 2
    Rg = gix.export()["R"]
    blk = oracle.rotation_block(oracle.dim_variances(X, 5), M, D, 2)
    assert blk.tolist() == list(range(16, 24)) + list(range(48, 56))
    out = np.setdiff1d(np.arange(D), blk)
    assert np.array_equal(Rg[out], np.eye(D, dtype=np.float32)[out])
    assert np.array_equal(Rg[:, out], np.eye(D, dtype=np.float32)[:, out])
    assert np.abs(Rg - ox["R"]).max() < 1e-5
    gix.free()
    ix = crisp.Index.build(X, M, R=ox["R"], codebooks=ox["cb"], K=10, seed=5)
    compare_index(ix, ox)
    assert np.array_equal(ix.export()["X"][:, out], X[:, out])
    ix.set_search_params(budget=600, tau=2, patience_factor=3)
    ids, d, t = ix.trace(Qv, 10, mode)
    r_ids, r_d, ot = oracle.search(ox, Qv, 10, mode, 600, 2, patience_factor=3, trace=True)
    compare_trace(t, ot, mode, N)
    assert_topk_parity(ids, d, r_ids, r_d, "block-wise rotation")


def test_search_async_returns_before_the_kernels_finish(crisp):
    """crisp_search_async is stream-ordered: it enqueues the whole search and
    returns (no read-back inside: the candidate capacity is an exact bound known
    in advance).  Evidence without a tracer: with the stream held busy by a
    kernel queued first, the call returns while that kernel still runs, and the
    results are then complete and exact."""
    import time

    import torch

    X, Qv, ox = make_case(cfg=1, N=20000, D=256, Q=200, M=8, K=50, seed=0)
    ix = build_gpu(crisp, X, ox)
    ix.set_search_params(budget=300, tau=3, patience_factor=40)
    ref_ids, ref_d = ix.search(Qv, 10, 1)
    q = torch.from_numpy(Qv).cuda()
    ids = torch.empty((200, 10), dtype=torch.int64, device="cuda")
    dd = torch.empty((200, 10), dtype=torch.float32, device="cuda")
    stream = torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        torch.cuda._sleep(int(2e9))  # ~1 s of GPU time queued ahead of the search
        t0 = time.perf_counter()
        ix.search_async(q, 10, 1, ids, dd, stream.cuda_stream)
        t_call = time.perf_counter() - t0
        busy = not stream.query()
    torch.cuda.synchronize()
    assert busy, "the stream finished before the call returned"
    assert t_call < 0.3, f"crisp_search_async blocked for {t_call:.3f} s"
    assert np.array_equal(ids.cpu().numpy(), ref_ids) and np.array_equal(dd.cpu().numpy(), ref_d)


@pytest.mark.parametrize("parts", ["2", "3"])
@pytest.mark.parametrize("mode", [0, 1])
def test_pipelined_chunks_equal_one_pass(crisp, monkeypatch, mode, parts):
    """CRISP_PIPE: the batch in query chunks on two side streams (one chunk's
    count overlapping the previous chunk's verification) gives the one-pass
    results exactly, and the oracle's on a sample."""
    import torch

    X, Qv, ox = make_case(cfg=1, N=20000, D=256, Q=4100, M=8, K=50, seed=0)
    ix = build_gpu(crisp, X, ox)
    ix.set_search_params(budget=300, tau=3, patience_factor=40)
    q = torch.from_numpy(Qv).cuda()
    outs = []
    for p in ("1", parts):
        monkeypatch.setenv("CRISP_PIPE", p)
        ids = torch.empty((4100, 10), dtype=torch.int64, device="cuda")
        dd = torch.empty((4100, 10), dtype=torch.float32, device="cuda")
        ix.search_async(q, 10, mode, ids, dd, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        outs.append((ids.cpu().numpy(), dd.cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    sample = np.arange(0, 4100, 41)
    r_ids, r_d, _ = oracle.search(ox, Qv[sample], 10, mode, 300, 3, patience_factor=40)
    assert_topk_parity(outs[1][0][sample], outs[1][1][sample], r_ids, r_d, f"pipe={parts}")


def _skewed(seed, N, D, Q, decay=10.0):
    r = np.random.default_rng(seed)
    scale = np.exp(-np.arange(D) / decay) * 4.0 + 0.05
    X = (r.standard_normal((N, D)) * scale).astype(np.float32)
    Qv = (r.standard_normal((Q, D)) * scale).astype(np.float32)
    return X, Qv


@pytest.mark.parametrize("mode", [0, 1])
def test_adaptive_subspaces_f4(crisp, mode):
    """f4, adaptive subspace decomposition (DESIGN R18): on a decaying
    spectrum (unrotated) the GPU build picks the oracle's widths (the rule on
    the CEV sample's variances, same sequential fp64 order), trains the same
    codebooks on the zero-padded halves, and assigns, lists and searches
    exactly as the oracle's variable-width index (a1 on the exact probe: the
    rule's half starts are not 16-byte aligned)."""
    X, Qv = _skewed(21, 15000, 96, 48)
    M = 6
    ox = oracle.build(X, M, K=12, rotation_mode=0, kmeans_iters=5, seed=4, adaptive_subspaces=True)
    w = (ox["hoff"][2::2] - ox["hoff"][:-1:2]).tolist()
    assert w[0] < 16 < w[-1], w
    ix = crisp.Index.build(X, M, K=12, rotation=0, kmeans_iters=5, seed=4, adaptive_subspaces=1)
    info, e = ix.info(), ix.export()
    assert info["adaptive"] == 1 and info["dh"] == ox["dh"]
    assert e["subspace_widths"].tolist() == w
    assert np.array_equal(e["codebooks"], ox["cb"]), "k-means codebooks of the variable halves"
    compare_index(ix, ox)
    B, tau, k = 900, 2, 10
    ix.set_search_params(budget=B, tau=tau, patience_factor=4)
    ids, d, t = ix.trace(Qv, k, mode)
    r_ids, r_d, ot = oracle.search(ox, Qv, k, mode, B, tau, patience_factor=4, trace=True)
    compare_trace(t, ot, mode, X.shape[0])
    assert_topk_parity(ids, d, r_ids, r_d, "adaptive widths")
    ids2, d2 = ix.search(Qv, k, mode)
    assert np.array_equal(ids2, ids) and np.array_equal(d2, d)


@pytest.mark.parametrize("mode", [0, 1])
def test_adaptive_widths_given_screened_and_injected(crisp, mode):
    """Given widths (8, 8, 16, 32): half starts at multiples of 4, so a1 runs the
    tensor-core screen with per-half TMA offsets; the GPU's own build and the
    oracle's codebooks injected (crisp_build_with + subspace_widths) both match
    the oracle stage by stage."""
    import torch

    X, Qv = _skewed(22, 12000, 64, 40, decay=14.0)
    widths = [8, 8, 16, 32]
    ox = oracle.build(X, 4, K=16, rotation_mode=0, kmeans_iters=4, seed=6, subspace_widths=widths)
    assert ox["hoff"].tolist() == [0, 4, 8, 12, 16, 24, 32, 48, 64] and ox["dh"] == 16
    own = crisp.Index.build(X, 4, K=16, rotation=0, kmeans_iters=4, seed=6, subspace_widths=widths)
    assert np.array_equal(own.export()["codebooks"], ox["cb"])
    compare_index(own, ox)
    own.free()
    ix = crisp.Index.build(X, 4, codebooks=ox["cb"], K=16, subspace_widths=widths)
    compare_index(ix, ox)
    B, tau, k = 700, 2, 10
    ix.set_search_params(budget=B, tau=tau, patience_factor=4)
    crisp.set_stage_timing(True)
    crisp.search_counters(reset=True)
    ids, d, t = ix.trace(Qv, k, mode)
    cnt = crisp.search_counters(reset=True)
    crisp.set_stage_timing(False)
    torch.cuda.synchronize()
    r_ids, r_d, ot = oracle.search(ox, Qv, k, mode, B, tau, patience_factor=4, trace=True)
    compare_trace(t, ot, mode, X.shape[0])
    assert_topk_parity(ids, d, r_ids, r_d, "given widths")
    assert cnt["probe_exact_half_distances"] < 40 * 4 * 2 * 16, "the screen must run (and save exact distances)"


def test_adaptive_subspaces_rotated_rule_on_stored_vectors(crisp):
    """Rotated + adaptive: the widths come from the variances of the stored
    X' (here teacher-forced: the oracle rule on the GPU's exported X', the CEV
    sample's sequential fp64 variances) and the build is self-consistent."""
    X, _ = _skewed(23, 8000, 64, 1, decay=6.0)
    ix = crisp.Index.build(X, 4, K=8, rotation=1, kmeans_iters=3, seed=2, adaptive_subspaces=1)
    e = ix.export()
    w = oracle.adaptive_widths(oracle.dim_variances(e["X"], 2), 4, 64)
    assert e["subspace_widths"].tolist() == w
    ox = oracle.build(e["X"], 4, K=8, rotation_mode=0, codebooks=e["codebooks"], seed=2, subspace_widths=w)
    assert np.array_equal(e["cells"], ox["cells"]) and np.array_equal(e["ids"], ox["ids"])


@pytest.mark.parametrize("pf", [3, 40])
def test_hamming_order_multiwindow_bins(crisp, pf):
    """k_hsort_cta's per-warp counters cover windows of 1024 Hamming bins: at
    D' = 2560 the candidates' h spread past bin 1024, so the traced search
    (the whole order) and the untraced one (the order up to its cut, LIST
    phase B for k = 10) sort across several windows; order, patience stop,
    ids and distances equal the oracle's."""
    r = np.random.default_rng(31)
    N, D, Q, M = 8000, 2560, 24, 8
    X = r.standard_normal((N, D)).astype(np.float32)
    Qv = (X[r.choice(N, Q, replace=False)] + 0.8 * r.standard_normal((Q, D))).astype(np.float32)
    ox = oracle.build(X, M, K=16, rotation_mode=0, kmeans_iters=3, seed=4)
    ix = build_gpu(crisp, X, ox)
    B, tau, k = 3000, 2, 10
    ix.set_search_params(budget=B, tau=tau, patience_factor=pf)
    ids, d, t = ix.trace(Qv, k, 1)
    r_ids, r_d, ot = oracle.search(ox, Qv, k, 1, B, tau, patience_factor=pf, trace=True)
    compare_trace(t, ot, 1, N)
    qc = oracle.codes(ot["qrot"])
    hmax = 0
    for q in range(Q):
        n = int(ot["cand_n"][q])
        if n:
            x = ox["codes"][ot["order"][q, :n]] ^ qc[q]
            hmax = max(hmax, int(np.unpackbits(x.view(np.uint8), axis=1).sum(axis=1).max()))
    assert hmax > 1024, f"candidates' h must reach past the first window ({hmax})"
    assert_topk_parity(ids, d, r_ids, r_d, f"multi-window hsort pf={pf}")
    ids2, d2 = ix.search(Qv, k, 1)
    assert np.array_equal(ids2, r_ids)
