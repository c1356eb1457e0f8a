"""Pins for the CPU oracle (-m "not gpu").

Each test checks the oracle against something other than itself: values the
paper/SPEC print for a worked example (tests/golden/, cited), closed forms,
invariants, brute force on tiny inputs, or special cases that reduce to a
textbook routine.  They are chosen so that a dropped term, a wrong sign or
index, or a transposed operand fails at least one of them.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def rng(seed=0):
    return np.random.default_rng(seed)


# ---------------------------------------------------------------- generator
def test_philox_kat():
    for v in gold("philox_kat.json")["vectors"]:
        h = lambda x: int(x, 16) if isinstance(x, str) else x
        out = oracle.philox([h(c) for c in v["ctr"]], [h(k) for k in v["key"]])
        assert [int(o) for o in out] == [int(x, 16) for x in v["out"]]


def test_normals_moments():
    L = oracle.lib()
    z = np.array([L.or_normal(7, 2, i, 0) for i in range(20000)])
    assert abs(z.mean()) < 0.03 and abs(z.std() - 1) < 0.03
    u = np.array([L.or_uniform(7, 2, i, 0) for i in range(20000)])
    assert u.min() >= 0 and u.max() < 1 and abs(u.mean() - 0.5) < 0.01


# ---------------------------------------------------------------- dist64
def test_dist64_closed_forms():
    assert oracle.dist64([0, 0], [3, 4]) == 25.0
    x = rng().standard_normal(37).astype(np.float32)
    assert oracle.dist64(x, x) == 0.0
    y = rng(1).standard_normal(37).astype(np.float32)
    ref = math.fsum(((x.astype(np.float64) - y.astype(np.float64)) ** 2).tolist())
    assert abs(oracle.dist64(x, y) - ref) <= 1e-14 * ref
    # sequential fma semantics: 1 + 2^-30 squared is kept exactly by fma
    a = np.array([1 + 2.0 ** -20], np.float32)
    assert oracle.dist64(a, [0.0]) == (1 + 2.0 ** -20) ** 2


# ---------------------------------------------------------------- sampling / CEV
def test_cev_sample_size_S117():
    assert oracle.cev_sample_size(100) == 10
    assert oracle.cev_sample_size(10_000_000) == 100_000
    assert oracle.cev_sample_size(5) == 5
    assert oracle.cev_sample_size(11) == 2  # ceil(1.1)


def test_sample_rows_uniform_without_replacement():
    s = oracle.sample_rows(1000, 100, 3, 1)
    assert len(set(s.tolist())) == 100 and np.all(np.diff(s) > 0)
    assert np.array_equal(s, oracle.sample_rows(1000, 100, 3, 1))
    hits = np.zeros(50)
    for seed in range(400):
        hits[oracle.sample_rows(50, 10, seed, 1)] += 1
    # inclusion probability 0.2 for every row
    assert np.all(np.abs(hits / 400 - 0.2) < 0.1)


def test_eigs_known_spectrum_and_trace():
    D = 12
    Qm, _ = np.linalg.qr(rng(2).standard_normal((D, D)))
    lam = np.arange(1, D + 1, dtype=np.float64) ** 1.3
    A = Qm @ np.diag(lam) @ Qm.T
    w = np.sort(oracle.eig_sym(A))
    assert np.allclose(w, lam, rtol=1e-11, atol=1e-11)
    assert abs(w.sum() - np.trace(A)) < 1e-10 * np.trace(A)
    # 2x2 closed form: [[a,b],[b,c]] eigenvalues (a+c)/2 +- sqrt(((a-c)/2)^2 + b^2)
    a, b, c = 2.0, 0.7, -1.0
    w2 = np.sort(oracle.eig_sym([[a, b], [b, c]]))
    r = math.sqrt(((a - c) / 2) ** 2 + b * b)
    assert np.allclose(w2, [(a + c) / 2 - r, (a + c) / 2 + r], rtol=1e-14)


def test_cev_formula_P266():
    # top floor(0.2*10)=2 of [5,4,1,...] / total, negatives clamped
    w = [1, 5, 4, 1, 1, 1, 1, 1, 1, -0.5]
    assert abs(oracle.cev_from_eigs(w) - 9.0 / 16.0) < 1e-15
    assert oracle.cev_from_eigs([1, 1, 1]) == pytest.approx(1 / 3)  # k = max(1, floor(0.6))
    assert oracle.cev_from_eigs([0.0] * 5) == 0.0


def test_cev_isotropic_and_single_axis_S130():
    X = rng(3).standard_normal((500_000, 10)).astype(np.float32)  # sample = 50k rows
    assert abs(oracle.cev(X, 0) - 0.2) < 0.05
    Y = np.zeros((2000, 10), np.float32)
    Y[:, 0] = rng(4).standard_normal(2000)
    assert oracle.cev(Y, 0) > 0.999


def test_covariance_matches_definition():
    X = rng(5).standard_normal((300, 6)).astype(np.float32)
    rows = np.arange(300)
    Cm = oracle.covariance(X, rows)
    assert np.allclose(Cm, np.cov(X.astype(np.float64), rowvar=False, ddof=1), rtol=1e-12, atol=1e-14)


# ---------------------------------------------------------------- rotation
@pytest.mark.parametrize("D", [1, 2, 8, 64])
def test_qr_householder_is_the_unique_positive_qr(D):
    G = oracle.gaussian_matrix(D, 11)
    Qm, rd = oracle.qr(G)
    assert np.abs(Qm @ Qm.T - np.eye(D)).max() <= 1e-12
    Rp = Qm.T @ G  # must be upper triangular with positive diagonal: G = Q R'
    assert np.abs(np.tril(Rp, -1)).max() <= 1e-11 * np.abs(G).max()
    assert np.all(np.diag(Rp) > 0)
    assert np.allclose(np.diag(Rp), rd, rtol=1e-12)
    if D == 1:
        assert Qm[0, 0] == np.sign(G[0, 0])


def test_rotation_orthogonal_isometric_S141():
    R32, R64 = oracle.rotation(64, 5)
    assert np.abs(R64 @ R64.T - np.eye(64)).max() <= 1e-10
    assert np.abs(R32.astype(np.float64) @ R32.T.astype(np.float64) - np.eye(64)).max() <= 1e-5
    x = rng(6).standard_normal((100, 64)).astype(np.float32)
    y = oracle.rotate_rows(x, R32)
    n0 = (x.astype(np.float64) ** 2).sum(1)
    n1 = (y.astype(np.float64) ** 2).sum(1)
    assert np.max(np.abs(n1 - n0) / n0) < 1e-5


def test_rotate_rows_is_fp32_of_exact_product():
    x = rng(7).standard_normal((50, 32)).astype(np.float32)
    R = rng(8).standard_normal((32, 32)).astype(np.float32)
    y = oracle.rotate_rows(x, R)
    ref = x.astype(np.float64) @ R.astype(np.float64)
    # fp64 accumulation then one rounding: within 1 ulp of the correctly rounded value
    ulp = np.spacing(np.abs(ref).astype(np.float32))
    assert np.all(np.abs(y.astype(np.float64) - ref) <= ulp)
    # x = e_3 selects row 3 of R exactly
    e = np.zeros((1, 32), np.float32)
    e[0, 3] = 1
    assert np.array_equal(oracle.rotate_rows(e, R)[0], R[3])


# ---------------------------------------------------------------- k-means
def test_kmeans_k1_is_mean():
    pts = rng(9).standard_normal((777, 5)).astype(np.float32)
    Cm, _ = oracle.kmeans(pts, 1, 20, 0)
    assert np.allclose(Cm[0], pts.astype(np.float64).mean(0), atol=1e-5)


def test_kmeans_exact_cover_and_duplicates():
    pts = rng(10).standard_normal((8, 3)).astype(np.float32)
    Cm, obj = oracle.kmeans(pts, 8, 20, 1)
    assert sorted(map(tuple, Cm.tolist())) == sorted(map(tuple, pts.tolist()))
    assert obj[0] == 0.0
    # fewer distinct points than K: surplus centroids duplicate points
    Cm2, _ = oracle.kmeans(pts[:3], 5, 5, 2)
    assert set(map(tuple, Cm2.tolist())) <= set(map(tuple, pts[:3].tolist()))


def test_kmeans_lloyd_monotone_and_blobs():
    r = rng(11)
    a = r.standard_normal((400, 4)) * 0.1
    b = r.standard_normal((400, 4)) * 0.1 + 10
    pts = np.vstack([a, b]).astype(np.float32)
    Cm, _ = oracle.kmeans(pts, 2, 20, 3)
    means = sorted([a.mean(0).tolist(), (b.mean(0)).tolist()])
    got = sorted(Cm.tolist())
    assert np.allclose(got, means, atol=0.1 * 10)
    P = r.standard_normal((3000, 6)).astype(np.float32)
    _, obj = oracle.kmeans(P, 20, 15, 4)
    obj = obj[obj >= 0]
    assert len(obj) >= 2 and np.all(np.diff(obj) <= 1e-9 * obj[0])


# ---------------------------------------------------------------- assignment / CSR / codes
def test_assign_examples_S234():
    L = oracle.lib()
    C = np.array([[0, 0], [1, 1]], np.float32)
    x = np.array([1, 1], np.float32)
    assert L.or_argmin_centroid(oracle._p(x), oracle._p(C), 2, 2, None) == 1
    # equidistant -> lowest id
    x = np.array([0.5, 0.5], np.float32)
    assert L.or_argmin_centroid(oracle._p(x), oracle._p(C), 2, 2, None) == 0
    # cell = i*K + j with K=2: left = centroid 1, right = centroid 0 -> 2
    cb = np.zeros((1, 2, 2, 1), np.float32)
    cb[0, 0, :, 0] = [0, 5]
    cb[0, 1, :, 0] = [3, 9]
    cells = oracle.assign(np.array([[5, 3]], np.float32), cb)
    assert cells[0, 0] == 2


def test_assign_matches_naive_scan():
    r = rng(12)
    X = r.standard_normal((300, 16)).astype(np.float32)
    cb = r.standard_normal((2, 2, 7, 4)).astype(np.float32)
    cells = oracle.assign(X, cb)
    for m in range(2):
        for p in range(0, 300, 17):
            best = []
            for side in range(2):
                xs = X[p, m * 8 + side * 4: m * 8 + side * 4 + 4].astype(np.float64)
                d = ((cb[m, side].astype(np.float64) - xs) ** 2).sum(1)
                best.append(int(np.argmin(d)))
            assert cells[m, p] == best[0] * 7 + best[1]


def test_csr_paper_example_P363():
    g = gold("csr_example_P363.json")
    N, K = 23, 2
    cells = np.full((1, N), 3, np.int32)  # everything else in the last cell
    cells[0, g["cell_j_points"]] = 0      # C_j precedes C_i in cell order
    cells[0, g["cell_i_points"]] = 1
    off, ids = oracle.csr(cells, K)
    n = len(g["expected_ids_order"])
    assert ids[0, :n].tolist() == g["expected_ids_order"]
    assert off[0].tolist()[:3] == [0, 4, 10] and off[0, -1] == N


def test_csr_equals_naive_map_of_lists():
    r = rng(13)
    M, K, N = 3, 4, 2000
    cells = r.integers(0, K * K, (M, N)).astype(np.int32)
    off, ids = oracle.csr(cells, K)
    for m in range(M):
        assert off[m, 0] == 0 and off[m, -1] == N and np.all(np.diff(off[m]) >= 0)
        assert sorted(ids[m].tolist()) == list(range(N))  # partition property
        for c in range(K * K):
            naive = [p for p in range(N) if cells[m, p] == c]
            assert ids[m, off[m, c]:off[m, c + 1]].tolist() == naive


def test_codes_S254():
    c = oracle.codes(np.array([[1.5, -0.2, 0.0, 3.0]], np.float32))
    assert int(c[0, 0]) == 0b1001
    x = rng(14).standard_normal((5, 130)).astype(np.float32)
    x[0, 5] = 0.0
    a, b = oracle.codes(x), oracle.codes(-x)
    full = (1 << 64) - 1
    for w in range(3):
        nbits = min(64, 130 - 64 * w)
        mask = full if nbits == 64 else (1 << nbits) - 1
        comp = (~a[1:, w] & np.uint64(mask))
        assert np.array_equal(b[1:, w], comp)
    assert not (int(a[0, 0]) >> 5) & 1 and not (int(b[0, 0]) >> 5) & 1


# ---------------------------------------------------------------- a1 / a2 (Alg. 1 lines 3-17)
def test_half_sorted_matches_full_sort():
    r = rng(15)
    C = r.standard_normal((50, 9)).astype(np.float32)
    C[7] = C[3]  # forced tie -> lower id first
    q = r.standard_normal(9).astype(np.float32)
    d, p = oracle.half_sorted(q, C)
    ref = sorted((oracle.dist64(q, C[c]), c) for c in range(50))
    assert list(zip(d.tolist(), p.tolist())) == ref
    d0, p0 = oracle.half_sorted(C[12], C)
    assert d0[0] == 0.0 and p0[0] == 12


def test_multisequence_spec_example_S346():
    g = gold("multisequence_S346.json")
    a, b = np.array(g["dist_left"], float), np.array(g["dist_right"], float)
    pa = pb = np.arange(3, dtype=np.int32)
    cells, w, ret = oracle.multisequence(a, pa, b, pb, np.ones(9, np.int64), budget=10**9)
    assert [[c // 3, c % 3] for c in cells] == g["order"]
    assert [a[c // 3] + b[c % 3] for c in cells] == g["costs"]
    assert all(x == 1 for x in w) and ret == 9


def test_multisequence_equals_full_sort_with_ties():
    r = rng(16)
    for trial in range(300):
        K = int(r.integers(1, 10))
        a = np.sort(r.integers(0, 4, K).astype(float))
        b = np.sort(r.integers(0, 4, K).astype(float))
        pa = r.permutation(K).astype(np.int32)
        pb = r.permutation(K).astype(np.int32)
        cells, _, _ = oracle.multisequence(a, pa, b, pb, np.ones(K * K, np.int64), budget=10**9)
        ref = sorted((a[i] + b[j], i, j) for i in range(K) for j in range(K))
        assert cells.tolist() == [int(pa[i] * K + pb[j]) for _, i, j in ref]


def test_multisequence_fig3_weights_and_budget():
    """Fig. 3: 5x5 grid, budget reached at rank 13, k_size=6 -> ranks
    1-6 weigh 2, ranks 7-13 weigh 1; the whole last cell counts (Z3) and empty
    cells take ranks (Z5)."""
    K = 5
    a = np.arange(K, dtype=float)
    b = np.arange(K, dtype=float) * 1.01
    pa = pb = np.arange(K, dtype=np.int32)
    size = np.full(K * K, 3, np.int64)
    ref = sorted((a[i] + b[j], i, j) for i in range(K) for j in range(K))
    size[ref[4][1] * K + ref[4][2]] = 0  # rank 5 is an empty cell
    budget = 3 * 12 - 2  # reached while popping rank 13 (12 non-empty cells before it give 33 < 34)
    cells, w, ret = oracle.multisequence(a, pa, b, pb, size, budget, wk=6)
    assert len(cells) == 13 and ret == 36
    assert w.tolist() == [2] * 6 + [1] * 7
    cells0, w0, _ = oracle.multisequence(a, pa, b, pb, size, budget, wk=0)
    assert cells0.tolist() == cells.tolist() and set(w0.tolist()) == {1}


# ---------------------------------------------------------------- end-to-end search
def small_index(N=1500, D=32, M=4, K=6, seed=0, rot=0):
    r = rng(seed)
    X = (r.standard_normal((N, D)) @ np.diag(np.linspace(2, 0.2, D))).astype(np.float32)
    Qv = (r.standard_normal((20, D)) @ np.diag(np.linspace(2, 0.2, D))).astype(np.float32)
    ix = oracle.build(X, M, K=K, rotation_mode=rot, kmeans_iters=8, seed=seed)
    return ix, X, Qv


def test_scores_equal_bruteforce_collision_counts_S402():
    ix, X, Qv = small_index()
    for mode in (0, 1):
        budget = 120
        _, _, t = oracle.search(ix, Qv, k=5, mode=mode, budget=budget, tau=1, trace=True)
        S = oracle.bruteforce_scores(ix["cells"], ix["cb"], t["qrot"], budget, wk=5 if mode else 0)
        assert np.array_equal(t["V"], S)
        if mode == 1:
            _, _, t0 = oracle.search(ix, Qv, k=5, mode=0, budget=budget, tau=1, trace=True)
            assert np.all(t["V"] >= t0["V"])  # weighted >= binary
        for q in range(Qv.shape[0]):  # B <= R_qm < B + max cell
            assert np.all(t["retrieved"][q] >= budget)


@pytest.mark.parametrize("rot", [0, 1])
def test_full_coverage_is_exact_knn_S396(rot):
    ix, X, Qv = small_index(rot=rot)
    ids, d, t = oracle.search(ix, Qv, k=10, mode=0, budget=ix["N"], tau=1, trace=True)
    bi, bd = oracle.bruteforce_knn(ix["X"], t["qrot"], 10)
    assert np.array_equal(ids, bi) and np.array_equal(d, bd)
    # K = 1: a single cell per subspace covers everything even with budget 1
    ix1 = oracle.build(X, 4, K=1, rotation_mode=0, kmeans_iters=3)
    ids1, d1, _ = oracle.search(ix1, Qv, k=10, mode=0, budget=1, tau=1)
    bi1, bd1 = oracle.bruteforce_knn(ix1["X"], Qv, 10)
    assert np.array_equal(ids1, bi1)


def test_self_query_first_S398():
    ix, X, _ = small_index()
    ids, d, _ = oracle.search(ix, X[[5, 77, 901]], k=3, mode=0, budget=60, tau=2)
    assert ids[:, 0].tolist() == [5, 77, 901] and np.all(d[:, 0] == 0.0)


def test_mode_consistency_without_patience_S405():
    ix, _, Qv = small_index()
    a = oracle.search(ix, Qv, k=7, mode=0, budget=150, tau=1)
    b = oracle.search(ix, Qv, k=7, mode=1, budget=150, tau=1, patience_factor=0)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_candidates_threshold_and_fallback():
    ix, _, Qv = small_index()
    M = ix["M"]
    _, _, t = oracle.search(ix, Qv, k=8, mode=0, budget=100, tau=3, trace=True)
    for q in range(Qv.shape[0]):
        n = t["cand_n"][q]
        if not t["fallback"][q]:
            assert t["cand"][q, :n].tolist() == np.nonzero(t["V"][q] >= 3)[0].tolist()
    # tau above any reachable score -> fallback: top-k touched by (V desc, id asc)
    _, _, t = oracle.search(ix, Qv, k=8, mode=0, budget=100, tau=M + 1, trace=True)
    for q in range(Qv.shape[0]):
        V = t["V"][q].astype(int)
        touched = np.nonzero(V)[0]
        order = sorted(touched.tolist(), key=lambda x: (-V[x], x))[:8]
        n = t["cand_n"][q]
        assert t["fallback"][q] == 1 and t["cand"][q, :n].tolist() == sorted(order)


def test_hamming_order_and_patience_prefix_property():
    ix, _, Qv = small_index(N=3000)
    k, P = 5, 2
    ids, d, t = oracle.search(ix, Qv, k=k, mode=1, budget=400, tau=1, patience_factor=P, trace=True)
    W = ix["codes"].shape[1]
    for q in range(Qv.shape[0]):
        n = int(t["cand_n"][q])
        order = t["order"][q, :n]
        qc = oracle.codes(t["qrot"][q:q + 1])[0]
        h = [sum(bin(int(qc[w]) ^ int(ix["codes"][x, w])).count("1") for w in range(W)) for x in order]
        assert all((h[i], order[i]) < (h[i + 1], order[i + 1]) for i in range(n - 1))
        nv = int(t["n_verified"][q])
        assert nv >= min(n, k + P * k)
        dd = [(oracle.dist64(t["qrot"][q], ix["X"][x]), x) for x in order]
        top = sorted(dd[:nv])[:k]
        assert [x for _, x in top] == ids[q, :len(top)].tolist()
        if nv < n:  # stopped early: the last P*k verifications changed nothing
            assert sorted(dd[:nv - P * k])[:k] == top


def test_recall_monotone_in_budget_S404():
    ix, X, Qv = small_index(N=3000, seed=3)
    gt, _ = oracle.bruteforce_knn(ix["X"], Qv, 10)
    prev = -1
    for B in (30, 150, 600, 3000):
        ids, _, _ = oracle.search(ix, Qv, k=10, mode=0, budget=B, tau=1)
        rec = np.mean([len(set(ids[i]) & set(gt[i])) / 10 for i in range(len(ids))])
        assert rec >= prev
        prev = rec
    assert prev == 1.0


def test_exact_parameters_O1():
    assert oracle.budget_ids(0.035, 20000) == 700
    assert oracle.tau_int(0.07, 100) == 7
    assert oracle.tau_int(0.3, 10) == 3
    assert oracle.tau_int(0.1, 4) == 1
    assert oracle.padded_dim(130, 4) == 136


def test_sharded_search_equals_single_index():
    """phi=0 with global cell sizes: per-shard top-k merged by (d, gid) equals
    the 1-index result."""
    ix, X, Qv = small_index(N=2400)
    full = oracle.search(ix, Qv, k=6, mode=0, budget=200, tau=2)
    G = 3
    n = ix["N"] // G
    ds, ids = [], []
    for g in range(G):
        sh = oracle.build(X[g * n:(g + 1) * n], ix["M"], K=ix["K"], rotation_mode=0,
                          codebooks=ix["cb"], gid_base=g * n)
        sh["gsize"] = ix["gsize"]
        i, d, _ = oracle.search(sh, Qv, k=6, mode=0, budget=200, tau=2)
        ds.append(d)
        ids.append(i)
    md, mi = oracle.merge_topk(np.stack(ds), np.stack(ids))
    # the fallback is per shard here, so compare only queries with no fallback
    _, _, t = oracle.search(ix, Qv, k=6, mode=0, budget=200, tau=2, trace=True)
    ok = t["cand_n"] >= 6 * G
    assert ok.sum() > 10
    assert np.array_equal(mi[ok], full[0][ok]) and np.array_equal(md[ok], full[1][ok])


# ---------------------------------------------------------------- Theorem 1
def test_theorem1_closed_form_S450():
    g = gold("theorem1_S450.json")
    assert abs(oracle.hoeffding_bound(g["M"], g["p_star"], g["tau"]) - g["bound"]) < 1e-12
    assert abs(oracle.binomial_failure(16, 0.5, 4) - g["exact_failure_num"] / g["exact_failure_den"]) < 1e-15
    assert math.isnan(oracle.hoeffding_bound(16, 0.25, 4))  # vacuous at equality
    assert oracle.binomial_failure(16, 0.3, 0) == 0.0
    assert oracle.binomial_failure(16, 1.0, 16) == 0.0
    assert abs(oracle.hoeffding_bound(8, 0.5, 0) - (1 - math.exp(-2 * 8 * 0.25))) < 1e-15


def test_theorem1_dominance_grid_S485():
    for M, p in itertools.product((4, 8, 16, 64), (0.3, 0.5, 0.8)):
        for tau in range(0, int(math.ceil(M * p))):
            if M * p > tau:
                fail = oracle.binomial_failure(M, p, tau)
                assert fail <= 1 - oracle.hoeffding_bound(M, p, tau) + 1e-15


def test_guaranteed_mode_recall_bound_invariant():
    """x* in C <=> V(x*) >= tau (deterministic), and on isotropic rotated data
    the measured recall of x* respects Thm 1 at the mean collision rate."""
    r = rng(21)
    N, D, M = 4000, 64, 16
    X = r.standard_normal((N, D)).astype(np.float32)
    Qv = (X[r.integers(0, N, 60)] + 0.3 * r.standard_normal((60, D))).astype(np.float32)
    ix = oracle.build(X, M, K=6, rotation_mode=1, kmeans_iters=8, seed=2)
    tau = 3
    _, _, t = oracle.search(ix, Qv, k=1, mode=0, budget=400, tau=tau, trace=True)
    gt, _ = oracle.bruteforce_knn(ix["X"], t["qrot"], 1)
    hit, pst = [], []
    for q in range(60):
        xs = gt[q, 0]
        n = t["cand_n"][q]
        inC = xs in set(t["cand"][q, :n].tolist())
        if not t["fallback"][q]:
            assert inC == (t["V"][q, xs] >= tau)
        hit.append(t["V"][q, xs] >= tau)
        pst.append(t["V"][q, xs] / M)
    p_lo = float(np.quantile(pst, 0.25))
    if M * p_lo > tau:
        assert np.mean(hit) >= oracle.hoeffding_bound(M, p_lo, tau) - 0.02


def test_rotation_library_qr_matches_plain_householder():
    """oracle.rotation uses LAPACK's QR as a library step; the plain C
    Householder (pinned above) gives the same sign-fixed Q."""
    G = oracle.gaussian_matrix(48, 5)
    Qh, _ = oracle.qr(G)
    _, R64 = oracle.rotation(48, 5)
    assert np.abs(Qh - R64).max() < 1e-12


def test_jacobi_matches_lapack_eigvalsh():
    r = rng(30)
    A = r.standard_normal((40, 40))
    A = A @ A.T
    assert np.allclose(np.sort(oracle.eig_sym(A)), np.linalg.eigvalsh(A), rtol=1e-10, atol=1e-9)


# ---------------------------------------------------------------- f1: ADSampling (Eq. 2)
def test_adsampling_spec_example_S386():
    """SPEC adsampling_verify: D=64, stride 32, a candidate whose first 32 dims
    contribute 100 with r_k^2 = 10 is pruned at t = 32 (100 > ~9.4); r_k^2 = inf
    never prunes and gives the exact squared distance."""
    q = np.zeros(64, np.float32)
    x = np.zeros(64, np.float32)
    x[:32] = np.float32(math.sqrt(100 / 32))
    x[32:] = 1000.0  # a candidate pruned at t = 32 never reads these
    pruned, part = oracle.adsampling_verify(q, x, 10.0)
    assert pruned and abs(part - 100.0) < 1e-4
    pruned, full = oracle.adsampling_verify(q, x, math.inf)
    assert not pruned and full == oracle.dist64(q, x)


def test_adsampling_threshold_brackets_spec_value():
    """The t = 32 threshold of the SPEC example (r_k^2 = 10, D = 64) lies
    between 9.0 and 9.6 (SPEC prints ~9.37): partial 9.0 survives, 9.6 is pruned."""
    q = np.zeros(64, np.float32)
    for part, expect in ((9.0, False), (9.6, True)):
        x = np.zeros(64, np.float32)
        x[:32] = np.float32(math.sqrt(part / 32))
        assert oracle.adsampling_verify(q, x, 10.0)[0] is expect


def test_adsampling_checks_only_at_stride_multiples():
    """A large early contribution is caught at the first checkpoint, t = 32: the
    returned partial covers exactly the first 32 dimensions."""
    q = np.zeros(96, np.float32)
    x = np.full(96, 0.5, np.float32)
    x[:4] = 50.0
    pruned, part = oracle.adsampling_verify(q, x, 1.0)
    assert pruned and part == oracle.dist64(q[:32], x[:32])
    # stride 0 disables the checks entirely
    assert oracle.adsampling_verify(q, x, 1.0, stride=0) == (False, oracle.dist64(q, x))


def test_adsampling_prune_monotone_in_rk_and_margin():
    """A smaller r_k or a smaller margin can only prune more (Eq. 2 is monotone)."""
    r = rng(3)
    D = 128
    for _ in range(300):
        q = r.standard_normal(D).astype(np.float32)
        x = (q + 0.5 * r.standard_normal(D)).astype(np.float32)
        full = oracle.dist64(q, x)
        for rk2 in (0.3 * full, 0.6 * full, 0.9 * full, 1.2 * full):
            if oracle.adsampling_verify(q, x, rk2, eps0=2.1)[0]:
                assert oracle.adsampling_verify(q, x, 0.7 * rk2, eps0=2.1)[0]
                assert oracle.adsampling_verify(q, x, rk2, eps0=1.0)[0]


def test_adsampling_degenerate_margin_is_exact_verification():
    """eps0 -> 1e9: no candidate is ever pruned, so Optimized Mode with
    ADSampling equals Optimized Mode with exact L2 (SPEC mode-consistency),
    including the patience stop."""
    ix, _, Qv = small_index(N=3000)
    kw = dict(k=5, mode=1, budget=400, tau=1, patience_factor=2, trace=True)
    a = oracle.search(ix, Qv, **kw)
    b = oracle.search(ix, Qv, adsampling=True, eps0=1e9, **kw)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.array_equal(a[2]["n_verified"], b[2]["n_verified"])


def test_adsampling_search_exact_distances_and_recall():
    """With ADSampling on a rotated index: every returned distance is the exact
    dist64 of its id (a pruned candidate is never returned), prunes count as
    non-improving verifications, and the result stays close to exact
    verification ("negligible cost to recall")."""
    ix, X, Qv = small_index(N=4000, D=64, M=4, K=8, rot=1)
    kw = dict(k=10, mode=1, budget=800, tau=1, patience_factor=5, trace=True)
    ids_e, d_e, _ = oracle.search(ix, Qv, **kw)
    ids_a, d_a, t = oracle.search(ix, Qv, adsampling=True, **kw)
    hits = 0
    for q in range(Qv.shape[0]):
        for i, x in enumerate(ids_a[q]):
            assert x >= 0 and d_a[q, i] == oracle.dist64(t["qrot"][q], ix["X"][x])
        hits += len(set(ids_a[q].tolist()) & set(ids_e[q].tolist()))
    assert hits / ids_e.size >= 0.9


# --------------------------------------------------------------------------
# Exact patience stop (O15 step 4; Z11) and ADSampling prune-as-miss
# (Eq. 2 with P:L458), on integer-valued data so every squared distance is an
# exact integer (no rounding on either side: the Python sums below are exact).
# --------------------------------------------------------------------------
def _int_index(N=2500, D=32, M=4, K=6, seed=21, lo=-6, hi=7, rot=0):
    r = rng(seed)
    X = r.integers(lo, hi, (N, D)).astype(np.float32)
    X[N // 2: N // 2 + 40] = X[:40]  # duplicate rows: exact distance ties, broken by id
    Qv = r.integers(lo, hi, (12, D)).astype(np.float32)
    ix = oracle.build(X, M, K=K, rotation_mode=rot, kmeans_iters=6, seed=seed)
    return ix, X, Qv


def _exact_d2(q, x):
    return int(np.sum((q.astype(np.int64) - x.astype(np.int64)) ** 2))


@pytest.mark.parametrize("P", [1, 2, 3])
def test_patience_stop_is_exact(P):
    """The stop index n_verified is pinned exactly: the verification at
    position nv - P*k - 1 (0-based) improved the top-k (the counter was reset
    there), the P*k after it did not, and no run of P*k consecutive
    non-improvements ends earlier; an oracle stopping one verification late or
    early fails one of the three."""
    ix, X, Qv = _int_index()
    k = 4
    ids, d, t = oracle.search(ix, Qv, k=k, mode=1, budget=300, tau=1, patience_factor=P, trace=True)
    Pk = P * k
    stopped = 0
    for q in range(Qv.shape[0]):
        n, nv = int(t["cand_n"][q]), int(t["n_verified"][q])
        order = t["order"][q, :n]
        dd = [(_exact_d2(Qv[q], X[x]), int(x)) for x in order]
        # improvement flags by definition: |H| < k or (d, id) < max(H) (Z11)
        imp = []
        for i in range(n):
            prev = sorted(dd[:i])[:k]
            imp.append(len(prev) < k or dd[i] < prev[-1])
        assert [x for _, x in sorted(dd[:nv])[:k]] == ids[q, :min(k, nv)].tolist()
        if nv < n:
            stopped += 1
            assert imp[nv - Pk - 1], "the counter was reset P*k verifications before the stop"
            assert not any(imp[nv - Pk:nv]), "the last P*k verifications changed nothing"
        run = 0
        for i in range(nv - Pk if nv < n else n - 1):  # (a run may end exactly at the last candidate)
            run = 0 if imp[i] else run + 1
            assert run < Pk, "an earlier run of P*k non-improvements would have stopped"
    assert stopped >= 3


def test_adsampling_prune_counts_as_non_improvement():
    """A constructed case where only prunes can end the search: the query's k
    near neighbours come first in Hamming order (all coordinates positive, like
    the query), then only far points (all negative: every one is pruned at
    the first checkpoint t = 32 by Eq. 2).  Since a prune is a non-improving
    verification, the search stops after exactly k + P*k candidates;
    an oracle whose prunes did not advance the counter would verify all."""
    r = rng(5)
    D, k, P = 64, 5, 2
    q = np.full((1, D), 3.0, np.float32)
    near = (3.0 + r.integers(-1, 2, (k, D))).astype(np.float32)
    far = (-6.0 - r.integers(0, 3, (300, D))).astype(np.float32)
    X = np.vstack([far[:150], near, far[150:]])
    ix = oracle.build(X, 2, K=2, rotation_mode=0, kmeans_iters=3, seed=1)
    N = X.shape[0]
    kw = dict(k=k, mode=1, budget=N, tau=1, patience_factor=P, trace=True)
    ids, d, t = oracle.search(ix, q, adsampling=True, **kw)
    assert int(t["cand_n"][0]) == N
    assert sorted(t["order"][0, :k].tolist()) == list(range(150, 150 + k)), "near points first in Hamming order"
    assert int(t["n_verified"][0]) == k + P * k
    assert sorted(ids[0].tolist()) == list(range(150, 150 + k))
    # every far point is pruned at t = 32 (its partial sum alone exceeds Eq. 2's bound)
    rk2 = max(_exact_d2(q[0], X[i]) for i in range(150, 150 + k))
    thr = oracle.adsampling_threshold(float(rk2), 32, D, 2.1)
    assert all(_exact_d2(q[0, :32], X[i, :32]) > thr for i in list(range(150)) + list(range(155, N)))


# --------------------------------------------------------------------------
# f4: block-wise variance redistribution (DESIGN reading R16)
# --------------------------------------------------------------------------
def test_blockwise_rotation_selects_the_energetic_subspaces():
    """A dataset whose subspace 2 carries 100x the variance of the others (and
    subspace 5 10x): the block of b = 1 is subspace 2's dimensions, of b = 2
    subspaces 2 and 5, in ascending order; equal energies go to the smaller m."""
    r = rng(7)
    M, D = 8, 64
    scale = np.ones(D)
    scale[16:24] = 10.0   # subspace 2 (8 dims each)
    scale[40:48] = np.sqrt(10.0)  # subspace 5
    X = (r.standard_normal((20000, D)) * scale).astype(np.float32)
    var = oracle.dim_variances(X, 3)  # the 2000-row CEV sample
    assert np.allclose(var, scale ** 2, rtol=0.2)
    assert oracle.rotation_block(var, M, D, 1).tolist() == list(range(16, 24))
    assert oracle.rotation_block(var, M, D, 2).tolist() == list(range(16, 24)) + list(range(40, 48))
    assert oracle.rotation_block(np.ones(D), M, D, 2).tolist() == list(range(0, 16))


def test_blockwise_rotation_is_identity_outside_and_orthogonal_inside():
    """R is the identity outside the block (exactly), orthogonal on it; X' keeps
    every dimension outside the block bit for bit and the block's norm per row
    (isometry), and the block is really mixed."""
    r = rng(8)
    M, D = 8, 64
    scale = np.ones(D)
    scale[24:32] = 20.0
    X = (r.standard_normal((3000, D)) * scale).astype(np.float32)
    R, blk = oracle.blockwise_rotation(X, M, D, 2, 5)
    out = np.setdiff1d(np.arange(D), blk)
    assert np.array_equal(R[np.ix_(out, np.arange(D))], np.eye(D, dtype=np.float32)[out])
    assert np.array_equal(R[np.ix_(np.arange(D), out)], np.eye(D, dtype=np.float32)[:, out])
    Rb = R[np.ix_(blk, blk)].astype(np.float64)
    assert np.abs(Rb @ Rb.T - np.eye(len(blk))).max() < 1e-5
    assert np.abs(Rb - np.eye(len(blk))).max() > 0.1
    ox = oracle.build(X, M, K=6, rotation_mode=1, kmeans_iters=2, seed=5, rotation_block=2)
    assert np.array_equal(ox["R"], R)
    assert np.array_equal(ox["X"][:, out], X[:, out])
    nb = np.linalg.norm(X[:, blk].astype(np.float64), axis=1)
    assert np.allclose(np.linalg.norm(ox["X"][:, blk].astype(np.float64), axis=1), nb, rtol=1e-5)


# --------------------------------------------------------------------------
# f4: adaptive subspace decomposition (DESIGN reading R18)
# --------------------------------------------------------------------------
def test_adaptive_widths_rule_by_hand_and_limits():
    """Worked case: v = (8,4,2,1,1,1,1,.5 x5), M = 3, T = 20.5: cut 1 is the
    first even e with S(e) >= 6.83 (S(2) = 12), cut 2 the first even e >= 4
    with S(e) >= 13.67 (S(4) = 15): widths (2, 2, 8), the high-variance region
    in narrow subspaces.  A flat spectrum gives the paper's equal split; a
    single spike squeezes every cut to the minimum width 2."""
    v = [8, 4, 2, 1, 1, 1, 1, .5, .5, .5, .5, .5]
    assert oracle.adaptive_widths(v, 3, 12) == [2, 2, 8]
    assert oracle.adaptive_widths(np.ones(48), 4, 48) == [12] * 4
    assert oracle.adaptive_widths(np.ones(40), 4, 48) == [10, 10, 10, 18]  # zero-variance padding
    assert oracle.adaptive_widths([100.0] + [0.0] * 31, 4, 32) == [2, 2, 2, 26]
    for seed in range(5):
        w = oracle.adaptive_widths(rng(seed).exponential(1.0, 60) ** 3, 6, 60)
        assert sum(w) == 60 and all(x >= 2 and x % 2 == 0 for x in w)
    h = oracle.half_offsets([2, 2, 8])
    assert h.tolist() == [0, 1, 2, 3, 4, 8, 12] and oracle.half_stride(h) == 4


def _pad_halves(X, hoff, dh):
    """each half's dims first in a slot of dh, zeros after (the equal-width layout)"""
    out = np.zeros((X.shape[0], (len(hoff) - 1) * dh), dtype=np.float32)
    for h in range(len(hoff) - 1):
        w = hoff[h + 1] - hoff[h]
        out[:, h * dh: h * dh + w] = X[:, hoff[h]: hoff[h + 1]]
    return out


@pytest.mark.parametrize("mode", [0, 1])
def test_adaptive_subspaces_equal_zero_padded_equal_split(mode):
    """An index with widths (2, 2, 8) equals, bit for bit, the equal-split index
    of the same vectors with each half moved into a dh = 4 slot and zero
    filled: zero dimensions add exact zeros to every dist64 (k-means++, Lloyd,
    assignment, half distances, verification keep their real terms in the same
    order) and a 0 bit to both codes.  A wrong half offset, width or codebook
    stride breaks the equality."""
    r = rng(11)
    N, D, M, K = 3000, 12, 3, 5
    X = (r.standard_normal((N, D)) * np.array([6, 5, 4, 3, 1, 1, 1, 1, .5, .5, .5, .5])).astype(np.float32)
    Qv = (r.standard_normal((20, D)) * 2).astype(np.float32)
    oa = oracle.build(X, M, K=K, rotation_mode=0, kmeans_iters=6, seed=2, subspace_widths=[2, 2, 8])
    assert oa["hoff"].tolist() == [0, 1, 2, 3, 4, 8, 12] and oa["dh"] == 4
    Xp = _pad_halves(X, oa["hoff"], 4)
    ou = oracle.build(Xp, M, K=K, rotation_mode=0, kmeans_iters=6, seed=2)
    assert ou["dh"] == 4 and ou["hoff"] is None
    assert np.array_equal(oa["cb"], ou["cb"]) and np.array_equal(oa["cells"], ou["cells"])
    assert np.array_equal(oa["ids"], ou["ids"])
    B, tau, k = 600, 2, 10
    ia, da, ta = oracle.search(oa, Qv, k, mode, B, tau, patience_factor=3, trace=True)
    iu, du, tu = oracle.search(ou, _pad_halves(Qv, oa["hoff"], 4), k, mode, B, tau, patience_factor=3, trace=True)
    assert np.array_equal(ia, iu) and np.array_equal(da, du)
    assert np.array_equal(ta["act_cell"], tu["act_cell"]) and np.array_equal(ta["V"], tu["V"])
    assert np.array_equal(ta["n_verified"], tu["n_verified"])
    # the brute-force scores (no CSR, no heap) agree with the search's V
    S = oracle.bruteforce_scores(oa["cells"], oa["cb"], ta["qrot"], B, k if mode == 1 else 0, oa["hoff"])
    assert np.array_equal(S, ta["V"])


def test_adaptive_rule_in_build_and_equal_widths_are_the_default():
    """adaptive_subspaces=True takes the widths of the rule on the stored
    vectors' CEV-sample variances (a decaying spectrum: narrow leading
    subspaces); explicit equal widths reproduce the default index."""
    r = rng(12)
    N, D, M = 4000, 32, 4
    X = (r.standard_normal((N, D)) * np.exp(-np.arange(D) / 6.0)).astype(np.float32)
    oa = oracle.build(X, M, K=4, rotation_mode=0, kmeans_iters=3, seed=1, adaptive_subspaces=True)
    w = oracle.adaptive_widths(oracle.dim_variances(X, 1), M, 32)
    assert (oa["hoff"][2::2] - oa["hoff"][:-1:2]).tolist() == w
    assert w[0] < 8 < w[-1]
    o1 = oracle.build(X, M, K=4, rotation_mode=0, kmeans_iters=3, seed=1)
    o2 = oracle.build(X, M, K=4, rotation_mode=0, kmeans_iters=3, seed=1, subspace_widths=[8] * 4)
    assert np.array_equal(o1["cb"], o2["cb"]) and np.array_equal(o1["cells"], o2["cells"])
