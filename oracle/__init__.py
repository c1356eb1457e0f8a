"""CPU oracle for CRISP (arXiv 2603.05180) -- TEST INFRASTRUCTURE ONLY.

Plain, slow, fp64 reference of the method, written from PAPER.md.  The
arithmetic lives in ``crisp_oracle.c`` (plain C, -O2 -ffp-contract=off,
OpenMP over queries); this module only marshals numpy arrays and composes the
C steps in the paper's order.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` leg may import it.  It shares
no code with ``paper_2603_05180_b200`` (the CUDA path) and never imports it.

Parity status: pinned by ``tests/test_oracle_*.py`` (see DESIGN.md
"Oracle pins").  Unpinned: absolute recall values, k-means centroid values
beyond the closed-form cases (Lloyd monotonicity, k=1 mean, k=n cover).
"""
from __future__ import annotations

import ctypes as C
import math
import hashlib
import os
import subprocess
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "crisp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O3", "-march=x86-64-v3", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def compile_oracle(force: bool = False) -> str:
    """Compile liboracle.so in-tree with gcc (the checker, not the product)."""
    with open(_SRC, "rb") as f:
        digest = hashlib.sha256(f.read() + " ".join(CFLAGS).encode()).hexdigest()
    stamp = _LIB + ".sha256"
    fresh = os.path.exists(_LIB) and os.path.exists(stamp) and open(stamp).read().strip() == digest
    if force or not fresh:  # content-based: a checkout that changes the source always rebuilds
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
        with open(stamp, "w") as f:
            f.write(digest + "\n")
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(compile_oracle())
        _declare(_lib)
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _declare(L):
    vp, i32, i64, u32, u64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double
    L.or_philox4x32_10.argtypes = [vp, vp, vp]
    L.or_uniform.argtypes = [u64, u32, u64, u32]
    L.or_uniform.restype = f64
    L.or_normal.argtypes = [u64, u32, u64, u32]
    L.or_normal.restype = f64
    L.or_dist64.argtypes = [vp, vp, i64]
    L.or_dist64.restype = f64
    L.or_sample_rows.argtypes = [i64, i64, u64, u32, vp]
    L.or_cev_sample_size.argtypes = [i64]
    L.or_cev_sample_size.restype = i64
    L.or_covariance.argtypes = [vp, i64, vp, i64, i32, vp]
    L.or_eig_sym_jacobi.argtypes = [vp, i32, vp]
    L.or_cev_from_eigs.argtypes = [vp, i32]
    L.or_cev_from_eigs.restype = f64
    L.or_cev.argtypes = [vp, i64, i64, i32, u64]
    L.or_cev.restype = f64
    L.or_gaussian_matrix.argtypes = [i32, u64, vp]
    L.or_qr_householder.argtypes = [vp, i32, vp, vp]
    L.or_rotation.argtypes = [i32, u64, vp, vp]
    L.or_rotate_rows.argtypes = [vp, i64, i32, i64, vp, vp, i64]
    L.or_argmin_centroid.argtypes = [vp, vp, i32, i32, vp]
    L.or_argmin_centroid.restype = i32
    L.or_kmeans.argtypes = [vp, i64, i64, i32, i32, i32, u64, u32, vp, vp]
    L.or_train_codebooks.argtypes = [vp, i64, i64, i32, i32, i32, i32, i64, u64, vp, vp]
    L.or_assign.argtypes = [vp, i64, i64, i32, i32, i32, vp, vp, vp]
    L.or_csr.argtypes = [vp, i64, i32, i32, vp, vp]
    L.or_codes.argtypes = [vp, i64, i64, i32, vp]
    L.or_half_sorted.argtypes = [vp, vp, i32, i32, vp, vp]
    L.or_multisequence.argtypes = [vp, vp, vp, vp, i32, vp, i64, i32, vp, vp, vp]
    L.or_multisequence.restype = i32
    L.or_search.argtypes = [i64, i64, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, i64, i32, i32, i32, f64, i32,
                            i32, vp, vp, vp, i64, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    L.or_adsampling_threshold.argtypes = [f64, i32, i32, f64]
    L.or_adsampling_threshold.restype = f64
    L.or_adsampling_verify.argtypes = [vp, vp, i32, f64, f64, i32, vp]
    L.or_adsampling_verify.restype = i32
    L.or_max_threads.restype = i32
    L.or_bruteforce_knn.argtypes = [vp, i64, i32, vp, i64, i32, vp, vp]
    L.or_bruteforce_scores.argtypes = [vp, i64, i32, i32, i32, i32, vp, vp, vp, i64, i64, i32, vp]
    L.or_merge_topk.argtypes = [vp, vp, i32, i64, i32, vp, vp]
    L.or_hoeffding_bound.argtypes = [i32, f64, f64]
    L.or_hoeffding_bound.restype = f64
    L.or_binomial_failure.argtypes = [i32, f64, i32]
    L.or_binomial_failure.restype = f64


# --------------------------------------------------------------------------
# Exact integer parameters: B = ceil(beta*N), tau = ceil(alpha*M)
# with beta/alpha read as the decimal they were written as.
# --------------------------------------------------------------------------
def exact_ceil(ratio, n: int) -> int:
    return int(math.ceil(Fraction(str(ratio)) * n))


def budget_ids(beta, N: int) -> int:
    """B = ceil(beta * N) ids per subspace (Z1, Z3)."""
    return max(1, exact_ceil(beta, N))


def tau_int(alpha, M: int) -> int:
    """tau = ceil(alpha * M) (Z1), at least 1 (touched points only)."""
    return max(1, exact_ceil(alpha, M))


def padded_dim(D: int, M: int) -> int:
    """Zero-pad D up to a multiple of 2M (Z17)."""
    return ((D + 2 * M - 1) // (2 * M)) * (2 * M)


# --------------------------------------------------------------------------
# Wrappers of single steps
# --------------------------------------------------------------------------
def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().or_philox4x32_10(_p(c), _p(k), _p(o))
    return o


def dist64(a, b) -> float:
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    return lib().or_dist64(_p(a), _p(b), a.size)


def sample_rows(N: int, n: int, seed: int, stream: int):
    out = np.zeros(n, dtype=np.int64)
    lib().or_sample_rows(N, n, seed, stream, _p(out))
    return out


def cev_sample_size(N: int) -> int:
    return lib().or_cev_sample_size(N)


def covariance(X, rows):
    X = np.ascontiguousarray(X, dtype=np.float32)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    D = X.shape[1]
    Cm = np.zeros((D, D), dtype=np.float64)
    lib().or_covariance(_p(X), D, _p(rows), rows.size, D, _p(Cm))
    return Cm


def eig_sym(A):
    A = np.array(A, dtype=np.float64, order="C", copy=True)
    D = A.shape[0]
    w = np.zeros(D, dtype=np.float64)
    lib().or_eig_sym_jacobi(_p(A), D, _p(w))
    return w


def cev_from_eigs(w) -> float:
    w = np.array(w, dtype=np.float64, copy=True)
    return lib().or_cev_from_eigs(_p(w), w.size)


def cev(X, seed: int) -> float:
    """Spectral check: covariance of the bounded sample (C, fp64),
    eigenvalues by LAPACK (numpy.linalg.eigvalsh, a library step), CEV (C)."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    N = X.shape[0]
    n = cev_sample_size(N)
    if n < 2:
        return 0.0
    rows = np.arange(N, dtype=np.int64) if n == N else sample_rows(N, n, seed, 1)
    w = np.linalg.eigvalsh(covariance(X, rows))
    return cev_from_eigs(w)


def dim_variances(X, seed: int):
    """Per-dimension variances of the CEV sample (the diagonal of its covariance,
    divisor n-1), fp64; zeros if the sample has fewer than 2 rows."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    N, D = X.shape
    n = cev_sample_size(N)
    if n < 2:
        return np.zeros(D)
    rows = np.arange(N, dtype=np.int64) if n == N else sample_rows(N, n, seed, 1)
    return np.diag(covariance(X, rows)).copy()


def rotation_block(var, M: int, Dp: int, b: int):
    """Block-wise variance redistribution (reading R16): the b subspaces
    of largest variance energy E_m = sum of the per-dimension variances of
    their 2 d_h dimensions (summed in ascending dimension, fp64; ties to the
    smaller m), returned as their dimensions in ascending order."""
    v = np.zeros(Dp)
    v[: len(var)] = var
    w = Dp // M
    E = []
    for m in range(M):
        e = 0.0
        for i in range(m * w, (m + 1) * w):
            e += v[i]
        E.append(e)
    top = sorted(range(M), key=lambda m: (-E[m], m))[:b]
    return np.concatenate([np.arange(m * w, (m + 1) * w) for m in sorted(top)])


def blockwise_rotation(X, M: int, Dp: int, b: int, seed: int):
    """R = I except on the block's dimensions, where it is Q of QR of a d_sub x
    d_sub Gaussian (the rotation of P:L225 restricted to the block)."""
    blk = rotation_block(dim_variances(X, seed), M, Dp, b)
    Rs, _ = rotation(len(blk), seed)
    R = np.eye(Dp, dtype=np.float32)
    R[np.ix_(blk, blk)] = Rs
    return R, blk


def adaptive_widths(var, M: int, Dp: int):
    """Adaptive subspace decomposition (reading R18): contiguous
    subspace widths, even and >= 2, cut where the running variance first
    reaches j/M of the total, so that high-variance regions get fewer
    dimensions and low-variance regions more.  var: per-dimension variances
    (zero beyond its length); sums in ascending dimension, fp64.  Cut j is the
    smallest even e in [c_{j-1} + 2, Dp - 2(M - j)] with S(e) >= T j / M
    (S(e) = sum of v_i for i < e, T = S(Dp)), else the upper end."""
    v = np.zeros(Dp)
    v[: len(var)] = var
    S = [0.0]
    for x in v:
        S.append(S[-1] + float(x))
    T = S[Dp]
    cuts = [0]
    for j in range(1, M):
        e, hi, target = cuts[-1] + 2, Dp - 2 * (M - j), (T * j) / M
        while e < hi and S[e] < target:
            e += 2
        cuts.append(e)
    cuts.append(Dp)
    return [cuts[j + 1] - cuts[j] for j in range(M)]


def half_offsets(widths):
    """2M+1 half offsets from M even subspace widths (equal halves)."""
    h, o = [], 0
    for w in widths:
        assert w >= 2 and w % 2 == 0, "subspace widths must be even and >= 2"
        h += [o, o + w // 2]
        o += w
    return np.array(h + [o], dtype=np.int32)


def half_stride(hoff) -> int:
    """codebook row stride: the largest half width"""
    hoff = np.asarray(hoff)
    return int(np.max(hoff[1:] - hoff[:-1]))


def _hoff(hoff):
    return None if hoff is None else np.ascontiguousarray(hoff, dtype=np.int32)


def qr(G):
    A = np.array(G, dtype=np.float64, order="C", copy=True)
    D = A.shape[0]
    Q = np.zeros((D, D), dtype=np.float64)
    rd = np.zeros(D, dtype=np.float64)
    lib().or_qr_householder(_p(A), D, _p(Q), _p(rd))
    return Q, rd


def gaussian_matrix(D: int, seed: int):
    G = np.zeros((D, D), dtype=np.float64)
    lib().or_gaussian_matrix(D, seed, _p(G))
    return G


def rotation(D: int, seed: int):
    """R (fp32) and its fp64 source Q: G from the Philox generator, Q of
    QR(G) by LAPACK (numpy.linalg.qr, a library step) with diag(R') > 0.
    The plain Householder or_qr_householder is pinned against it in the tests."""
    G = gaussian_matrix(D, seed)
    Qm, Rm = np.linalg.qr(G)
    sg = np.where(np.diag(Rm) < 0, -1.0, 1.0)
    R64 = np.ascontiguousarray(Qm * sg[None, :])
    return R64.astype(np.float32), R64


def rotate_rows(X, R):
    X = np.ascontiguousarray(X, dtype=np.float32)
    R = np.ascontiguousarray(R, dtype=np.float32)
    n, D = X.shape
    Y = np.zeros_like(X)
    lib().or_rotate_rows(_p(X), n, D, D, _p(R), _p(Y), D)
    return Y


def kmeans(pts, K: int, iters: int, seed: int, half: int = 0):
    pts = np.ascontiguousarray(pts, dtype=np.float32)
    n, dh = pts.shape
    Cm = np.zeros((K, dh), dtype=np.float32)
    obj = np.zeros(max(iters, 1), dtype=np.float64)
    lib().or_kmeans(_p(pts), n, dh, dh, K, iters, seed, half, _p(Cm), _p(obj))
    return Cm, obj[:iters]


def train_codebooks(X, M: int, K: int, iters: int, sample: int, seed: int, hoff=None):
    """Codebooks of the 2M halves; hoff (2M+1 half offsets, R18) or equal halves."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    N, Dp = X.shape
    dh = Dp // (2 * M) if hoff is None else half_stride(hoff)
    cb = np.zeros((M, 2, K, dh), dtype=np.float32)
    lib().or_train_codebooks(_p(X), N, Dp, M, K, dh, iters, sample, seed, _p(_hoff(hoff)), _p(cb))
    return cb


def assign(X, cb, hoff=None):
    X = np.ascontiguousarray(X, dtype=np.float32)
    cb = np.ascontiguousarray(cb, dtype=np.float32)
    N, Dp = X.shape
    M, _, K, dh = cb.shape
    cells = np.zeros((M, N), dtype=np.int32)
    lib().or_assign(_p(X), N, Dp, M, K, dh, _p(_hoff(hoff)), _p(cb), _p(cells))
    return cells


def csr(cells, K: int):
    cells = np.ascontiguousarray(cells, dtype=np.int32)
    M, N = cells.shape
    off = np.zeros((M, K * K + 1), dtype=np.int64)
    ids = np.zeros((M, N), dtype=np.int32)
    lib().or_csr(_p(cells), N, M, K, _p(off), _p(ids))
    return off, ids


def codes(X):
    X = np.ascontiguousarray(X, dtype=np.float32)
    N, D = X.shape
    W = (D + 63) // 64
    out = np.zeros((N, W), dtype=np.uint64)
    lib().or_codes(_p(X), N, D, D, _p(out))
    return out


def half_sorted(qh, Ch):
    qh = np.ascontiguousarray(qh, dtype=np.float32)
    Ch = np.ascontiguousarray(Ch, dtype=np.float32)
    K, dh = Ch.shape
    d = np.zeros(K, dtype=np.float64)
    p = np.zeros(K, dtype=np.int32)
    lib().or_half_sorted(_p(qh), _p(Ch), K, dh, _p(d), _p(p))
    return d, p


def multisequence(a, pa, b, pb, gsize, budget: int, wk: int = 0):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    pa = np.ascontiguousarray(pa, dtype=np.int32)
    pb = np.ascontiguousarray(pb, dtype=np.int32)
    gsize = np.ascontiguousarray(gsize, dtype=np.int64)
    K = a.size
    cl = np.zeros(K * K, dtype=np.int32)
    wl = np.zeros(K * K, dtype=np.int32)
    ret = np.zeros(1, dtype=np.int64)
    L = lib().or_multisequence(_p(a), _p(pa), _p(b), _p(pb), K, _p(gsize), budget, wk, _p(cl), _p(wl), _p(ret))
    return cl[:L], wl[:L], int(ret[0])


def hoeffding_bound(M: int, pstar: float, tau: float) -> float:
    return lib().or_hoeffding_bound(M, pstar, tau)


def binomial_failure(M: int, p: float, tau: int) -> float:
    return lib().or_binomial_failure(M, p, tau)


def bruteforce_knn(X, Qv, k: int):
    X = np.ascontiguousarray(X, dtype=np.float32)
    Qv = np.ascontiguousarray(Qv, dtype=np.float32)
    ids = np.zeros((Qv.shape[0], k), dtype=np.int64)
    d = np.zeros((Qv.shape[0], k), dtype=np.float64)
    lib().or_bruteforce_knn(_p(X), X.shape[0], X.shape[1], _p(Qv), Qv.shape[0], k, _p(ids), _p(d))
    return ids, d


def bruteforce_scores(cells, cb, qrot, budget: int, wk: int = 0, hoff=None):
    cells = np.ascontiguousarray(cells, dtype=np.int32)
    cb = np.ascontiguousarray(cb, dtype=np.float32)
    qrot = np.ascontiguousarray(qrot, dtype=np.float32)
    M, N = cells.shape
    _, _, K, dh = cb.shape
    Q, D = qrot.shape
    S = np.zeros((Q, N), dtype=np.uint16)
    lib().or_bruteforce_scores(_p(cells), N, D, M, K, dh, _p(_hoff(hoff)), _p(cb), _p(qrot), Q, budget, wk, _p(S))
    return S


def merge_topk(d, ids):
    """d, ids: (G, Q, k) per-shard lists -> (Q, k) by (d, gid)."""
    d = np.ascontiguousarray(d, dtype=np.float64)
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    G, Q, k = d.shape
    od = np.zeros((Q, k), dtype=np.float64)
    oi = np.zeros((Q, k), dtype=np.int64)
    lib().or_merge_topk(_p(d), _p(ids), G, Q, k, _p(od), _p(oi))
    return od, oi


def max_threads() -> int:
    return lib().or_max_threads()


# --------------------------------------------------------------------------
# Composition: build (P:L249-256 phases 1-2) and search (Alg. 1)
# --------------------------------------------------------------------------
def build(X, M: int, K: int = 50, tau_cev: float = 0.85, rotation_mode: int = -1, kmeans_iters: int = 20,
          kmeans_sample: int = 100000, seed: int = 0, R=None, codebooks=None, gid_base: int = 0,
          rotation_block: int = 0, adaptive_subspaces: bool = False, subspace_widths=None):
    """Index build: spectral check + adaptive rotation, codebooks,
    cell assignment, CSR, binary codes.

    ``R`` / ``codebooks`` inject the rotation / codebooks (as crisp_build_with).
    ``subspace_widths`` (M even widths summing to Dp) or ``adaptive_subspaces``
    (widths from the stored vectors' per-dimension variances, R18) replace the
    equal split."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    N, D = X.shape
    Dp = padded_dim(D, M)
    dh = Dp // (2 * M)
    Xp = np.zeros((N, Dp), dtype=np.float32)
    Xp[:, :D] = X
    cev_v = cev(X, seed) if N >= 2 else 0.0
    if R is not None:
        rotated = True
        R = np.ascontiguousarray(R, dtype=np.float32)
    else:
        rotated = (cev_v > tau_cev) if rotation_mode < 0 else bool(rotation_mode)  # strict ">" (Z15)
        if rotated:
            # rotation_block = b > 0: block-wise variance redistribution over the b subspaces of
            # largest variance energy (reading R16); else the global rotation
            R = blockwise_rotation(X, M, Dp, rotation_block, seed)[0] if rotation_block > 0 else rotation(Dp, seed)[0]
    if rotated:
        Xp = rotate_rows(Xp, R)
    hoff = None
    if subspace_widths is not None or adaptive_subspaces:
        widths = list(subspace_widths) if subspace_widths is not None else adaptive_widths(
            dim_variances(Xp, seed), M, Dp)
        assert len(widths) == M and sum(widths) == Dp, "M widths summing to the padded dimensionality"
        hoff = half_offsets(widths)
        dh = half_stride(hoff)
    if codebooks is None:
        cb = train_codebooks(Xp, M, K, kmeans_iters, min(N, kmeans_sample), seed, hoff)
    else:
        cb = np.ascontiguousarray(codebooks, dtype=np.float32).reshape(M, 2, K, dh)
    cells = assign(Xp, cb, hoff)
    off, ids = csr(cells, K)
    cds = codes(Xp)
    gsize = (off[:, 1:] - off[:, :-1]).astype(np.int64)
    return dict(N=N, D=D, Dp=Dp, M=M, K=K, dh=dh, hoff=hoff, X=Xp, R=R if rotated else None, rotated=rotated, cev=cev_v,
                cb=cb, cells=cells, off=off, ids=ids, codes=cds, gsize=gsize, gid_base=gid_base, N_budget=N)


def adsampling_threshold(rk2: float, t: int, D: int, eps0: float = 2.1) -> float:
    """Eq. 2: r_k^2 * (t/D) * (1 + eps0/sqrt(t))^2."""
    return lib().or_adsampling_threshold(rk2, t, D, eps0)


def adsampling_verify(q, x, rk2: float, eps0: float = 2.1, stride: int = 32):
    """SPEC adsampling_verify: (pruned, partial-or-exact squared distance)."""
    q = np.ascontiguousarray(q, dtype=np.float32)
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.zeros(1, dtype=np.float64)
    pr = lib().or_adsampling_verify(_p(q), _p(x), q.size, rk2, eps0, stride, _p(out))
    return bool(pr), float(out[0])


def search(index, queries, k: int, mode: int, budget: int, tau: int, patience_factor: int = 40,
           trace: bool = False, nthreads: int = 0, fallback: bool = True, ext_cand=None, ext_n=None,
           adsampling: bool = False, eps0: float = 2.1, ad_stride: int = 32):
    """Alg. 1 for a batch of queries.  budget/tau are the exact integers (O1).
    fallback=False skips the underflow fallback (first phase of the sharded
    protocol); ext_cand/ext_n (Q x N, Q; n < 0 = not given) replace C_q by a
    given ascending candidate list (its final phase).
    adsampling=True verifies Optimized Mode candidates by ADSampling (Eq. 2).
    Returns (ids int64 QxK global, d64 QxK, trace dict or None)."""
    ix = index
    q = np.ascontiguousarray(queries, dtype=np.float32)
    Q = q.shape[0]
    qp = np.zeros((Q, ix["Dp"]), dtype=np.float32)
    qp[:, : q.shape[1]] = q
    N, M, K = ix["N"], ix["M"], ix["K"]
    KK = K * K
    out_ids = np.zeros((Q, k), dtype=np.int64)
    out_d = np.zeros((Q, k), dtype=np.float64)
    t = None
    if trace:
        t = dict(act_len=np.zeros((Q, M), np.int32), act_cell=np.zeros((Q, M, KK), np.int32),
                 act_w=np.zeros((Q, M, KK), np.int32), retrieved=np.zeros((Q, M), np.int64),
                 V=np.zeros((Q, N), np.uint16), cand_n=np.zeros(Q, np.int64), cand=np.zeros((Q, N), np.int32),
                 order=np.zeros((Q, N), np.int32), n_verified=np.zeros(Q, np.int64),
                 fallback=np.zeros(Q, np.int32), qrot=np.zeros((Q, ix["Dp"]), np.float32))
    T = (lambda key: _p(t[key])) if t is not None else (lambda key: None)
    patience = patience_factor * k if patience_factor > 0 else 0
    gsize = np.ascontiguousarray(ix["gsize"], dtype=np.int64)
    ec = np.ascontiguousarray(ext_cand, dtype=np.int32) if ext_cand is not None else None
    en = np.ascontiguousarray(ext_n, dtype=np.int64) if ext_n is not None else None
    lib().or_search(N, ix["gid_base"], ix["Dp"], M, K, ix["dh"], _p(_hoff(ix.get("hoff"))), _p(ix["X"]),
                    _p(ix["R"]) if ix["R"] is not None else None, _p(ix["cb"]), _p(ix["off"]), _p(ix["ids"]),
                    _p(ix["codes"]), _p(gsize), budget, tau, patience, 1 if adsampling else 0, eps0, ad_stride,
                    0 if fallback else 1, _p(ec), _p(en),
                    _p(qp), Q, k, mode, nthreads, _p(out_ids), _p(out_d),
                    T("act_len"), T("act_cell"), T("act_w"), T("retrieved"), T("V"), T("cand_n"), T("cand"),
                    T("order"), T("n_verified"), T("fallback"), T("qrot"))
    return out_ids, out_d, t
