"""paper_2603_05180_b200 -- B200-native CRISP query engine (arXiv 2603.05180).

Thin ctypes binding over the C ABI of ``libcrisp.so`` (include/crisp.h).  This
module only marshals arguments: every step of build and search runs in the
CUDA kernels of ``csrc/``.  There is no CPU fallback: if the shared library is
missing or no CUDA device is present, calls raise ``CrispError``.

Host inputs may be numpy arrays; device inputs may be torch CUDA tensors
(only their data pointers are used).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CRISP_LIB") or os.path.join(_HERE, "libcrisp.so")  # CRISP_LIB: an A/B build variant

GUARANTEED, OPTIMIZED = 0, 1
STAGES = ("transform", "probe", "count_select", "fallback", "verify", "merge", "hamming", "hsort")


class CrispError(RuntimeError):
    pass


class Params(C.Structure):
    _fields_ = [
        ("M", C.c_int32), ("K", C.c_int32), ("tau_cev", C.c_float), ("rotation", C.c_int32),
        ("kmeans_iters", C.c_int32), ("kmeans_sample", C.c_int64), ("seed", C.c_uint64), ("device", C.c_int32),
        ("budget_ratio", C.c_double), ("budget", C.c_int64), ("min_collision_ratio", C.c_double), ("tau", C.c_int32),
        ("patience_factor", C.c_int32), ("workspace_bytes", C.c_int64), ("rotation_block", C.c_int32),
        ("adaptive_subspaces", C.c_int32), ("subspace_widths", C.c_void_p),
    ]


class Info(C.Structure):
    _fields_ = [
        ("N", C.c_int64), ("N_global", C.c_int64), ("gid_base", C.c_int64), ("D", C.c_int32),
        ("padded_D", C.c_int32), ("pitch", C.c_int32), ("M", C.c_int32), ("K", C.c_int32), ("dh", C.c_int32),
        ("rotated", C.c_int32), ("cev", C.c_double), ("budget", C.c_int64), ("tau", C.c_int32),
        ("patience_factor", C.c_int32), ("block_ids", C.c_int32), ("n_blocks", C.c_int32), ("hbm_bytes", C.c_int64),
        ("logical_bytes", C.c_int64), ("slice_hint", C.c_double), ("rotation_block", C.c_int32),
        ("adaptive", C.c_int32),
    ]


class Export(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("R", "X", "codebooks", "cells", "offsets", "ids", "codes", "cell_sizes",
                                          "subspace_widths")]


class Trace(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("act_len", "act_cell", "act_w", "retrieved", "V", "cand_n", "cand", "order",
                                          "n_verified", "fallback", "qrot")]


# Every symbol include/crisp.h declares (checked by tests/test_abi.py).
ABI_SYMBOLS = (
    "crisp_default_params", "crisp_build", "crisp_build_with", "crisp_build_shard", "crisp_local_cell_sizes",
    "crisp_set_global_cell_sizes", "crisp_set_search_params", "crisp_index_info", "crisp_search",
    "crisp_search_async", "crisp_search_shard_async", "crisp_merge_topk", "crisp_search_trace", "crisp_export",
    "crisp_set_stage_timing", "crisp_stage_times", "crisp_search_counters", "crisp_free", "crisp_last_error", "crisp_version",
    "crisp_shard_search_begin", "crisp_shard_search_hist", "crisp_shard_search_finish", "crisp_shard_search_free",
    "crisp_transform_queries_async", "crisp_shard_search_begin_transformed",
    "crisp_shard_gp_order", "crisp_shard_gp_prepare", "crisp_shard_gp_round", "crisp_shard_gp_fetch",
    "crisp_shard_gp_replay", "crisp_shard_gp_result",
    "crisp_set_adsampling", "crisp_set_verify_filter", "crisp_exact_ceil", "crisp_cev_sample_size", "crisp_sample_rows", "crisp_build_model",
)

_lib = None


def lib():
    """Load libcrisp.so (fails loudly when the CUDA extension is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CrispError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        P = C.POINTER
        L.crisp_default_params.argtypes = [P(Params)]
        L.crisp_build.argtypes = [vp, i64, i32, P(Params), P(vp)]
        L.crisp_build_with.argtypes = [vp, i64, i32, P(Params), vp, vp, P(vp)]
        L.crisp_build_shard.argtypes = [vp, i64, i64, i32, P(Params), vp, vp, P(vp)]
        L.crisp_local_cell_sizes.argtypes = [vp, vp]
        L.crisp_set_adsampling.argtypes = [vp, i32, f64, i32]
        L.crisp_set_verify_filter.argtypes = [vp, i32]
        L.crisp_set_global_cell_sizes.argtypes = [vp, vp]
        L.crisp_set_search_params.argtypes = [vp, f64, i64, f64, i32, i32]
        L.crisp_index_info.argtypes = [vp, P(Info)]
        L.crisp_search.argtypes = [vp, vp, i64, i32, i32, vp, vp]
        L.crisp_search_async.argtypes = [vp, vp, i64, i32, i32, vp, vp, vp]
        L.crisp_search_shard_async.argtypes = [vp, vp, i64, i32, i32, vp, vp, vp]
        L.crisp_merge_topk.argtypes = [vp, vp, i32, i64, i32, vp, vp, vp, vp]
        L.crisp_search_trace.argtypes = [vp, vp, i64, i32, i32, vp, vp, P(Trace)]
        L.crisp_export.argtypes = [vp, P(Export)]
        L.crisp_set_stage_timing.argtypes = [i32]
        L.crisp_stage_times.argtypes = [vp, i32, i32]
        L.crisp_search_counters.argtypes = [vp, i32, i32]
        L.crisp_shard_search_begin.argtypes = [vp, vp, i64, i32, i32, vp, P(vp), vp]
        L.crisp_shard_search_begin_transformed.argtypes = [vp, vp, i64, i32, i32, vp, P(vp), vp]
        L.crisp_transform_queries_async.argtypes = [vp, vp, i64, vp, vp]
        L.crisp_shard_search_hist.argtypes = [vp, vp, vp, vp]
        L.crisp_shard_search_finish.argtypes = [vp, vp, vp, i32, i32, vp, vp, vp]
        L.crisp_shard_gp_order.argtypes = [vp, vp, vp, i32, i32, vp, vp]
        L.crisp_shard_gp_prepare.argtypes = [vp, vp, i32, i32, vp, vp]
        L.crisp_shard_gp_round.argtypes = [vp, P(i64), vp]
        L.crisp_shard_gp_fetch.argtypes = [vp, vp, vp, vp]
        L.crisp_shard_gp_replay.argtypes = [vp, vp, vp, i64, i32, P(i32), vp]
        L.crisp_shard_gp_result.argtypes = [vp, vp, vp, vp]
        L.crisp_shard_search_free.argtypes = [vp]
        L.crisp_shard_search_free.restype = None
        L.crisp_free.argtypes = [vp]
        L.crisp_free.restype = None
        L.crisp_last_error.restype = C.c_char_p
        L.crisp_version.restype = C.c_char_p
        L.crisp_exact_ceil.argtypes = [f64, i64]
        L.crisp_exact_ceil.restype = i64
        L.crisp_cev_sample_size.argtypes = [i64]
        L.crisp_cev_sample_size.restype = i64
        L.crisp_sample_rows.argtypes = [i64, i64, C.c_uint64, C.c_uint32, vp]
        L.crisp_build_model.argtypes = [vp, i64, vp, i64, i32, vp, vp, vp, vp, vp]
        _lib = L
    return _lib


def _check(st: int):
    if st != 0:
        raise CrispError(f"crisp status {st}: {lib().crisp_last_error().decode()}")


def _ptr(a):
    """Data pointer of a numpy array or torch tensor (no copies)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


_TORCH_DT = {np.float32: "float32", np.int64: "int64", np.float64: "float64", np.int32: "int32"}


def _host(a, dtype, ndim=2):  # ndim None: any rank
    """numpy: a C-contiguous copy/view of the given dtype.  torch: the tensor
    itself after checking that the library can read it as packed row-major
    `dtype` (the C ABI takes raw pointers, so a wrong dtype, a strided view or
    a wrong rank would be misread)."""
    if hasattr(a, "data_ptr"):
        want = _TORCH_DT[dtype]
        if str(a.dtype) != "torch." + want:
            raise CrispError(f"tensor dtype {a.dtype}, expected torch.{want}")
        if not a.is_contiguous():
            raise CrispError("tensor must be contiguous (row-major)")
        if ndim is not None and a.dim() != ndim:
            raise CrispError(f"tensor must have {ndim} dimensions, got {a.dim()}")
        return a
    return np.ascontiguousarray(a, dtype=dtype)


def exact_ceil(ratio, n: int) -> int:
    """crisp_exact_ceil: ceil(ratio*n) with ratio read as the shortest decimal
    that rounds to it (the library's rule for B and tau)."""
    return int(lib().crisp_exact_ceil(float(ratio), int(n)))


STREAM_CEV_SAMPLE, STREAM_KM_SAMPLE = 1, 3  # the build's Philox streams (DESIGN R3)


def sample_rows(N: int, n: int, seed: int, stream: int) -> np.ndarray:
    """crisp_sample_rows: the n sampled global row ids (ascending) of a dataset of N rows."""
    out = np.zeros(max(n, 1), np.int32)
    _check(lib().crisp_sample_rows(int(N), int(n), int(seed), int(stream), _ptr(out)))
    return out[:n]


def model_samples(N: int, seed: int, kmeans_sample: int = 100000):
    """(CEV sample row ids, k-means sample row ids) of a dataset of N rows."""
    n_cev = int(lib().crisp_cev_sample_size(int(N)))
    n_km = min(int(N), max(1, int(kmeans_sample)))
    return sample_rows(N, n_cev, seed, STREAM_CEV_SAMPLE), sample_rows(N, n_km, seed, STREAM_KM_SAMPLE)


def build_model(cev_rows, km_rows, M: int, **params):
    """crisp_build_model: (R or None, codebooks, cev) from the gathered sample rows."""
    p = default_params(M=M, **params)
    cr = _host(cev_rows, np.float32)
    kr = _host(km_rows, np.float32)
    D = int(kr.shape[1])
    Dp = ((D + 2 * M - 1) // (2 * M)) * (2 * M)
    R = np.zeros((Dp, Dp), np.float32)
    cb = np.zeros((M, 2, p.K, Dp // (2 * M)), np.float32)
    rot = C.c_int32(0)
    cev = C.c_double(0.0)
    _check(lib().crisp_build_model(_ptr(cr), int(cr.shape[0]), _ptr(kr), int(kr.shape[0]), D, C.byref(p), _ptr(R),
                                   _ptr(cb), C.byref(rot), C.byref(cev)))
    return (R if rot.value else None), cb, cev.value


def _dev(t, dtype, shape=None, what="tensor"):
    """A device tensor handed to a *_async call: CUDA, dtype, contiguous, shape."""
    if not hasattr(t, "data_ptr") or not t.is_cuda:
        raise CrispError(f"{what} must be a CUDA tensor")
    _host(t, dtype, None if shape is None else len(shape))
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise CrispError(f"{what} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    return t


def default_params(**kw) -> Params:
    p = Params()
    _check(lib().crisp_default_params(C.byref(p)))
    for k, v in kw.items():
        if not hasattr(p, k):
            raise TypeError(f"unknown parameter {k}")
        setattr(p, k, v)
    return p


@dataclass
class SearchKnobs:
    beta: float | None = None
    budget: int | None = None
    alpha: float | None = None
    tau: int | None = None
    patience_factor: int = 40


class Index:
    """An index in HBM (crisp_index*)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    # ---------------------------------------------------------------- build
    @staticmethod
    def build(data, M: int, R=None, codebooks=None, gid_base: int | None = None, **params) -> "Index":
        """crisp_build (or crisp_build_with when R/codebooks are given, or
        crisp_build_shard when gid_base is given).  subspace_widths: M even
        widths summing to the padded dimensionality (R18), or None."""
        widths = params.pop("subspace_widths", None)
        p = default_params(M=M, **params)
        if widths is not None:
            wv = np.ascontiguousarray(widths, dtype=np.int32)
            if wv.shape != (M,):
                raise CrispError(f"subspace_widths must hold M={M} widths")
            p.subspace_widths = wv.ctypes.data  # wv stays alive for the call
        x = _host(data, np.float32)
        N, D = int(x.shape[0]), int(x.shape[1])
        out = C.c_void_p()
        if gid_base is not None:
            Rh = _host(R, np.float32) if R is not None else None
            cbh = _host(codebooks, np.float32, None)
            _check(lib().crisp_build_shard(_ptr(x), N, gid_base, D, C.byref(p), _ptr(Rh), _ptr(cbh), C.byref(out)))
        elif R is not None or codebooks is not None:
            Rh = _host(R, np.float32) if R is not None else None
            cbh = _host(codebooks, np.float32, None)
            _check(lib().crisp_build_with(_ptr(x), N, D, C.byref(p), _ptr(Rh), _ptr(cbh), C.byref(out)))
        else:
            _check(lib().crisp_build(_ptr(x), N, D, C.byref(p), C.byref(out)))
        return Index(out.value)

    def free(self):
        if self._h and self._h.value:
            lib().crisp_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    # ---------------------------------------------------------------- knobs
    def info(self) -> dict:
        i = Info()
        _check(lib().crisp_index_info(self._h, C.byref(i)))
        return {n: getattr(i, n) for n, _ in Info._fields_}

    def set_search_params(self, beta=None, budget=None, alpha=None, tau=None, patience_factor=40):
        """crisp_set_search_params: the library derives B = ceil(beta*N_global)
        and tau = ceil(alpha*M) from the ratios (decimal semantics, SURVEY 8(c)
        O1) unless the integers are given."""
        _check(lib().crisp_set_search_params(self._h, float(beta if beta is not None else 0.01), int(budget or 0),
                                             float(alpha if alpha is not None else 0.3), int(tau or 0),
                                             int(patience_factor)))

    def set_adsampling(self, enable: bool = True, eps0: float = 2.1, stride: int = 32):
        """crisp_set_adsampling: Optimized Mode verification by ADSampling (Eq. 2)."""
        _check(lib().crisp_set_adsampling(self._h, 1 if enable else 0, float(eps0), int(stride)))

    def set_verify_filter(self, enable: bool = True):
        """crisp_set_verify_filter: the certified int8 distance bound in front of the
        exact re-rank (results unchanged; DESIGN R17)."""
        _check(lib().crisp_set_verify_filter(self._h, 1 if enable else 0))

    def local_cell_sizes(self) -> np.ndarray:
        i = self.info()
        out = np.zeros((i["M"], i["K"] * i["K"]), np.int64)
        _check(lib().crisp_local_cell_sizes(self._h, _ptr(out)))
        return out

    def set_global_cell_sizes(self, sizes):
        s = np.ascontiguousarray(sizes, dtype=np.int64)
        _check(lib().crisp_set_global_cell_sizes(self._h, _ptr(s)))

    # ---------------------------------------------------------------- search
    def search(self, queries, k: int, mode: int = GUARANTEED):
        """crisp_search: host (numpy) or device (torch CUDA) queries.  Returns
        (ids int64 Qxk, dist2 float32 Qxk) on the same side as the input."""
        q = _host(queries, np.float32)
        Q = int(q.shape[0])
        if hasattr(q, "data_ptr"):
            import torch
            ids = torch.empty((Q, k), dtype=torch.int64, device=q.device)
            d = torch.empty((Q, k), dtype=torch.float32, device=q.device)
        else:
            ids = np.zeros((Q, k), np.int64)
            d = np.zeros((Q, k), np.float32)
        _check(lib().crisp_search(self._h, _ptr(q), Q, k, mode, _ptr(ids), _ptr(d)))
        return ids, d

    def search_async(self, q_dev, k: int, mode: int, ids_dev, d_dev, stream_ptr: int = 0):
        """crisp_search_async on device tensors; stream_ptr = torch stream.cuda_stream."""
        Q = int(q_dev.shape[0])
        _dev(q_dev, np.float32, None, "queries")
        _dev(ids_dev, np.int64, (Q, k), "ids")
        if d_dev is not None:
            _dev(d_dev, np.float32, (Q, k), "distances")
        _check(lib().crisp_search_async(self._h, _ptr(q_dev), int(q_dev.shape[0]), k, mode, _ptr(ids_dev),
                                        _ptr(d_dev), C.c_void_p(stream_ptr)))

    def search_shard_async(self, q_dev, k: int, mode: int, ids_dev, d64_dev, stream_ptr: int = 0):
        Q = int(q_dev.shape[0])
        _dev(q_dev, np.float32, None, "queries")
        _dev(ids_dev, np.int64, (Q, k), "ids")
        _dev(d64_dev, np.float64, (Q, k), "distances")
        _check(lib().crisp_search_shard_async(self._h, _ptr(q_dev), int(q_dev.shape[0]), k, mode, _ptr(ids_dev),
                                              _ptr(d64_dev), C.c_void_p(stream_ptr)))

    # ------------------------------------------------- phased shard search
    def shard_begin(self, q_dev, k: int, mode: int, local_counts_dev, stream_ptr: int = 0):
        """crisp_shard_search_begin -> session handle (see include/crisp.h)."""
        ss = C.c_void_p()
        _check(lib().crisp_shard_search_begin(self._h, _ptr(q_dev), int(q_dev.shape[0]), k, mode,
                                              _ptr(local_counts_dev), C.byref(ss), C.c_void_p(stream_ptr)))
        return ss

    def transform_queries(self, q_dev, qrot_dev, stream_ptr: int = 0):
        """crisp_transform_queries_async: qrot (Q x pitch) = a0 of q (Q x D), device tensors."""
        q_dev = _host(q_dev, np.float32)
        _check(lib().crisp_transform_queries_async(self._h, _ptr(q_dev), int(q_dev.shape[0]), _ptr(qrot_dev),
                                                   C.c_void_p(stream_ptr)))

    def shard_begin_transformed(self, qrot_dev, k: int, mode: int, local_counts_dev, stream_ptr: int = 0):
        """crisp_shard_search_begin_transformed: crisp_shard_search_begin on q' (Q x pitch)."""
        ss = C.c_void_p()
        _check(lib().crisp_shard_search_begin_transformed(self._h, _ptr(qrot_dev), int(qrot_dev.shape[0]), k, mode,
                                                          _ptr(local_counts_dev), C.byref(ss),
                                                          C.c_void_p(stream_ptr)))
        return ss

    @staticmethod
    def shard_hist(ss, global_counts_dev, local_hist_dev, stream_ptr: int = 0):
        _check(lib().crisp_shard_search_hist(ss, _ptr(global_counts_dev), _ptr(local_hist_dev),
                                             C.c_void_p(stream_ptr)))

    @staticmethod
    def shard_finish(ss, global_counts_dev, all_hist_dev, G: int, rank: int, ids_dev, d64_dev, stream_ptr: int = 0):
        _check(lib().crisp_shard_search_finish(ss, _ptr(global_counts_dev), _ptr(all_hist_dev), G, rank,
                                               _ptr(ids_dev), _ptr(d64_dev), C.c_void_p(stream_ptr)))

    @staticmethod
    def shard_free(ss):
        lib().crisp_shard_search_free(ss)

    # exact global patience (Optimized Mode over G shards; include/crisp.h)
    @staticmethod
    def gp_order(ss, global_counts_dev, all_hist_dev, G: int, rank: int, local_hh_dev, stream_ptr: int = 0):
        _check(lib().crisp_shard_gp_order(ss, _ptr(global_counts_dev), _ptr(all_hist_dev), G, rank,
                                          _ptr(local_hh_dev), C.c_void_p(stream_ptr)))

    @staticmethod
    def gp_prepare(ss, all_hh_dev, G: int, rank: int, gid_bases, stream_ptr: int = 0):
        gb = np.ascontiguousarray(gid_bases, dtype=np.int64)
        _check(lib().crisp_shard_gp_prepare(ss, _ptr(all_hh_dev), G, rank, _ptr(gb), C.c_void_p(stream_ptr)))

    @staticmethod
    def gp_round(ss, stream_ptr: int = 0) -> int:
        n = C.c_int64(0)
        _check(lib().crisp_shard_gp_round(ss, C.byref(n), C.c_void_p(stream_ptr)))
        return int(n.value)

    @staticmethod
    def gp_fetch(ss, entries_dev, counts_dev, stream_ptr: int = 0):
        _check(lib().crisp_shard_gp_fetch(ss, _ptr(entries_dev), _ptr(counts_dev), C.c_void_p(stream_ptr)))

    @staticmethod
    def gp_replay(ss, all_counts_dev, all_entries_dev, stride: int, G: int, stream_ptr: int = 0) -> int:
        r = C.c_int32(0)
        _check(lib().crisp_shard_gp_replay(ss, _ptr(all_counts_dev), _ptr(all_entries_dev), int(stride), G,
                                           C.byref(r), C.c_void_p(stream_ptr)))
        return int(r.value)

    @staticmethod
    def gp_result(ss, ids_dev, d64_dev, stream_ptr: int = 0):
        _check(lib().crisp_shard_gp_result(ss, _ptr(ids_dev), _ptr(d64_dev), C.c_void_p(stream_ptr)))

    def trace(self, queries, k: int, mode: int = GUARANTEED):
        """crisp_search_trace: stage outputs as numpy arrays."""
        i = self.info()
        q = np.ascontiguousarray(queries, dtype=np.float32)
        Q, M, N, KK, Dp = q.shape[0], i["M"], i["N"], i["K"] ** 2, i["padded_D"]
        t = dict(act_len=np.zeros((Q, M), np.int32), act_cell=np.zeros((Q, M, KK), np.int32),
                 act_w=np.zeros((Q, M, KK), np.int32), retrieved=np.zeros((Q, M), np.int64),
                 V=np.zeros((Q, N), np.uint8), cand_n=np.zeros(Q, np.int64), cand=np.zeros((Q, N), np.int32),
                 order=np.zeros((Q, N), np.int32), n_verified=np.zeros(Q, np.int64), fallback=np.zeros(Q, np.int32),
                 qrot=np.zeros((Q, Dp), np.float32))
        tr = Trace(**{n: t[n].ctypes.data for n in t})
        ids = np.zeros((Q, k), np.int64)
        d = np.zeros((Q, k), np.float32)
        _check(lib().crisp_search_trace(self._h, _ptr(q), Q, k, mode, _ptr(ids), _ptr(d), C.byref(tr)))
        return ids, d, t

    def export(self) -> dict:
        i = self.info()
        N, M, K, Dp, dh = i["N"], i["M"], i["K"], i["padded_D"], i["dh"]
        W = (Dp + 63) // 64
        e = dict(X=np.zeros((N, Dp), np.float32), codebooks=np.zeros((M, 2, K, dh), np.float32),
                 cells=np.zeros((M, N), np.int32), offsets=np.zeros((M, K * K + 1), np.int64),
                 ids=np.zeros((M, N), np.int32), codes=np.zeros((N, W), np.uint64),
                 cell_sizes=np.zeros((M, K * K), np.int64), subspace_widths=np.zeros(M, np.int32))
        if i["rotated"]:
            e["R"] = np.zeros((Dp, Dp), np.float32)
        ex = Export(**{n: e[n].ctypes.data for n in e})
        _check(lib().crisp_export(self._h, C.byref(ex)))
        if not i["rotated"]:
            e["R"] = None
        return e


def merge_topk(d64_dev, ids_dev, out_d64, out_d, out_ids, stream_ptr: int = 0):
    """crisp_merge_topk over (G, Q, k) device tensors."""
    G, Q, k = d64_dev.shape
    _check(lib().crisp_merge_topk(_ptr(d64_dev), _ptr(ids_dev), G, Q, k, _ptr(out_d64), _ptr(out_d), _ptr(out_ids),
                                  C.c_void_p(stream_ptr)))


def set_stage_timing(on):
    """crisp_set_stage_timing: True / 1 stage events + work counters, 2 stage
    events only, False / 0 off."""
    _check(lib().crisp_set_stage_timing(int(on) if not isinstance(on, bool) else (1 if on else 0)))


def stage_times(reset: bool = True) -> dict:
    a = np.zeros(8, np.float64)
    _check(lib().crisp_stage_times(_ptr(a), 8, 1 if reset else 0))
    return {STAGES[i]: float(a[i]) for i in range(len(STAGES))}


def search_counters(reset: bool = True) -> dict:
    """Work counters of the searches run with stage timing on (crisp_search_counters)."""
    a = np.zeros(9, np.int64)
    _check(lib().crisp_search_counters(_ptr(a), 9, 1 if reset else 0))
    return dict(ids_streamed=int(a[0]), candidates=int(a[1]), verified=int(a[2]), fallback=int(a[3]),
                launches=int(a[4]), probe_exact_half_distances=int(a[5]), probe_screen_redone=int(a[6]),
                filter_rows=int(a[7]), filter_exact=int(a[8]))
