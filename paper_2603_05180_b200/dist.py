"""Point-sharded multi-GPU search: one process per GPU.

Collective call sites:
  N0     all-gathers of each rank's rows of the CEV and k-means samples (fixed
         global ids of the counter-based sampler) to rank 0, which builds the
         model (crisp_build_model: the R and codebooks of a build over all rows)
  N1/N2  broadcast of R and the codebooks from rank 0 (shared by every shard)
  N3     all-reduce (sum) of the local cell sizes -> global sizes, so every
         shard's budget walk activates exactly the cells a single index would
  N5     all-reduce (sum) of the local |C_q| (exact global fallback)
  N6     all-gather of the V histograms (used by underflowing queries only)
  N7     one all-gather of the per-shard top-k (dist64, gid) packed together,
         then the a6 merge kernel (crisp_merge_topk) by (d, gid)
  N8     (Optimized Mode, search_step_global) all-gather of the per-shard Hamming
         histograms, then per verification round all-gathers of the entries that
         may improve a top-k: the patience rule runs over the GLOBAL (h, gid)
         order, so the result equals a single index for every G
  N9     all-gather of q' (sharded_transform): each rank runs a0 on its slice of
         the batch only

The orchestration is written against a small engine interface so the same
code runs with the CUDA engine (NCCL over NVLink) and, in the CPU tests, with
a test-supplied engine over gloo.  torch.distributed is plumbing only.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


class CudaEngine:
    """Engine over libcrisp.so for one rank (device tensors)."""

    def __init__(self, crisp, device):
        self.crisp = crisp
        self.device = device
        self.index = None

    def build_model(self, cev_rows, km_rows, M, **params):
        """crisp_build_model on this rank (rank 0) from the gathered sample rows."""
        R, cb, _ = self.crisp.build_model(cev_rows, km_rows, M, **params)
        return (torch.from_numpy(R) if R is not None else None), torch.from_numpy(cb)

    def sample_ids(self, N_global, seed, kmeans_sample=100000):
        cev_ids, km_ids = self.crisp.model_samples(N_global, seed, kmeans_sample)
        return torch.from_numpy(cev_ids.astype(np.int64)), torch.from_numpy(km_ids.astype(np.int64))

    def build_shard(self, X_shard, gid_base, M, R, codebooks, **params):
        R = R.cpu().numpy() if R is not None else None
        self.index = self.crisp.Index.build(X_shard, M, R=R, codebooks=codebooks.cpu().numpy(), gid_base=gid_base,
                                            **params)

    def local_cell_sizes(self):
        return torch.from_numpy(self.index.local_cell_sizes())

    def set_global_cell_sizes(self, sizes):
        self.index.set_global_cell_sizes(sizes.cpu().numpy())

    def set_search_params(self, **kw):
        self.index.set_search_params(**kw)

    def search_shard(self, q_dev, k, mode, stream=0):
        Q = q_dev.shape[0]
        ids = torch.empty((Q, k), dtype=torch.int64, device=q_dev.device)
        d64 = torch.empty((Q, k), dtype=torch.float64, device=q_dev.device)
        self.index.search_shard_async(q_dev, k, mode, ids, d64, stream)
        return ids, d64

    # a0 alone (crisp_transform_queries_async): q' of a slice of the batch, rows of pitch floats
    def transform(self, q_dev, stream=0):
        pitch = self.index.info()["pitch"]
        out = torch.empty((q_dev.shape[0], pitch), dtype=torch.float32, device=q_dev.device)
        if q_dev.shape[0]:
            self.index.transform_queries(q_dev.contiguous(), out, stream)
        return out

    def begin_transformed(self, qrot, k, mode, stream=0):
        counts = torch.empty(qrot.shape[0], dtype=torch.int32, device=qrot.device)
        self._ss = self.index.shard_begin_transformed(qrot, k, mode, counts, stream)
        self._Q, self._k = qrot.shape[0], k
        return counts

    # phased shard search (exact global fallback), see include/crisp.h
    def begin(self, q_dev, k, mode, stream=0):
        counts = torch.empty(q_dev.shape[0], dtype=torch.int32, device=q_dev.device)
        self._ss = self.index.shard_begin(q_dev, k, mode, counts, stream)
        self._Q, self._k = q_dev.shape[0], k
        return counts

    def hist(self, global_counts, stream=0):
        M = self.index.info()["M"]
        h = torch.zeros((self._Q, 2 * M + 2), dtype=torch.int32, device=global_counts.device)
        self.index.shard_hist(self._ss, global_counts, h, stream)
        return h

    def finish(self, global_counts, all_hist, G, rank, stream=0):
        ids = torch.empty((self._Q, self._k), dtype=torch.int64, device=global_counts.device)
        d64 = torch.empty((self._Q, self._k), dtype=torch.float64, device=global_counts.device)
        self.index.shard_finish(self._ss, global_counts, all_hist, G, rank, ids, d64, stream)
        self.index.shard_free(self._ss)
        self._ss = None
        return ids, d64

    # exact global patience (phi=1), see include/crisp.h crisp_shard_gp_*
    def gp_order(self, global_counts, all_hist, G, rank, stream=0):
        H = self.index.info()["padded_D"] + 1
        hh = torch.zeros((self._Q, H), dtype=torch.int32, device=global_counts.device)
        self.index.gp_order(self._ss, global_counts, all_hist, G, rank, hh, stream)
        return hh

    def gp_prepare(self, all_hh, G, rank, gid_bases, stream=0):
        self.index.gp_prepare(self._ss, all_hh, G, rank, gid_bases, stream)

    def gp_round(self, stream=0):
        return self.index.gp_round(self._ss, stream)

    def gp_fetch(self, n_pad, stream=0):
        dev = torch.device("cuda", torch.cuda.current_device())
        ent = torch.zeros((max(1, n_pad), 16), dtype=torch.uint8, device=dev)
        cnt = torch.empty(self._Q, dtype=torch.int32, device=dev)
        self.index.gp_fetch(self._ss, ent, cnt, stream)
        return ent, cnt

    def gp_replay(self, all_counts, all_entries, stride, G, stream=0):
        return self.index.gp_replay(self._ss, all_counts, all_entries, stride, G, stream)

    def gp_result(self, stream=0):
        dev = torch.device("cuda", torch.cuda.current_device())
        ids = torch.empty((self._Q, self._k), dtype=torch.int64, device=dev)
        d64 = torch.empty((self._Q, self._k), dtype=torch.float64, device=dev)
        self.index.gp_result(self._ss, ids, d64, stream)
        self.index.shard_free(self._ss)
        self._ss = None
        return ids, d64

    def merge(self, d64_all, ids_all, stream=0):
        G, Q, k = d64_all.shape
        od64 = torch.empty((Q, k), dtype=torch.float64, device=d64_all.device)
        od = torch.empty((Q, k), dtype=torch.float32, device=d64_all.device)
        oi = torch.empty((Q, k), dtype=torch.int64, device=d64_all.device)
        self.crisp.merge_topk(d64_all, ids_all, od64, od, oi, stream)
        return oi, od


def shard_range(N: int, rank: int, world: int):
    """Contiguous global id ranges [g*N/G, (g+1)*N/G)."""
    lo = (N * rank) // world
    hi = (N * (rank + 1)) // world
    return lo, hi


def share_model(R, codebooks, like, src=0):
    """N1/N2: broadcast R (or 'no rotation') and the codebooks from rank src."""
    flag = torch.tensor([1 if R is not None else 0], dtype=torch.int64, device=like.device)
    dist.broadcast(flag, src)
    cb = codebooks.to(like.device) if codebooks is not None else None
    shape = torch.tensor(list(cb.shape) if cb is not None else [0, 0, 0, 0], dtype=torch.int64, device=like.device)
    dist.broadcast(shape, src)
    if cb is None:
        cb = torch.empty(tuple(shape.tolist()), dtype=torch.float32, device=like.device)
    dist.broadcast(cb, src)
    Rt = None
    if int(flag.item()):
        Dp = int(shape[0] * 2 * shape[3])  # padded_D = M * 2 * dh
        Rt = R.to(like.device) if R is not None else torch.empty((Dp, Dp), dtype=torch.float32, device=like.device)
        dist.broadcast(Rt, src)
    return Rt, cb


def gather_sample_rows(X_local, lo, ids, dst=0):
    """Rows `ids` (ascending global ids) of the point-sharded dataset, gathered on
    rank dst in ascending global id: each rank contributes its rows in [lo,
    lo + len(X_local)) (a padded all-gather; shards are contiguous id ranges in
    rank order, so concatenating by rank keeps the order).  Returns the (n, D)
    tensor on rank dst, None elsewhere."""
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = _coll_device()
    ids = torch.as_tensor(ids, dtype=torch.int64)
    hi = lo + X_local.shape[0]
    mine = ids[(ids >= lo) & (ids < hi)] - lo
    rows = X_local[mine.to(X_local.device)].to(dev).contiguous()
    cnt = torch.tensor([rows.shape[0]], dtype=torch.int64, device=dev)
    cnts = [torch.empty_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt)
    mx = int(max(int(c.item()) for c in cnts))
    D = X_local.shape[1]
    pad = torch.zeros((mx, D), dtype=rows.dtype, device=dev)
    pad[: rows.shape[0]] = rows
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad)
    if rank != dst:
        return None
    return torch.cat([o[: int(c.item())] for o, c in zip(outs, cnts)])


def model_from_shards(engine, X_local, lo, N_global, M, seed, kmeans_sample=100000, **params):
    """N1/N2 without a full index on one rank: every rank contributes its rows of
    the CEV and k-means samples (fixed global row ids, counter-based sampling),
    rank 0 builds the model (R, codebooks) from them (crisp_build_model), and the
    model is broadcast (share_model).  Identical to a single build over all rows."""
    cev_ids, km_ids = engine.sample_ids(N_global, seed, kmeans_sample)
    cev_rows = gather_sample_rows(X_local, lo, cev_ids)
    km_rows = gather_sample_rows(X_local, lo, km_ids)
    R = cb = None
    if dist.get_rank() == 0:
        R, cb = engine.build_model(cev_rows.cpu().numpy(), km_rows.cpu().numpy(), M, seed=seed,
                                   kmeans_sample=kmeans_sample, **params)
    return share_model(R, cb, torch.empty(0, device=_coll_device()))


def global_cell_sizes(engine):
    """N3: sum of the local cell-size tables."""
    s = engine.local_cell_sizes()
    dev = _coll_device()
    t = s.to(dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    engine.set_global_cell_sizes(t)
    return t


def gather_topk(ids, d64):
    """N7 as ONE all-gather: the per-shard (dist64, gid) lists packed as a
    (2, Q, k) int64 tensor (the fp64 distances travel as their bit patterns,
    unchanged), unpacked into (G, Q, k) fp64 and int64 for the a6 merge."""
    world = dist.get_world_size()
    packed = torch.stack((d64.view(torch.int64), ids))
    out = [torch.empty_like(packed) for _ in range(world)]
    dist.all_gather(out, packed)
    allp = torch.stack(out)
    return allp[:, 0].contiguous().view(torch.float64), allp[:, 1].contiguous()


def search_step(engine, q_dev, k, mode, stream=0):
    """One sharded search of the batch: local a0..a5, then N7 + a6."""
    ids, d64 = engine.search_shard(q_dev, k, mode, stream)
    gd, gi = gather_topk(ids, d64)
    return engine.merge(gd, gi, stream)


def sharded_transform(engine, q_dev, stream=0):
    """a0 sharded by query (N9): rank r transforms rows [r P, (r+1) P) of the batch (P =
    ceil(Q/G)) and one all-gather assembles q' for every rank, instead of every rank
    transforming every query; q' is bit-exact either way, so the results are unchanged."""
    world, rank = dist.get_world_size(), dist.get_rank()
    Q = q_dev.shape[0]
    per = (Q + world - 1) // world
    lo, hi = min(Q, rank * per), min(Q, (rank + 1) * per)
    part = engine.transform(q_dev[lo:hi], stream)
    pad = torch.zeros((per, part.shape[1]), dtype=part.dtype, device=part.device)
    pad[: hi - lo] = part
    out = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(out, pad)
    return torch.cat(out)[:Q].contiguous()


def _begin(engine, q_dev, k, mode, stream=0):
    """The phased search's first phase: with G > 1 and an engine that supports it, on q'
    transformed once across the ranks (sharded_transform; CRISP_SHARD_A0=0 keeps every
    rank transforming the whole batch)."""
    import os

    if (dist.get_world_size() > 1 and hasattr(engine, "begin_transformed")
            and os.environ.get("CRISP_SHARD_A0", "1") != "0"):
        return engine.begin_transformed(sharded_transform(engine, q_dev, stream), k, mode, stream)
    return engine.begin(q_dev, k, mode, stream)


def search_step_exact(engine, q_dev, k, mode, stream=0):
    """One sharded search with the EXACT global underflow fallback: N5
    all-reduce of |C_q|, all-gather of the V histograms of underflowing
    queries, then a5 on each shard and N7 + a6.  For phi=0 the result equals
    the single index for every G."""
    world, rank = dist.get_world_size(), dist.get_rank()
    counts = _begin(engine, q_dev, k, mode, stream)
    dist.all_reduce(counts, op=dist.ReduceOp.SUM)
    hist = engine.hist(counts, stream)
    all_h = [torch.empty_like(hist) for _ in range(world)]
    dist.all_gather(all_h, hist)
    ids, d64 = engine.finish(counts, torch.stack(all_h), world, rank, stream)
    gd, gi = gather_topk(ids, d64)
    return engine.merge(gd, gi, stream)


def _all_gather_stack(t):
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return torch.stack(out)


def search_step_global(engine, q_dev, k, mode, gid_bases, stream=0):
    """One sharded search whose Optimized-Mode verification follows the
    patience rule over the GLOBAL (h, gid) order (exact for every G: the result
    equals a single index over all rows).  Collectives per step: N5 all-reduce
    of |C_q|, N6 all-gather of the V histograms (exact fallback), N8 all-gather
    of the Hamming histograms, then per verification round one all-gather of
    the entry counts and one of the entries that may improve a top-k (their
    number first, for the padded size).  Guaranteed Mode is search_step_exact."""
    if mode != 1:
        return search_step_exact(engine, q_dev, k, mode, stream)
    world, rank = dist.get_world_size(), dist.get_rank()
    counts = _begin(engine, q_dev, k, mode, stream)
    dist.all_reduce(counts, op=dist.ReduceOp.SUM)
    hist = engine.hist(counts, stream)
    hh = engine.gp_order(counts, _all_gather_stack(hist), world, rank, stream)
    engine.gp_prepare(_all_gather_stack(hh), world, rank, gid_bases, stream)
    dev = counts.device
    while True:
        n = engine.gp_round(stream)
        ns = _all_gather_stack(torch.tensor([n], dtype=torch.int64, device=dev))
        stride = max(1, int(ns.max().item()))
        ent, cnt = engine.gp_fetch(stride, stream)
        running = engine.gp_replay(_all_gather_stack(cnt), _all_gather_stack(ent), stride, world, stream)
        if running == 0:
            break
    ids, d64 = engine.gp_result(stream)
    return ids, d64.to(torch.float32)


def emulate_global_search(engines, gid_bases, q_dev, k, mode, stream=0, stats=None, sharded_a0=False):
    """The search_step_global protocol for G shard engines in ONE process (the
    collectives done by concatenation): a single-GPU emulation for the tests.
    sharded_a0: each engine transforms its slice of the batch (N9) and every
    engine begins on the concatenated q'."""
    G = len(engines)
    if sharded_a0:
        Q = q_dev.shape[0]
        per = (Q + G - 1) // G
        qrot = torch.cat([e.transform(q_dev[min(Q, r * per):min(Q, (r + 1) * per)], stream)
                          for r, e in enumerate(engines)]).contiguous()
        counts = [e.begin_transformed(qrot, k, mode, stream) for e in engines]
    else:
        counts = [e.begin(q_dev, k, mode, stream) for e in engines]
    gc = torch.stack(counts).sum(0).to(torch.int32)
    hists = torch.stack([e.hist(gc, stream) for e in engines])
    if mode != 1:
        outs = [e.finish(gc, hists, G, r, stream) for r, e in enumerate(engines)]
        ids, d64 = torch.stack([o[0] for o in outs]), torch.stack([o[1] for o in outs])
        return engines[0].merge(d64, ids, stream)
    hh = torch.stack([e.gp_order(gc, hists, G, r, stream) for r, e in enumerate(engines)])
    for r, e in enumerate(engines):
        e.gp_prepare(hh, G, r, gid_bases, stream)
    rounds = 0
    while True:
        ns = [e.gp_round(stream) for e in engines]
        stride = max(1, max(ns))
        got = [e.gp_fetch(stride, stream) for e in engines]
        all_ent = torch.stack([g_[0] for g_ in got])
        all_cnt = torch.stack([g_[1] for g_ in got])
        running = [e.gp_replay(all_cnt, all_ent, stride, G, stream) for e in engines]
        assert len(set(running)) == 1, "replicated replay diverged"
        rounds += 1
        if running[0] == 0:
            break
    if stats is not None:
        stats["rounds"] = rounds
    res = [e.gp_result(stream) for e in engines]
    for r in range(1, G):
        assert torch.equal(res[r][0], res[0][0]) and torch.equal(res[r][1], res[0][1]), "ranks disagree"
    return res[0][0], res[0][1].to(torch.float32)


def _coll_device():
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
