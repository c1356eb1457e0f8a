"""Multi-process (world_size 2, gloo, CPU) test of the point-sharded
orchestration in paper_2603_05180_b200/dist.py: R/codebook broadcast (N1/N2),
global cell sizes (N3), per-shard search + all-gather + merge (N7/a6).  The
engine here is a test-side wrapper over the CPU oracle (the CUDA engine needs
GPUs); the orchestration code under test is the same."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class OracleEngine:
    def __init__(self):
        self.ix = None
        self.B = self.tau = None

    def build_global(self, X, M, **kw):
        import oracle

        ix = oracle.build(X, M, K=kw.get("K", 6), rotation_mode=kw.get("rotation", 1), kmeans_iters=5, seed=3)
        R = torch.from_numpy(ix["R"]) if ix["R"] is not None else None
        return R, torch.from_numpy(ix["cb"])

    def build_shard(self, X_shard, gid_base, M, R, codebooks, **kw):
        import oracle

        self.ix = oracle.build(X_shard, M, K=codebooks.shape[2], R=None if R is None else R.numpy(),
                               codebooks=codebooks.numpy(), gid_base=gid_base)

    def local_cell_sizes(self):
        return torch.from_numpy(self.ix["gsize"].copy())

    def set_global_cell_sizes(self, sizes):
        self.ix["gsize"] = sizes.numpy().astype(np.int64)

    def set_search_params(self, budget, tau, patience_factor=0):
        self.B, self.tau, self._pf = budget, tau, patience_factor

    def search_shard(self, q, k, mode, stream=0):
        import oracle

        ids, d, _ = oracle.search(self.ix, q.numpy(), k, mode, self.B, self.tau, patience_factor=0)
        return torch.from_numpy(ids), torch.from_numpy(d)

    # a0 alone: the oracle engine's "q'" is the query itself (its search rotates internally),
    # so the query-sharded a0 of dist.sharded_transform is exercised for its slicing and the
    # all-gather that reassembles the batch
    def transform(self, q, stream=0):
        return q.clone()

    def begin_transformed(self, qrot, k, mode, stream=0):
        return self.begin(qrot, k, mode, stream)

    # phased protocol (exact global fallback), emulated on the oracle
    def begin(self, q, k, mode, stream=0):
        import oracle

        _, _, t = oracle.search(self.ix, q.numpy(), k, mode, self.B, self.tau, patience_factor=0, trace=True,
                                fallback=False)
        self._t, self._q, self._k, self._mode = t, q.numpy(), k, mode
        return torch.from_numpy(t["cand_n"].astype(np.int32))

    def hist(self, gcounts, stream=0):
        M, k = self.ix["M"], self._k
        h = np.zeros((len(gcounts), 2 * M + 2), np.int32)
        for q in range(len(gcounts)):
            if int(gcounts[q]) < k:
                h[q] = np.bincount(self._t["V"][q], minlength=2 * M + 2)[: 2 * M + 2]
                h[q, 0] = 0
        return torch.from_numpy(h)

    def finish(self, gcounts, all_hist, G, rank, stream=0):
        import oracle

        cand, n = self._cands(gcounts, all_hist, G, rank)
        ids, d, _ = oracle.search(self.ix, self._q, self._k, self._mode, self.B, self.tau, patience_factor=0,
                                  ext_cand=cand, ext_n=n)
        return torch.from_numpy(ids), torch.from_numpy(d)

    def _cands(self, gcounts, all_hist, G, rank):
        M, k, t = self.ix["M"], self._k, self._t
        N = self.ix["N"]
        Q = len(gcounts)
        cand = np.zeros((Q, N), np.int32)
        n = np.zeros(Q, np.int64)
        ah = all_hist.numpy()
        for q in range(Q):
            if int(gcounts[q]) >= k:
                c = t["cand"][q, : t["cand_n"][q]]
            else:  # global top-k touched by (V desc, gid asc); V* / quota from the summed histogram
                tot = ah[:, q].sum(0)
                acc, vstar, quota = 0, 1, int(tot[1])
                for v in range(2 * M, 0, -1):
                    if acc + tot[v] >= k:
                        vstar, quota = v, k - acc
                        break
                    acc += tot[v]
                share = max(0, min(int(ah[rank, q, vstar]), quota - int(ah[:rank, q, vstar].sum())))
                V = t["V"][q].astype(int)
                eq = np.nonzero(V == vstar)[0][:share]
                c = np.sort(np.concatenate([np.nonzero(V > vstar)[0], eq])).astype(np.int32)
            cand[q, : len(c)] = c
            n[q] = len(c)
        return cand, n

    # exact global patience (dist.search_step_global), emulated in numpy: the same
    # records and rule as the CUDA kernels (search.cu k_gp_*), on the oracle's index
    def gp_order(self, gcounts, all_hist, G, rank, stream=0):
        import oracle

        cand, n = self._cands(gcounts, all_hist, G, rank)
        Dp = self.ix["Dp"]
        qc = oracle.codes(self._t["qrot"][:, :Dp].astype(np.float32))
        self._qr = self._t["qrot"][:, :Dp].astype(np.float64)
        H = Dp + 1
        hh = np.zeros((len(n), H), np.int32)
        self._ord = []
        for q in range(len(n)):
            c = cand[q, : n[q]]
            x = np.bitwise_xor(self.ix["codes"][c], qc[q][None, :])
            h = np.array([sum(bin(int(w)).count("1") for w in row) for row in x], np.int64)
            o = np.lexsort((c, h))
            self._ord.append(c[o])
            hh[q] = np.bincount(h, minlength=H)[:H]
        return torch.from_numpy(hh)

    def gp_prepare(self, all_hh, G, rank, gid_bases, stream=0):
        ah = all_hh.numpy().astype(np.int64)
        tot, pre, mine = ah.sum(0), ah[:rank].sum(0), ah[rank]
        z = np.zeros((tot.shape[0], 1), np.int64)
        self._base = np.hstack([z, np.cumsum(tot, 1)])
        self._base[:, :-1] += pre
        self._lcum = np.hstack([z, np.cumsum(mine, 1)])
        self._gtot = tot.sum(1)
        self._gb = np.asarray(gid_bases, np.int64)
        Q = tot.shape[0]
        self._top = [[] for _ in range(Q)]  # sorted (d, gid)
        self._pat = np.zeros(Q, np.int64)
        self._done = np.zeros(Q, bool)
        self._gpos = np.zeros(Q, np.int64)
        self._glen = np.full(Q, 64, np.int64)

    def _loc(self, q, P):
        b, l = self._base[q], self._lcum[q]
        H = len(b) - 1
        if b[0] > P:
            return 0
        h = int(np.nonzero(b <= P)[0].max())
        mine = l[h + 1] - l[h] if h < H else 0
        return int(l[h] + min(max(P - b[h], 0), mine))

    def gp_round(self, stream=0):
        recs, cnt = [], []
        for q in range(len(self._done)):
            c = 0
            if not self._done[q]:
                P0, P1 = self._gpos[q], min(self._gpos[q] + self._glen[q], self._gtot[q])
                a, e = self._loc(q, P0), self._loc(q, P1)
                top = self._top[q]
                for i in range(a, e):
                    lid = int(self._ord[q][i])
                    d = float(((self._qr[q] - self.ix["X"][lid].astype(np.float64)) ** 2).sum())
                    gid = int(self.ix["gid_base"]) + lid
                    if len(top) < self._k or (d, gid) < top[-1]:
                        h = int(np.nonzero(self._lcum[q] <= i)[0].max())
                        recs.append((int(self._base[q][h] + i - self._lcum[q][h]), lid, d))
                        c += 1
            cnt.append(c)
        self._recs = np.array(recs, dtype=[("gpos", "<i4"), ("lid", "<i4"), ("d", "<f8")])
        self._cnt = np.array(cnt, np.int32)
        return len(recs)

    def gp_fetch(self, n_pad, stream=0):
        buf = np.zeros(max(1, n_pad) * 16, np.uint8)
        raw = self._recs.tobytes()
        buf[: len(raw)] = np.frombuffer(raw, np.uint8)
        return torch.from_numpy(buf.reshape(-1, 16)), torch.from_numpy(self._cnt)

    def gp_replay(self, all_counts, all_entries, stride, G, stream=0):
        ac = all_counts.numpy()
        ents = [np.frombuffer(all_entries[g].numpy().tobytes(), dtype=self._recs.dtype) for g in range(G)]
        offs = np.hstack([np.zeros((G, 1), np.int64), np.cumsum(ac, 1)])
        P, k, running = self._pf * self._k, self._k, 0
        for q in range(len(self._done)):
            if self._done[q]:
                continue
            lst = []
            for g in range(G):
                for r in ents[g][offs[g, q]: offs[g, q] + ac[g, q]]:
                    lst.append((int(r["gpos"]), int(self._gb[g]) + int(r["lid"]), float(r["d"])))
            lst.sort()
            P0, P1 = self._gpos[q], min(self._gpos[q] + self._glen[q], self._gtot[q])
            last, stop, pat, top = P0 - 1, -1, self._pat[q], self._top[q]
            for gp, gid, d in lst:
                gap = gp - last - 1
                if P > 0 and pat + gap >= P:
                    stop = last + (P - pat)
                    break
                pat += gap
                if len(top) < k or (d, gid) < top[-1]:
                    top.append((d, gid))
                    top.sort()
                    del top[k:]
                    pat = 0
                else:
                    pat += 1
                    if P > 0 and pat >= P:
                        stop = gp
                        break
                last = gp
            if stop < 0:
                gap = P1 - 1 - last
                if P > 0 and pat + gap >= P:
                    stop = last + (P - pat)
                else:
                    pat += gap
            self._pat[q] = pat
            if stop >= 0 or P1 >= self._gtot[q]:
                self._done[q] = True
            else:
                self._gpos[q] = P1
                self._glen[q] = min(4096, max(64, P - pat)) if P > 0 else 4096
                running += 1
        return running

    def gp_result(self, stream=0):
        k = self._k
        ids = np.full((len(self._top), k), -1, np.int64)
        d = np.full((len(self._top), k), np.inf)
        for q, top in enumerate(self._top):
            for i, (dd, gid) in enumerate(top):
                ids[q, i], d[q, i] = gid, dd
        return torch.from_numpy(ids), torch.from_numpy(d)

    def merge(self, d_all, ids_all, stream=0):
        import oracle

        d, i = oracle.merge_topk(d_all.numpy(), ids_all.numpy())
        return torch.from_numpy(i), torch.from_numpy(d.astype(np.float32))


def _data():
    r = np.random.default_rng(5)
    X = (r.standard_normal((3000, 24)) @ np.diag(np.linspace(3, 0.2, 24))).astype(np.float32)
    Q = (r.standard_normal((16, 24)) @ np.diag(np.linspace(3, 0.2, 24))).astype(np.float32)
    return X, Q


def _gp_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_05180_b200 import dist as cdist

        X, Q = _data()
        M, k, B, tau, P = 4, 5, 300, 3, 8
        eng = OracleEngine()
        R, cb = eng.build_global(X, M) if rank == 0 else (None, None)
        R, cb = cdist.share_model(R, cb, torch.zeros(1))
        lo, hi = cdist.shard_range(X.shape[0], rank, world)
        eng.build_shard(X[lo:hi], lo, M, R, cb)
        cdist.global_cell_sizes(eng)
        eng.set_search_params(B, tau, P)
        bases = [cdist.shard_range(X.shape[0], r, world)[0] for r in range(world)]
        ids, d = cdist.search_step_global(eng, torch.from_numpy(Q), k, 1, bases)
        if rank == 0:
            np.savez(out, ids=ids.numpy(), d=d.numpy(), R=R.numpy(), cb=cb.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_global_patience_orchestration_matches_single_index(world):
    """dist.search_step_global over gloo (the numpy engine above stands in for
    the CUDA kernels): Optimized Mode with the patience rule over the global
    (h, gid) order equals the single index's search (oracle), fallback
    queries included."""
    import oracle

    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "r0.npz")
        mp.start_processes(_gp_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                           start_method="spawn")
        res = dict(np.load(out))
    X, Q = _data()
    full = oracle.build(X, 4, K=6, R=res["R"], codebooks=res["cb"])
    ids, d, t = oracle.search(full, Q, 5, 1, 300, 3, patience_factor=8, trace=True)
    assert np.array_equal(res["ids"], ids)
    fin = np.isfinite(d)
    assert np.allclose(res["d"][fin], d[fin].astype(np.float32))


def _worker(rank, world, port, out, exact=False, tau=2):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_05180_b200 import dist as cdist

        X, Q = _data()
        M, k, B = 4, 5, 300
        eng = OracleEngine()
        R, cb = eng.build_global(X, M) if rank == 0 else (None, None)
        R, cb = cdist.share_model(R, cb, torch.zeros(1))
        lo, hi = cdist.shard_range(X.shape[0], rank, world)
        eng.build_shard(X[lo:hi], lo, M, R, cb)
        sizes = cdist.global_cell_sizes(eng)
        eng.set_search_params(B, tau)
        step = cdist.search_step_exact if exact else cdist.search_step
        ids, d = step(eng, torch.from_numpy(Q), k, 0)
        if rank == 0:
            np.savez(out, ids=ids.numpy(), d=d.numpy(), sizes=sizes.numpy(), R=R.numpy(), cb=cb.numpy())
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(exact, tau):
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "r0.npz")
        mp.start_processes(_worker, args=(2, _free_port(), out, exact, tau), nprocs=2, join=True,
                           start_method="spawn")
        return dict(np.load(out))


def test_exact_global_fallback_matches_single_index():
    """search_step_exact: every query, fallback ones included, equals the
    single index (P:L449 applied to the whole dataset)."""
    import oracle

    tau = 4
    res = _run(True, tau)
    X, Q = _data()
    full = oracle.build(X, 4, K=6, R=res["R"], codebooks=res["cb"])
    ids, d, t = oracle.search(full, Q, 5, 0, 300, tau, trace=True)
    assert t["fallback"].sum() >= 2  # the case under test occurs
    assert np.array_equal(res["ids"], ids)
    fin = np.isfinite(d)
    assert np.allclose(res["d"][fin], d[fin].astype(np.float32))


def test_sharded_orchestration_matches_single_index():
    import oracle

    res = _run(False, 2)
    X, Q = _data()
    M, k, B, tau = 4, 5, 300, 2
    full = oracle.build(X, M, K=6, R=res["R"], codebooks=res["cb"])
    assert np.array_equal(res["sizes"], full["gsize"])  # N3: global sizes == single index
    ids, d, t = oracle.search(full, Q, k, 0, B, tau, trace=True)
    # phi=0 is G-invariant except where a shard's own |C| < k (per-shard fallback, DESIGN 9)
    ok = t["cand_n"] >= 2 * k
    assert ok.sum() >= 10
    assert np.array_equal(res["ids"][ok], ids[ok])
    assert np.allclose(res["d"][ok], d[ok].astype(np.float32))


def _gather_worker(rank, world, port, N, D, ids, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_05180_b200 import dist as cdist

    X = torch.arange(N * D, dtype=torch.float32).reshape(N, D)
    lo, hi = cdist.shard_range(N, rank, world)
    got = cdist.gather_sample_rows(X[lo:hi], lo, torch.from_numpy(ids))
    if rank == 0:
        torch.save(got, out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_sample_rows(world):
    """The model build's sample rows (fixed global ids from the counter-based
    sampler, here the oracle's) gathered from point shards arrive on rank 0 in
    ascending global id, equal to the rows of the whole dataset."""
    import oracle

    N, D = 1003, 5
    ids = oracle.sample_rows(N, 101, 7, 1)
    assert np.all(np.diff(ids) > 0)
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "g.pt")
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        mp.spawn(_gather_worker, args=(world, port, N, D, ids, out), nprocs=world, join=True)
        got = torch.load(out)
    X = np.arange(N * D, dtype=np.float32).reshape(N, D)
    assert np.array_equal(got.numpy(), X[ids])
