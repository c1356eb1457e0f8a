#!/usr/bin/env python
"""bench.py -- CRISP batched search on B200 (BASELINE.json metric:
"QPS at recall@10>=0.9 (1/2/4/8 B200); count/re-rank HBM GB/s vs peak").

A step = one crisp_search_async over the whole query batch (all hot-path
stages a0..a5, plus the a6 all-gather/merge when G > 1), inputs resident in
HBM.  Workload at N=1: BASELINE configs[3] (cfg4: N=2M, D=3072, Q=10k,
k=100, synthetic Simplewiki-OpenAI-like text embeddings), the
config the metric's "(1/2/4/8 B200)" names and the largest that fits one GPU,
at the operating point (M, beta, alpha, mode) of configs/operating_points.json,
which a sweep (--sweep) selected as the fastest with recall@10 >= 0.9 (of the
top 10 of the k=100 returned) against exact ground truth.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--cfg 4]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
OPS = os.path.join(ROOT, "configs", "operating_points.json")
FALLBACK_HBM = 6650.0  # B200_PROFILING.md fallback, GB/s


# --------------------------------------------------------------------------- utils
def log(*a):
    print(*a, file=sys.stderr, flush=True)


def env_int(n, d):
    return int(os.environ.get(n, d))


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.lines = []
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None
        return self

    def _read(self):
        for line in self.p.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, t0, t1):
        """Restrict the summary to samples that arrived inside [t0, t1] (host
        clock around the synchronized, timed region)."""
        self.win = (t0, t1)

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        win = getattr(self, "win", None)
        for ts, ln in self.lines:
            if win is not None and not (win[0] <= ts <= win[1] + 0.25):
                continue
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        out = {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}
        if win is not None:
            out["window_s"] = round(win[1] - win[0], 3)
        return out


def smem_update_peak():
    """(lane updates/s, source) of random-word red.shared.add measured in-repo
    (tools/peaks/smem_red_peak.cu -> profiles/r02_smem_peak.json), or None."""
    p = os.path.join(ROOT, "profiles", "r02_smem_peak.json")
    try:
        with open(p) as f:
            return json.load(f)["red_random"]["lane_updates_per_s"], "measured in-repo (profiles/r02_smem_peak.json)"
    except Exception:
        return None


def l2_peak():
    """In-repo L2 -> SM read bandwidth (tools/measure_peaks.py), if measured."""
    f = os.path.join(ROOT, "profiles", "r02_peaks.json")
    try:
        with open(f) as fh:
            return float(json.load(fh)["l2_read_gbs_48MiB"]), "measured in-repo (profiles/r02_peaks.json)"
    except Exception:
        return None


def hbm_peak():
    try:
        with open(PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


MODE_NAMES = ["guaranteed", "optimized", "optimized_adsampling"]


def phi(mode: int) -> int:
    """Execution flag of a bench mode: 0 Guaranteed, 1 Optimized; bench mode 2 is
    Optimized Mode verified by ADSampling (Eq. 2, crisp_set_adsampling)."""
    return 0 if mode == 0 else 1


def load_op(cfg: int, mode_override=None):
    """{M, seed, modes: {mode: {beta, alpha}}} restricted to --mode if given."""
    with open(OPS) as f:
        ops = json.load(f)
    op = dict(ops[str(cfg)])
    modes = {int(m): v for m, v in op["modes"].items()}
    if mode_override is not None:
        modes = {mode_override: modes.get(mode_override, next(iter(modes.values())))}
    op["modes"] = modes
    return op


def ground_truth(X, Qd, k, extra=32):
    """Exact kNN: fp32 screening on the GPU (TF32 off), exact fp64
    re-check of the best k+extra, ties by id.  Setup, not timed."""
    torch.backends.cuda.matmul.allow_tf32 = False
    xn = torch.empty(X.shape[0], dtype=torch.float32, device=X.device)
    for r0 in range(0, X.shape[0], 65536):  # row norms without an N x D fp64 temporary
        xn[r0:r0 + 65536] = (X[r0:r0 + 65536].double() ** 2).sum(1).float()
    out = torch.empty((Qd.shape[0], k), dtype=torch.int64, device=X.device)
    for q0 in range(0, Qd.shape[0], 256):
        q = Qd[q0:q0 + 256]
        d = xn[None, :] - 2.0 * (q @ X.T) + (q.double() ** 2).sum(1).float()[:, None]
        cand = torch.topk(d, k + extra, dim=1, largest=False).indices
        xc = X[cand].double()
        dd = ((xc - q.double()[:, None, :]) ** 2).sum(2)
        # sort by (d, id): ids are < 2^31, distances > 0 -> lexsort via two stable sorts
        o = torch.argsort(cand, dim=1, stable=True)
        dd, cand = dd.gather(1, o), cand.gather(1, o)
        o = torch.argsort(dd, dim=1, stable=True)
        out[q0:q0 + 256] = cand.gather(1, o)[:, :k]
    torch.cuda.empty_cache()
    return out


def recall_at(ids, gt, k=10):
    ids = ids[:, :k].cpu().numpy() if hasattr(ids, "cpu") else np.asarray(ids)[:, :k]
    gt = gt[:, :k].cpu().numpy() if hasattr(gt, "cpu") else np.asarray(gt)[:, :k]
    hits = [len(set(a.tolist()) & set(b.tolist())) for a, b in zip(ids, gt)]
    return float(np.mean(hits)) / k


# --------------------------------------------------------------------------- oracle (reference arm / cpu_baseline)
def cpu_info():
    """lscpu model / sockets / threads of the host the oracle runs on."""
    kv = {}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=20).stdout
        for ln in out.splitlines():
            if ":" in ln:
                a, b = ln.split(":", 1)
                kv[a.strip()] = b.strip()
    except Exception:
        pass

    def num(key):
        try:
            return int(kv[key])
        except Exception:
            return None

    return {"model": kv.get("Model name"), "sockets": num("Socket(s)"), "cores_per_socket": num("Core(s) per socket"),
            "threads_per_core": num("Thread(s) per core"), "cpus": num("CPU(s)") or os.cpu_count()}


def oracle_index_of(index):
    """The oracle's index dict holding the arrays the GPU index exports (X', R,
    codebooks, cell assignment, CSR, codes): the same index the GPU searches.
    The oracle's own build cannot run at cfg4/cfg5 within minutes (X' = X R
    over 2M x 3072^2 is ~38 TFLOP of sequential fp64 chains), and the build is
    not part of the timed step; only the oracle's search is timed."""
    e = index.export()
    i = index.info()
    return dict(N=i["N"], D=i["D"], Dp=i["padded_D"], M=i["M"], K=i["K"], dh=i["dh"], X=e["X"], R=e["R"],
                rotated=bool(i["rotated"]), cev=i["cev"], cb=e["codebooks"], cells=e["cells"], off=e["offsets"],
                ids=e["ids"], codes=e["codes"], gsize=e["cell_sizes"], gid_base=i["gid_base"], N_budget=i["N_global"])


def time_oracle(ox, Qh, k, mode, B, tau, budget_seconds=12.0, single_seconds=4.0, patience_factor=40):
    """The oracle's search (as it stands) on the host: all cores (OpenMP over
    queries) on a bounded sample sized to ~budget_seconds, then one thread on
    up to 100 queries (~single_seconds).  Returns a cpu_baseline dict."""
    import oracle

    cores = os.cpu_count() or 1
    Q = Qh.shape[0]
    kw = dict(patience_factor=patience_factor, adsampling=mode == 2)
    nq = min(32, Q)
    t0 = time.perf_counter()
    oracle.search(ox, Qh[:nq], k, phi(mode), B, tau, nthreads=cores, **kw)
    per_q = (time.perf_counter() - t0) / nq
    n = int(min(Q, max(nq, budget_seconds / max(per_q, 1e-7))))
    t0 = time.perf_counter()
    oracle.search(ox, Qh[:n], k, phi(mode), B, tau, nthreads=cores, **kw)
    dt = time.perf_counter() - t0
    per_q1 = dt / n * cores  # single-thread estimate for sizing only
    n1 = int(min(100, Q, max(4, single_seconds / max(per_q1, 1e-7))))
    t0 = time.perf_counter()
    oracle.search(ox, Qh[:n1], k, phi(mode), B, tau, nthreads=1, **kw)
    dt1 = time.perf_counter() - t0
    return {"value": n / dt, "unit": "queries/s", "cores": cores, "kind": "oracle",
            "single_thread": {"value": n1 / dt1, "unit": "queries/s", "queries": n1},
            "host": cpu_info(), "queries": n, "seconds": dt}


def run_reference(args):
    """--impl reference: the oracle's search, timed as it stands on the box's
    host cores, on the GPU arm's config (its index: oracle_index_of)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle

    cfg = args.cfg
    c = synth.CONFIGS[cfg]
    N, Q, k, D = args.N or c["N"], args.Q or c["Q"], c["k"], c["D"]
    op = load_op(cfg, args.mode)
    # Optimized Mode with exact verification (the GPU arm's headline mode), else
    # the config's last mode
    mode0 = (1 if 1 in op["modes"] else sorted(op["modes"])[-1]) if args.mode is None else args.mode
    mp = op["modes"][mode0]
    cores = os.cpu_count() or 1
    if torch.cuda.is_available():
        import __graft_entry__ as ge

        ge.build()
        import paper_2603_05180_b200 as crisp

        w = synth.Workload(cfg, device="cuda")
        X = w.base(N)
        Qd = w.queries(Q)
        gt = ground_truth(X, Qd, k)
        ix = crisp.Index.build(X, op["M"], K=50, seed=op.get("seed", 1))
        del X
        torch.cuda.empty_cache()
        ox = oracle_index_of(ix)
        ix.free()
        src = "the index the GPU arm searches (crisp_build, exported; build not timed)"
    else:  # CPU-only host (tests): the oracle builds its own index
        w = synth.Workload(cfg)
        X = w.base(N)
        Qd = w.queries(Q)
        gt = None
        ox = oracle.build(X.numpy(), op["M"], K=50, kmeans_iters=20, kmeans_sample=100000, seed=op.get("seed", 1))
        src = "built by the oracle (not timed)"
    Qh = Qd.cpu().numpy()
    B, tau = oracle.budget_ids(mp["beta"], N), oracle.tau_int(mp["alpha"], op["M"])
    kw = dict(patience_factor=mp.get("patience_factor", 40), adsampling=mode0 == 2)
    # per step: a bounded sample sized so the whole run takes ~args.cpu_seconds
    nq = min(32, Q)
    t0 = time.perf_counter()
    oracle.search(ox, Qh[:nq], k, phi(mode0), B, tau, nthreads=cores, **kw)
    per_q = (time.perf_counter() - t0) / nq
    per_step = max(1, min(Q, int(args.cpu_seconds / max(per_q, 1e-7) / max(1, args.steps + args.warmup))))
    for s in range(args.warmup):
        oracle.search(ox, Qh[:per_step], k, phi(mode0), B, tau, nthreads=cores, **kw)
    t0 = time.perf_counter()
    res = []
    for s in range(args.steps):
        lo = (s * per_step) % max(1, Q - per_step + 1)
        ids, _, _ = oracle.search(ox, Qh[lo:lo + per_step], k, phi(mode0), B, tau, nthreads=cores, **kw)
        res.append((lo, ids))
    dt = time.perf_counter() - t0
    qps = per_step * args.steps / dt
    rec = None
    if gt is not None:
        rec = float(np.mean([recall_at(ids, gt[lo:lo + per_step], 10) for lo, ids in res]))
    sample = (f"{per_step} queries per step x {args.steps} steps of {c['name']} (N={N}); oracle index = {src}")
    line = {
        "impl": "reference", "metric": "QPS at recall@10>=0.9", "value": qps, "unit": "queries/s", "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": c["name"], "N": N, "D": D, "Q": Q, "k": k, "M": op["M"], "beta": mp["beta"],
                   "alpha": mp["alpha"], "mode": MODE_NAMES[mode0]},
        "recall@10": rec,
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": cores, "kind": "oracle", "sample": sample,
                         "host": cpu_info()},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- crisp arm
def run_crisp(args):
    import __graft_entry__ as ge

    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: CRISP_BENCH_DEVICE pins every rank to one GPU, with the gloo
    # backend (no GPU kernel waits on another rank), to exercise the N>1 path
    # on a single-GPU box; the driver's N>1 runs use one GPU per rank and NCCL
    if os.environ.get("CRISP_BENCH_DEVICE") is not None:
        local = int(os.environ["CRISP_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if rank == 0:
        ge.build()
    if world > 1:
        import torch.distributed as dist

        if os.environ.get("CRISP_BENCH_DEVICE") is not None:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        dist.barrier()
    import paper_2603_05180_b200 as crisp
    from paper_2603_05180_b200 import dist as cdist

    cfg = args.cfg
    c = synth.CONFIGS[cfg]
    N, Q, k, D = args.N or c["N"], args.Q or c["Q"], c["k"], c["D"]
    op = load_op(cfg, args.mode)
    M = op["M"]
    w = synth.Workload(cfg, device=dev)
    t0 = time.time()
    Qd = w.queries(Q)
    X = w.base(N) if (rank == 0) else None
    gen_s = time.time() - t0
    bparams = dict(K=50, seed=op.get("seed", 1))
    t0 = time.time()
    if world == 1:
        index = crisp.Index.build(X, M, **bparams)
        engine = None
    else:
        engine = cdist.CudaEngine(crisp, dev)
        lo, hi = cdist.shard_range(N, rank, world)
        Xs = w.rows(lo, hi - lo)
        # N1/N2: the model from the gathered CEV / k-means sample rows (no full index on rank 0)
        R, cb = cdist.model_from_shards(engine, Xs, lo, N, M, seed=bparams["seed"], K=bparams["K"])
        engine.build_shard(Xs, lo, M, R, cb, **bparams)
        del Xs
        cdist.global_cell_sizes(engine)
        index = engine.index
    torch.cuda.synchronize()
    build_s = time.time() - t0
    if world > 1:
        # Optimized Mode: the patience rule over the global (h, gid) order (exact for every G,
        # dist.search_step_global); CRISP_SHARD_PATIENCE=local keeps per-shard patience (Z23)
        gid_bases = [cdist.shard_range(N, r, world)[0] for r in range(world)]
        local_pat = os.environ.get("CRISP_SHARD_PATIENCE", "global") == "local"

        def shard_step(eng, q, k_, m_, st_):
            if m_ == 1 and not local_pat:
                return cdist.search_step_global(eng, q, k_, m_, gid_bases, st_)
            return cdist.search_step_exact(eng, q, k_, m_, st_)
    gt = ground_truth(X, Qd, k) if rank == 0 else None
    stream = torch.cuda.current_stream().cuda_stream
    ids = torch.empty((Q, k), dtype=torch.int64, device=dev)
    dd = torch.empty((Q, k), dtype=torch.float32, device=dev)
    peak, peak_src = hbm_peak()
    K = args.steps
    results = {}
    for mode, mp in sorted(op["modes"].items()):
        index.set_search_params(beta=mp["beta"], alpha=mp["alpha"], patience_factor=mp.get("patience_factor", 40))
        index.set_adsampling(mode == 2)
        info = index.info()

        def step():
            if world == 1:
                index.search_async(Qd, k, phi(mode), ids, dd, stream)
                return ids
            oi, _ = shard_step(engine, Qd, k, phi(mode), stream)
            return oi

        # the clock sampler starts before the warm-up (nvidia-smi needs ~0.5 s to
        # report) and its summary keeps only the samples of the timed region
        with Clocks(local) as clk:
            for _ in range(args.warmup):
                out = step()
            torch.cuda.synchronize()
            crisp.stage_times(reset=True)
            crisp.search_counters(reset=True)
            # the timed steps record the stage events only (no tally kernels in the timed work);
            # the work counters of one step come from an extra step after the timed region
            crisp.set_stage_timing(2)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t_h0 = time.time()
            e0.record()
            for _ in range(K):
                out = step()
            e1.record()
            torch.cuda.synchronize()
            t_h1 = time.time()
            if world > 1:
                dist.barrier()
            clk.mark(t_h0, t_h1)
            time.sleep(0.3)  # let the sample of the region's last 200 ms arrive
        ms = e0.elapsed_time(e1)
        st = crisp.stage_times(reset=True)
        crisp.set_stage_timing(1)
        crisp.search_counters(reset=True)
        step()
        torch.cuda.synchronize()
        crisp.stage_times(reset=True)
        cnt = {kk: v * K for kk, v in crisp.search_counters(reset=True).items()}  # K identical steps
        crisp.set_stage_timing(False)
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        rec = recall_at(out, gt, 10) if rank == 0 else None

        # roofline of the hot kernels: algorithmic bytes / CUDA-event time per step
        row_bytes = 4 * info["pitch"]
        kernels = {}
        if st["verify"] > 0:
            vb = cnt["verified"] * row_bytes / K  # 4D per verified row (SURVEY 8(d) B_rerank)
            # phi=0: the grouped re-rank is opt-in (CRISP_RERANK_GROUP=1; search.cu Work)
            grp = os.environ.get("CRISP_RERANK_GROUP", "0") != "0"
            vname = ["k_rerank_group" if grp else "k_rerank_exact", "k_verify_rows+k_patience_scan+k_patience_tail",
                     "k_verify_rows(_ad)+k_patience_scan+k_patience_tail"][mode]
            model = "4 pitch B per verified row (SURVEY 8(d) B_rerank)"
            if cnt.get("filter_rows", 0) > 0:
                # verification filter (DESIGN R17): c8pitch + 16 B per row bounded through the
                # int8 copy, 4 pitch B per row read exactly (round 0, rows the bound keeps, the tail)
                hrow = (info["pitch"] + 15) // 16 * 16 + 16
                fr, fe = cnt["filter_rows"], cnt["filter_exact"]
                if mode == 0:
                    vb = (cnt["candidates"] * (hrow + 16) + fe * row_bytes) / K
                    vname = "k_lb_bounds+k_lb_threshold+k_rerank_exact"
                else:
                    vb = ((max(0, cnt["verified"] - fr) + fe) * row_bytes + fr * hrow) / K
                    vname = "k_verify_rows+k_verify_rows_lb+k_patience_scan+k_patience_tail"
                model = "c8pitch + 16 B per row bounded through the int8 copy + 4 pitch B per row read exactly (R17)"
            kernels["verify"] = {"kernel": vname, "bytes_per_step": vb, "ms_per_step": st["verify"] / K,
                                 "achieved_gbs": vb / (st["verify"] / K * 1e-3) / 1e9, "bytes_model": model}
        if st["count_select"] > 0:
            # a3 streams 4 B per id (SURVEY 8(d) B_count); at phi=1 the same kernel
            # (k_count_warp) also gathers 8*ceil(D'/64) B of code per candidate (B_ham)
            cb_ = cnt["ids_streamed"] * 4 / K
            ck = os.environ.get("CRISP_COUNT_KERNEL", "1" if info["slice_hint"] >= 8.0 else "2")
            warp_kernel = ck == "1"
            fused = warp_kernel and os.environ.get("CRISP_HAMMING_FUSED", "0") != "0"
            name = {"0": "k_count_select", "1": "k_count_warp", "2": "k_act_rows+k_count_frag"}[ck]
            if phi(mode) == 1 and fused:
                cb_ += cnt["candidates"] * 8 * ((info["padded_D"] + 63) // 64) / K
                name = "k_count_warp (collision count + fused Hamming)"
            kernels["count"] = {"kernel": name, "bytes_per_step": cb_, "ms_per_step": st["count_select"] / K,
                                "achieved_gbs": cb_ / (st["count_select"] / K * 1e-3) / 1e9}
            if phi(mode) == 1 and not fused and st.get("hamming", 0) > 0:
                hb = cnt["candidates"] * 8 * ((info["padded_D"] + 63) // 64) / K  # SURVEY 8(d) B_ham
                kernels["hamming"] = {"kernel": "k_qcodes+k_hamming_seg(or k_hamming_dense)+k_hhist",
                                      "bytes_per_step": hb, "ms_per_step": st["hamming"] / K,
                                      "achieved_gbs": hb / (st["hamming"] / K * 1e-3) / 1e9}
        l2 = l2_peak()
        for name_, kk in kernels.items():
            kk["frac_of_peak"] = kk["achieved_gbs"] / peak
            kk["bound"] = "hbm"
            if name_ == "hamming" and l2:
                # the code rows of one id block stay in L2 while every query's candidates in it are
                # scored (k_hamming_seg): the ceiling that binds is the L2 read rate
                kk["bound"], kk["peak"], kk["peak_source"] = "l2", l2[0], l2[1]
                kk["frac_of_peak"] = kk["achieved_gbs"] / l2[0]
            elif name_ == "count":
                # issue / LSU-latency bound (DESIGN 7: ncu with source, 0.17 of the measured red.shared
                # ceiling): the HBM fraction of its id stream is reported, the stream does not bind
                kk["bound"] = "issue/LSU latency (shared-memory reductions); frac = id stream / HBM, update_frac = updates / measured red.shared ceiling"
                sp = smem_update_peak()
                if sp:
                    # one counter update per streamed id (Alg. 1 l.14-17); the ceiling is the measured
                    # rate of random-word red.shared.add on this GPU in the count's launch shape
                    ups = cnt["ids_streamed"] / K / (kk["ms_per_step"] * 1e-3)
                    kk["updates_per_s"], kk["update_peak_per_s"], kk["update_peak_source"] = ups, sp[0], sp[1]
                    kk["update_frac"] = ups / sp[0]
        dom = max(kernels, key=lambda n: kernels[n]["ms_per_step"]) if kernels else None
        traffic = None
        tf = os.path.join(ROOT, "profiles", "traffic.json")
        if dom and os.path.exists(tf):
            try:
                with open(tf) as f:
                    tj = json.load(f)
                key = f"cfg{cfg}-mode{mode}-{kernels[dom]['kernel']}"
                if key in tj:
                    traffic = tj[key]["dram_bytes_per_step"]
            except Exception:
                traffic = None
        roof = None
        if dom:
            a = kernels[dom]["achieved_gbs"]
            sec = kernels[dom]["ms_per_step"] * 1e-3
            roof = {"bound": "hbm", "achieved": a, "peak": peak, "unit": "GB/s", "frac": a / peak, "traffic": traffic,
                    "kernel": kernels[dom]["kernel"], "peak_source": peak_src,
                    "per": "step (the stage's launches summed: bytes and CUDA-event time per step)"}
            if kernels[dom].get("bytes_model"):
                roof["bytes_model"] = kernels[dom]["bytes_model"]
            if traffic:
                # the DRAM side of the same stage: measured bytes (ncu) over the live time
                roof["dram_gbs"] = traffic / sec / 1e9
                roof["dram_frac"] = roof["dram_gbs"] / peak
            if l2:
                # the algorithmic stream is served from L2 and DRAM: its ceiling is the L2 read rate
                roof["l2_peak"] = l2[0]
                roof["l2_frac"] = a / l2[0]
                roof["l2_peak_source"] = l2[1]
        results[mode] = dict(qps=Q * K / (ms / 1e3), ms=ms / K, recall=rec, beta=mp["beta"], alpha=mp["alpha"],
                             budget_ids=info["budget"], tau=info["tau"],
                             patience_factor=info["patience_factor"] if phi(mode) == 1 else None,
                             roofline=roof, kernels=kernels,
                             stage_ms_per_step={k_: v / K for k_, v in st.items()},
                             counters_per_step={k_: v / K for k_, v in cnt.items()}, launches=cnt["launches"],
                             clocks=clk.summary())
        if rank == 0:
            log(f"mode {mode}: {results[mode]['qps']:.0f} QPS recall@10 {rec:.4f} stages {results[mode]['stage_ms_per_step']}")

    # headline: the fastest mode whose recall@10 >= 0.9
    ok = [m for m, r in results.items() if r["recall"] is None or r["recall"] >= 0.9]
    head = max(ok or list(results), key=lambda m: results[m]["qps"])
    hr = results[head]

    # e2e through the public API with host buffers (H2D queries + D2H results per step)
    e2e = None
    if rank == 0 and world == 1:
        mp = op["modes"][head]
        index.set_search_params(beta=mp["beta"], alpha=mp["alpha"], patience_factor=mp.get("patience_factor", 40))
        index.set_adsampling(head == 2)
        qh = torch.empty((Q, D), dtype=torch.float32).pin_memory()
        qh.copy_(Qd.cpu())
        qn = qh.numpy()
        ih = torch.empty((Q, k), dtype=torch.int64).pin_memory().numpy()
        dh = torch.empty((Q, k), dtype=torch.float32).pin_memory().numpy()
        for _ in range(max(3, args.warmup)):  # the same warm-up as the device-timed steps
            crisp._check(crisp.lib().crisp_search(index._h, crisp._ptr(qn), Q, k, phi(head), crisp._ptr(ih),
                                                  crisp._ptr(dh)))
        t0 = time.perf_counter()
        for _ in range(K):
            crisp._check(crisp.lib().crisp_search(index._h, crisp._ptr(qn), Q, k, phi(head), crisp._ptr(ih),
                                                  crisp._ptr(dh)))
        dt = time.perf_counter() - t0
        e2e = {"value": Q * K / dt, "unit": "queries/s", "h2d_bytes_per_step": Q * D * 4,
               "d2h_bytes_per_step": Q * k * 12, "recall@10": recall_at(ih, gt, 10), "api": "crisp_search (host buffers)"}

    if world > 1:
        # e2e at N GPUs: every rank copies the step's queries from pinned host memory,
        # runs the sharded search (collectives included) and rank 0 reads the merged
        # ids back; wall clock between barriers, max over ranks
        mp = op["modes"][head]
        index.set_search_params(beta=mp["beta"], alpha=mp["alpha"], patience_factor=mp.get("patience_factor", 40))
        index.set_adsampling(head == 2)
        qh = torch.empty((Q, D), dtype=torch.float32).pin_memory()
        qh.copy_(Qd.cpu())
        qe = torch.empty_like(Qd)
        ih = torch.empty((Q, k), dtype=torch.int64).pin_memory()

        def e2e_step():
            qe.copy_(qh, non_blocking=True)
            oi, _ = shard_step(engine, qe, k, phi(head), stream)
            if rank == 0:
                ih.copy_(oi, non_blocking=True)
            torch.cuda.current_stream().synchronize()

        for _ in range(2):
            e2e_step()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(K):
            e2e_step()
        dist.barrier()
        tt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64,
                          device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        e2e = {"value": Q * K / dt, "unit": "queries/s", "h2d_bytes_per_step": world * Q * D * 4,
               "d2h_bytes_per_step": Q * k * 8, "recall@10": recall_at(ih.numpy(), gt, 10) if rank == 0 else None,
               "api": "dist.search_step_global (host queries on every rank, merged ids to rank 0's host)"}

    # cpu baseline (rank 0, N=1 only): the oracle's search as it stands on the
    # host cores, on the index the GPU searched (oracle_index_of)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle

        mp = op["modes"][head]
        del X
        torch.cuda.empty_cache()
        ox = oracle_index_of(index)
        B, tau = oracle.budget_ids(mp["beta"], N), oracle.tau_int(mp["alpha"], M)
        cpu = time_oracle(ox, Qd.cpu().numpy(), k, head, B, tau, budget_seconds=args.cpu_seconds,
                          patience_factor=mp.get("patience_factor", 40))
        cpu["sample"] = (f"first {cpu['queries']} of the {Q} queries ({MODE_NAMES[head]} mode, all {cpu['cores']} "
                         f"host threads); single thread on the first {cpu['single_thread']['queries']}; oracle "
                         f"index = the GPU index's exported arrays (X', R, codebooks, CSR, codes)")
        del ox

    if rank == 0:
        info = index.info()
        line = {
            "metric": "QPS at recall@10>=0.9", "value": hr["qps"], "unit": "queries/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": hr["ms"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": c["name"], "N": N, "D": D, "Q": Q, "k": k, "M": M, "beta": hr["beta"],
                       "alpha": hr["alpha"], "mode": MODE_NAMES[head], "budget_ids": hr["budget_ids"],
                       "patience_factor": hr.get("patience_factor"),
                       "tau": hr["tau"], "rotated": bool(info["rotated"]), "cev": info["cev"],
                       "l2": "inputs larger than L2 (X = %.2f GB >> 126 MB); no flush" % (N * D * 4 / 1e9),
                       "parallelism": f"points sharded x{world}" if world > 1 else "single GPU"},
            "recall@10": hr["recall"],
            "roofline": hr["roofline"],
            "kernels": hr["kernels"],
            "stage_ms_per_step": hr["stage_ms_per_step"],
            "counters_per_step": hr["counters_per_step"],
            "gpu_launches": hr["launches"],
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": hr["clocks"],
            "per_mode": {MODE_NAMES[m]: {k_: v for k_, v in r.items() if k_ != "clocks"}
                         for m, r in results.items()},
            "build_seconds": build_s,
            "gen_seconds": gen_s,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# --------------------------------------------------------------------------- sweep
def run_sweep(args):
    """Grid over (M, beta, alpha, mode) -> recall@10 and QPS (1 timed step)."""
    import __graft_entry__ as ge

    ge.build()
    import paper_2603_05180_b200 as crisp

    cfg = args.cfg
    c = synth.CONFIGS[cfg]
    N, Q, k = args.N or c["N"], args.Q or c["Q"], c["k"]
    dev = torch.device("cuda", 0)
    w = synth.Workload(cfg, device=dev)
    X, Qd = w.base(N), w.queries(Q)
    gt = ground_truth(X, Qd, k)
    Ms = [int(m) for m in args.sweep_M.split(",")]
    betas = [float(b) for b in args.sweep_beta.split(",")]
    alphas = [float(a) for a in args.sweep_alpha.split(",")]
    modes = [int(m) for m in args.sweep_modes.split(",")]
    ids = torch.empty((Q, k), dtype=torch.int64, device=dev)
    dd = torch.empty((Q, k), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    rows = []
    for M in Ms:
        t0 = time.time()
        ix = crisp.Index.build(X, M, K=50, seed=c["seed"])
        log(f"built M={M} in {time.time() - t0:.1f}s rotated={ix.info()['rotated']} cev={ix.info()['cev']:.3f}")
        pfs = [int(x) for x in args.sweep_patience.split(",")]
        for mode in modes:
          for pf in (pfs if mode != 0 else [40]):
            for beta in betas:
                for alpha in alphas:
                    ix.set_search_params(beta=beta, alpha=alpha, patience_factor=pf)
                    ix.set_adsampling(mode == 2)
                    ix.search_async(Qd, k, phi(mode), ids, dd, stream)
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    ix.search_async(Qd, k, phi(mode), ids, dd, stream)
                    e1.record()
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1)
                    r = dict(cfg=cfg, M=M, mode=mode, beta=beta, alpha=alpha, patience_factor=pf,
                             recall=recall_at(ids, gt, 10), qps=Q / ms * 1e3, ms=ms)
                    rows.append(r)
                    print(json.dumps(r), flush=True)
        ix.free()
    best = {}
    for mode in modes:
        ok = [r for r in rows if r["mode"] == mode and r["recall"] >= 0.9]
        if ok:
            best[mode] = max(ok, key=lambda r: r["qps"])
    print(json.dumps({"best": best}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="crisp", choices=["crisp", "reference"])
    ap.add_argument("--cfg", type=int, default=4)
    ap.add_argument("--mode", type=int, default=None)
    ap.add_argument("--N", type=int, default=None)
    ap.add_argument("--Q", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--sweep-M", default="16")
    ap.add_argument("--sweep-beta", default="0.005,0.01,0.02,0.04")
    ap.add_argument("--sweep-alpha", default="0.1,0.2,0.3,0.4")
    ap.add_argument("--sweep-modes", default="0,1")
    ap.add_argument("--sweep-patience", default="40", help="patience factors for phi=1 (P = factor * k; P:L713-718)")
    args = ap.parse_args()
    if args.warmup < 3 and not args.sweep:
        log("warning: fewer than 3 warm-up steps")
    if args.sweep:
        return run_sweep(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_crisp(args)


if __name__ == "__main__":
    sys.exit(main())
