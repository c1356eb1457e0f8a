"""Summarise ncu outputs for profiles/: a launch list (--metrics gpu__time_duration.sum --csv)
into per-kernel totals/shares, and a --set full report into key per-kernel metrics."""
import csv
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__grid_size",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_wait",
        "smsp__pcsamp_warps_issue_stalled_mio_throttle", "smsp__pcsamp_sample_count"]


SEARCH = ("k_prep_queries", "k_gemm_seq", "k_slice_rows", "k_certify", "k_recompute", "gemm_s8", "k_probe", "k_query_key", "k_count_warp", "k_count_select", "k_count_frag", "k_fallback",
          "k_rerank_exact",
          "k_merge_lists", "k_rerank_patience", "k_stats", "k_hamming", "k_hsort", "k_verify", "k_patience")


def launches(path, search_only=True):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
                 "s": 1e3, "second": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        if search_only and not any(t in name for t in SEARCH):
            continue
        tot[name][0] += 1
        tot[name][1] += v * scale
    all_ms = sum(t for _, t in tot.values())
    return {k: {"launches": n, "total_ms": t, "share": t / all_ms} for k, (n, t) in
            sorted(tot.items(), key=lambda kv: -kv[1][1])}


def full(path):
    out = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for k in KEYS:
            if k in h:
                d[k] = f"{r[h.index(k)]} {u[h.index(k)]}".strip()
        res.append(d)
    return res


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launches(path) if kind == "launches" else full(path), indent=1))
