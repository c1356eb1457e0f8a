"""Per-kernel DRAM / L2 traffic of ONE search step from an ncu metrics capture
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
lts__t_sectors_srcunit_tex_op_read.sum --csv) of tools/one_search.py: the
launches from the last k_prep_queries on (the second search) are summed per
kernel and per bench stage.  Usage: traffic_summary.py <csv> <key-prefix> [out.json]
(cold-cache, serialised launches: use the bytes, not the times)."""
import csv
import json
import sys
from collections import OrderedDict

STAGE = {"k_rot_tc": "transform", "k_slice_rows": "transform", "k_recompute": "transform", "k_recompute_rows": "transform",
         "k_probe": "probe", "k_query_key": "probe", "k_act_rows": "count_select", "k_count_frag": "count_select",
         "k_count_warp": "count_select", "k_count_select": "count_select", "k_fallback": "fallback",
         "k_hamming_dense": "hamming", "k_hamming": "hamming", "k_hsort_cta": "hsort", "k_hsort": "hsort",
         "k_verify_rows": "verify", "k_verify_rows_ad": "verify", "k_patience_scan": "verify",
         "k_patience_tail": "verify", "k_rerank_exact": "verify", "k_merge_lists": "merge",
         "k_verify_rows_lb": "verify", "k_q8_prep": "verify", "k_lb_bounds": "verify", "k_lb_threshold": "verify",
         "k_screen_tc": "probe", "k_qcodes": "hamming", "k_hamming_seg": "hamming", "k_hhist": "hamming",
         "k_prep_queries": "transform"}


def main():
    path, prefix = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ui, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    launches = OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(r[idi], {"name": r[ki]})
        v = float(r[vi].replace(",", "")) if r[vi] not in ("", "n/a") else float("nan")
        scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                 "sector": 1.0}.get(r[ui], 1.0)
        d[r[mi]] = v * scale
    seq = list(launches.values())
    start = max(i for i, d in enumerate(seq) if "k_prep_queries" in d["name"])
    per_kernel, per_stage = OrderedDict(), OrderedDict()
    for d in seq[start:]:
        name = d["name"].split("(")[0].split("::")[-1].split("<")[0].replace("void ", "").strip()
        e = per_kernel.setdefault(name, {"launches": 0, "ms": 0.0, "dram_bytes": 0.0, "l2_read_bytes": 0.0})
        e["launches"] += 1
        e["ms"] += d.get("gpu__time_duration.sum", 0.0)
        e["dram_bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        e["l2_read_bytes"] += 32.0 * d.get("lts__t_sectors_srcunit_tex_op_read.sum", 0.0)
        st = STAGE.get(name, "other")
        s = per_stage.setdefault(st, {"ms": 0.0, "dram_bytes": 0.0, "l2_read_bytes": 0.0})
        for k_ in ("ms", "dram_bytes", "l2_read_bytes"):
            s[k_] += e[k_] if False else 0.0
    for name, e in per_kernel.items():
        s = per_stage[STAGE.get(name, "other")]
        for k_ in ("ms", "dram_bytes", "l2_read_bytes"):
            s[k_] += e[k_]
    out = {"source": path, "prefix": prefix, "per_kernel": per_kernel, "per_stage": per_stage}
    print(json.dumps(out, indent=1))
    if len(sys.argv) > 3:
        with open(sys.argv[3], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
