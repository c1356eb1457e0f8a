"""Print the hottest SASS instructions of an ncu source-page export
(ncu -i X.ncu-rep --page source --csv --print-source sass > f.csv):
per instruction the stall samples and the top stall reasons."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
data = []
tot = 0
for r in rows[2:]:
    if len(r) != len(h) or r[0] == "Address":
        if r and r[0] == "Kernel Name" and data:
            break  # several kernels in one export: the first only
        continue
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot += s
    data.append((s, r))
print("total samples", tot)
agg = {k: 0.0 for k in stalls}
for s, r in data:
    for k in stalls:
        agg[k] += float(r[ix[k]] or 0)
print("stall totals:", ", ".join(f"{k[6:]}={v/tot:.1%}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
for s, r in sorted(data, key=lambda x: -x[0])[:n]:
    top = sorted(((float(r[ix[k]] or 0), k[6:]) for k in stalls), reverse=True)[:3]
    print(f"{s/tot:6.1%} {r[ix['Address']]:>6} {r[ix['Source']][:60]:60s} ex={r[ix['Instructions Executed']]:>10} "
          + " ".join(f"{k}={v:.0f}" for v, k in top if v > 0))
