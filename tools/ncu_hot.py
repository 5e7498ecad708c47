"""Top SASS instructions by warp-stall samples from `ncu --page source --csv`
(SASS view) plus the dominant stall reasons of each.

    ncu -i rep.ncu-rep --page source --csv > src.csv; python tools/ncu_hot.py src.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = next(i for i, r in enumerate(rows) if len(r) > 2 and r[0] == "Address")
h = rows[hdr]
idx = h.index("Warp Stall Sampling (All Samples)")
stalls = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
data = [r for r in rows[hdr + 1:] if len(r) > idx]
tot = sum(float(r[idx] or 0) for r in data)
agg = {}
for r in data:
    for i in stalls:
        agg[h[i]] = agg.get(h[i], 0) + float(r[i] or 0)
print("total samples", tot, "by reason:",
      {k: f"{100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]})
pos = {r[0]: k for k, r in enumerate(data)}
for r in sorted(data, key=lambda r: -float(r[idx] or 0))[:n]:
    top = sorted(((float(r[i] or 0), h[i][6:]) for i in stalls), reverse=True)[:2]
    print(f"{100 * float(r[idx]) / tot:5.1f}% {pos[r[0]]:5d} {r[1].strip()[:70]:70s}",
          " ".join(f"{k}:{int(v)}" for v, k in top))
