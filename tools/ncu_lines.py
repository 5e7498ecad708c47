"""Warp-stall samples per CUDA source line: joins `ncu --page source --csv`
(SASS view, one kernel) with `nvdisasm -g` line info of the same cubin.

    python tools/ncu_lines.py src.csv kernel.sass <mangled-function> [N]
"""
import collections
import csv
import os
import re
import sys

src_csv, sass, fn = sys.argv[1:4]
n_top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = list(csv.reader(open(src_csv)))
hdr = next(i for i, r in enumerate(rows) if len(r) > 2 and r[0] == "Address")
h = rows[hdr]
idx = h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[hdr + 1:] if len(r) > idx]
base = int(data[0][0], 16)
samples = {int(r[0], 16) - base: float(r[idx] or 0) for r in data}
line_of = {}
cur = None
inside = False
for ln in open(sass):
    if ln.startswith(".text."):
        inside = ln.strip() == f".text.{fn}:"
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1), int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
agg = collections.Counter()
for off, v in samples.items():
    agg[line_of.get(off, ("?", 0))] += v
tot = sum(agg.values())
cache = {}
for (f, l), v in agg.most_common(n_top):
    if f not in cache:
        cache[f] = open(f).read().split("\n") if os.path.exists(f) else []
    txt = cache[f][l - 1].strip() if 0 < l <= len(cache[f]) else ""
    print(f"{100 * v / tot:5.1f}% {os.path.basename(f)}:{l:<5d} {txt[:90]}")
