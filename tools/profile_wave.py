"""Heavy ATLAS rows on the wave kernel (one warp per pipeline): per-row cycles
of the forward phase per warp, the drain, and the cycles each pipeline spent
waiting for the earlier pipelines' link frontiers.

    python tools/profile_wave.py [config2] [top=10]
"""
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_2411_14458_b200 import abi, workloads  # noqa: E402
from paper_2411_14458_b200.planner import Planner  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "config2"
top = int(sys.argv[2]) if len(sys.argv) > 2 else 10
topos, scens = getattr(workloads, cfg)()
p = Planner(0)
p.set_profile(True)
n = p.load(abi.array(abi.Topology, topos), abi.array(abi.Scenario, scens))
p.evaluate()
p.evaluate()
raw = (C.c_int64 * (17 * n))()
p._check(p.lib.gpb_fetch_row_cycles(p.ctx, raw, 17 * n))
rows = p.rows()
heavy = [b for b in p.bucket_infos() if b.policy == 3]
print("atlas buckets:", [(b.B, b.rows, round(b.ms, 3)) for b in heavy])
cand = []
for i in range(n):
    s = scens[rows[i].scenario]
    if s.policy == 3 and rows[i].feasible == 1:
        cand.append((raw[i], i))
cand.sort(reverse=True)
for cyc, i in cand[:top]:
    s = scens[rows[i].scenario]
    ph = list(raw[n + 16 * i: n + 16 * i + 16])
    S = -(-s.num_layers // s.layers_per_partition)
    print(f"row {i} S={S} C={s.pipelines_per_cell} M={s.num_microbatches} L={s.mem_limit}: "
          f"{cyc / 1e3:.0f} kcyc; fwd {ph[0] / 1e3:.0f} k (per warp {[round(x / 1e3) for x in ph[4:8]]}), "
          f"drain {ph[3] / 1e3:.0f} k, waits {[round(x / 1e3) for x in ph[8:12]]} k")
