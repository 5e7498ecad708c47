"""Bucket timeline of one rank's cost shard of the N-GPU headline space
(config2(N x 10^4, seed 1)) on one GPU, and its slowest rows.

    python tools/shard_buckets.py N [rank] [reps]
"""
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_2411_14458_b200 import abi, workloads, distributed as D  # noqa: E402
from paper_2411_14458_b200.planner import Planner  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
topos, scens = workloads.config2(10_000 * N, seed=1)
shard = D.shard_by_cost(scens, N)[rank]
sc = [scens[i] for i in shard]
p = Planner(0)
p.set_profile(True)
n = p.load(abi.array(abi.Topology, topos), abi.array(abi.Scenario, sc))
for _ in range(reps):
    p.evaluate()
t = p.timing()
print(f"N={N} rank {rank}: rows {n} evaluate_ms {t.evaluate_ms:.3f}")
for b in sorted(p.bucket_infos(), key=lambda b: -(b.start_ms + b.ms))[:8]:
    print(f"  {abi.POLICY_NAMES[b.policy]:7s} B={b.B} rows={b.rows} S<={b.max_s} C<={b.max_c} "
          f"M<={b.max_m} stream {b.stream} start {b.start_ms:.3f} ms {b.ms:.3f} end {b.start_ms + b.ms:.3f}")
raw = (C.c_int64 * (17 * n))()
p._check(p.lib.gpb_fetch_row_cycles(p.ctx, raw, 17 * n))
rows = p.rows()
worst = sorted(range(n), key=lambda i: -raw[i])[:6]
for i in worst:
    s = sc[rows[i].scenario]
    print(f"  row {i} {abi.POLICY_NAMES[s.policy]} S={-(-s.num_layers // s.layers_per_partition)} "
          f"C={s.pipelines_per_cell} M={s.num_microbatches} d={rows[i].d} feas={rows[i].feasible}: "
          f"{raw[i] / 1e3:.0f} kcyc; atlas phases casc/chain/fit/drain "
          f"{[round(x / 1e3) for x in raw[n + 16 * i: n + 16 * i + 4]]} k, scans/pairs/adm/rounds "
          f"{list(raw[n + 16 * i + 4: n + 16 * i + 8])}, drain greedy/scan/wave "
          f"{[round(x / 1e3) for x in raw[n + 16 * i + 12: n + 16 * i + 15]]} k")
