"""Bucket timeline of one rank's cost shard of a large BASELINE space
(config3 / config5, strong scaling over N GPUs) on one GPU, and the slowest
rows of each of its longest buckets (which rows bound a bucket's makespan).

    python tools/space_shard_rows.py config3|config5 N [rank] [reps]
"""
import collections
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_2411_14458_b200 import abi, workloads, distributed as D  # noqa: E402
from paper_2411_14458_b200.planner import Planner  # noqa: E402

cfg = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rank = int(sys.argv[3]) if len(sys.argv) > 3 else 0
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
topos, scens = workloads.config3(1_000_000, seed=2) if cfg == "config3" else workloads.config5()
shard = D.shard_by_cost(scens, N)[rank]
sc = [scens[i] for i in shard]
p = Planner(0)
tarr, sarr = abi.array(abi.Topology, topos), abi.array(abi.Scenario, sc)
n = p.load(tarr, sarr)
for _ in range(reps):
    p.evaluate()
t = p.timing()
print(f"{cfg} N={N} rank {rank}: rows {n} evaluate_ms {t.evaluate_ms:.3f}", flush=True)
for b in sorted(p.bucket_infos(), key=lambda b: -(b.start_ms + b.ms))[:10]:
    print(f"  {abi.POLICY_NAMES[b.policy]:7s} B={b.B} rows={b.rows} S<={b.max_s} C<={b.max_c} "
          f"M<={b.max_m} stream {b.stream} start {b.start_ms:.3f} ms {b.ms:.3f} end {b.start_ms + b.ms:.3f}")
if len(sys.argv) > 5 or "GPB_NO_ROWS" in __import__("os").environ: sys.exit(0)
p.set_profile(True)
p.load(tarr, sarr)
p.evaluate()
raw = (C.c_int64 * (17 * n))()
p._check(p.lib.gpb_fetch_row_cycles(p.ctx, raw, 17 * n))
rows = p.rows()


def shape(s):
    S = -(-s.num_layers // s.layers_per_partition)
    return S, s.pipelines_per_cell, s.num_microbatches


def est(s):  # the host bucket cost model (host.cu gpb_load)
    S, Cc, M = shape(s)
    return Cc * M * (2000.0 * Cc + 250.0 * S) if s.policy == 3 else 20.0 * M * S


by_pol = collections.defaultdict(list)
for i in range(n):
    if rows[i].feasible == 1:
        by_pol[sc[rows[i].scenario].policy].append(i)
for pol, lst in sorted(by_pol.items()):
    lst.sort(key=lambda i: -raw[i])
    print(f"{abi.POLICY_NAMES[pol]}: {len(lst)} feasible rows, cycles p50 "
          f"{raw[lst[len(lst) // 2]] / 1e3:.0f} k, p99 {raw[lst[len(lst) // 100]] / 1e3:.0f} k, max "
          f"{raw[lst[0]] / 1e3:.0f} k")
    for i in lst[:6]:
        s = sc[rows[i].scenario]
        S, Cc, M = shape(s)
        print(f"    row {i} S={S} C={Cc} M={M} L={s.mem_limit} d={rows[i].d}: "
              f"{raw[i] / 1e6:.2f} Mcyc (est {est(s) / 1e6:.2f} M)")
