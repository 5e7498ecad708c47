"""BASELINE config 5 throughput on one GPU: evaluate a config-5 plan space
(10^7 rows by default, or a prefix of it) and report plans/s (device time of
the evaluate launch sequence) plus the load time.

    python tools/config5_bench.py [rows=10000000] [reps=2]
"""
import sys
import time

sys.path.insert(0, ".")
from paper_2411_14458_b200 import abi, workloads  # noqa: E402
from paper_2411_14458_b200.planner import Planner  # noqa: E402

n_rows = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
t0 = time.perf_counter()
topos, scens = workloads.config5(n_rows)
t1 = time.perf_counter()
p = Planner(0)
tarr, sarr = abi.array(abi.Topology, topos), abi.array(abi.Scenario, scens)
t2 = time.perf_counter()
n = p.load(tarr, sarr)
p.evaluate()
t3 = time.perf_counter()
print(f"config5: {n} rows, {len(scens)} scenarios; generate {t1 - t0:.1f} s, ctypes {t2 - t1:.1f} s, "
      f"first load+evaluate {t3 - t2:.2f} s")
for _ in range(reps):
    p.evaluate()
    t = p.timing()
    print(f"evaluate {t.evaluate_ms:.1f} ms -> {n / (t.evaluate_ms * 1e-3):.3e} plans/s")
best = p.best()
print("best row", best.row, "throughput", best.throughput)
for b in sorted(p.bucket_infos(), key=lambda b: -(b.start_ms + b.ms))[:6]:
    print(f"  {abi.POLICY_NAMES[b.policy]:7s} B={b.B} rows={b.rows} S<={b.max_s} C<={b.max_c} "
          f"M<={b.max_m} start {b.start_ms:.1f} ms, {b.ms:.1f} ms")
