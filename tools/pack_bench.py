"""BubbleTea at BASELINE config-4 scale: evaluate a plan space, take its top-K
feasible plans by (throughput desc, row asc), pack one shared synthetic
request trace (synthetic_requests, bubbletea.cpp:269-284; horizon = the
largest makespan of the K) into every plan's bubbles, and report
request-plan pairs/s.

    python tools/pack_bench.py [config3|config2] [K=1000] [R=1000000] [reps=2]
"""
import sys
import time

sys.path.insert(0, ".")
from paper_2411_14458_b200 import abi, workloads  # noqa: E402
from paper_2411_14458_b200.planner import Planner, synthetic_requests  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "config3"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
R = int(sys.argv[3]) if len(sys.argv) > 3 else 1_000_000
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
topos, scens = getattr(workloads, cfg)()
p = Planner(0)
n = p.load(abi.array(abi.Topology, topos), abi.array(abi.Scenario, scens))
t0 = time.perf_counter()
p.evaluate()
t1 = time.perf_counter()
rows = p.rows()
feas = [(r.throughput, i) for i, r in enumerate(rows[:n]) if r.feasible == 1]
feas.sort(key=lambda x: (-x[0], x[1]))
top = [i for _, i in feas[:K]]
hmax = max(rows[i].makespan_ns for i in top) / 1e6
pm = abi.PrefillModel.default()
reqs = synthetic_requests(R, 42, hmax, pm)
pol = {}
for i in top:
    k = abi.POLICY_NAMES[scens[rows[i].scenario].policy]
    pol[k] = pol.get(k, 0) + 1
print(f"{cfg}: rows {n} evaluate {1e3 * (t1 - t0):.1f} ms; top {len(top)} plans {pol}; "
      f"requests {R} horizon {hmax:.1f} ms")
for _ in range(reps):
    t0 = time.perf_counter()
    summ, _ = p.pack_prefills(top, reqs, pm)
    dt = time.perf_counter() - t0
    acc = sum(s.accepted for s in summ)
    t = p.timing()
    print(f"pack: wall {dt * 1e3:.1f} ms device {t.pack_ms:.1f} ms; accepted {acc} of "
          f"{len(top) * R} request-plan pairs; {len(top) * R / (t.pack_ms * 1e-3):.3e} pairs/s")
