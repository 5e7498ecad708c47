"""Where the e2e step goes: gpb_load (host flatten + H2D), gpb_evaluate,
gpb_fetch_rows (D2H) wall times on a BASELINE workload.

    python tools/e2e_breakdown.py [config2|config3|config5] [K=20]
"""
import sys
import time

sys.path.insert(0, ".")
from paper_2411_14458_b200 import abi, workloads  # noqa: E402
from paper_2411_14458_b200.planner import Planner  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "config2"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
topos, scens = getattr(workloads, cfg)()
tarr = abi.array(abi.Topology, topos)
sarr = abi.array(abi.Scenario, scens)
p = Planner(0)
n = p.load(tarr, sarr)
import ctypes, torch
pinned = torch.empty(n * ctypes.sizeof(abi.Row), dtype=torch.uint8, pin_memory=True)
out = (abi.Row * n).from_address(pinned.data_ptr())
for _ in range(3):
    p.load(tarr, sarr)
    p.evaluate()
    p.lib.gpb_fetch_rows(p.ctx, out, n)
tl = te = tf = 0.0
for _ in range(K):
    t0 = time.perf_counter()
    p.load(tarr, sarr)
    t1 = time.perf_counter()
    p.evaluate(sync=False)
    t2 = time.perf_counter()
    p.lib.gpb_fetch_rows(p.ctx, out, n)
    t3 = time.perf_counter()
    tl += t1 - t0
    te += t2 - t1
    tf += t3 - t2
print(f"load {1e3 * tl / K:.3f} ms  evaluate(launch) {1e3 * te / K:.3f} ms  "
      f"fetch(wait+D2H) {1e3 * tf / K:.3f} ms  device evaluate {p.timing().evaluate_ms:.3f} ms")
