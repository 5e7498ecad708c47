"""Evaluate a BASELINE plan space `reps` times (a short command for ncu).

    python tools/run_eval.py [config2] [reps=2]
"""
import sys

sys.path.insert(0, ".")
from paper_2411_14458_b200 import abi, workloads  # noqa: E402
from paper_2411_14458_b200.planner import Planner  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "config2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
topos, scens = getattr(workloads, cfg)()
p = Planner(0)
n = p.load(abi.array(abi.Topology, topos), abi.array(abi.Scenario, scens))
for _ in range(reps):
    p.evaluate()
print(cfg, "rows", n, "evaluate_ms", round(p.timing().evaluate_ms, 3))
