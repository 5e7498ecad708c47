"""Evaluate one BASELINE plan space `reps` times (profiling driver).

    python tools/run_eval.py config2 [reps] [policy:S:C:M]   # optional filter
"""
import sys

sys.path.insert(0, ".")
from paper_2411_14458_b200 import abi, workloads  # noqa: E402
from paper_2411_14458_b200.planner import Planner  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "config2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
topos, scens = getattr(workloads, cfg)()
if len(sys.argv) > 3:
    pol, S, C, M = sys.argv[3].split(":")
    keep = [s for s in scens if abi.POLICY_NAMES[s.policy] == pol and
            (s.num_layers + s.layers_per_partition - 1) // s.layers_per_partition == int(S) and
            s.pipelines_per_cell == int(C) and s.num_microbatches == int(M)]
    scens = keep
p = Planner(0)
n = p.load(abi.array(abi.Topology, topos), abi.array(abi.Scenario, scens))
for _ in range(reps):
    p.evaluate()
t = p.timing()
print(cfg, "scenarios", len(scens), "rows", n, "evaluate_ms", round(t.evaluate_ms, 3), "policy_ms",
      [round(x, 3) for x in t.policy_ms])
