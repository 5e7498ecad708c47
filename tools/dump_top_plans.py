"""Dump the top-K feasible plans of a plan space by (throughput desc, row asc)
as evaluated on the GPU: the plan list BASELINE config 4 packs into (used to
freeze tests/golden/config4_pack.json with the reference's own
schedule_prefills, tests/golden/make_config4_golden.py).

    python tools/dump_top_plans.py [config3] [K=1000] [out=gpurun_out/top_plans.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_14458_b200 import abi, workloads  # noqa: E402
from paper_2411_14458_b200.planner import Planner  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "config3"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
out = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/top_plans.json"
topos, scens = getattr(workloads, cfg)()
p = Planner(0)
n = p.load(abi.array(abi.Topology, topos), abi.array(abi.Scenario, scens))
p.evaluate()
rows = p.rows()
feas = sorted(((r.throughput, i) for i, r in enumerate(rows[:n]) if r.feasible == 1),
              key=lambda x: (-x[0], x[1]))
top = []
for thr, i in feas[:K]:
    r = rows[i]
    top.append({"row": i, "scenario": r.scenario, "d": r.d, "throughput": r.throughput,
                "makespan_ns": r.makespan_ns, "policy": abi.POLICY_NAMES[scens[r.scenario].policy],
                "C": scens[r.scenario].pipelines_per_cell,
                "S": -(-scens[r.scenario].num_layers // scens[r.scenario].layers_per_partition)})
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
with open(out, "w") as f:
    json.dump({"config": cfg, "rows": n, "K": K, "top": top}, f)
print(f"{cfg}: {n} rows, top {len(top)} written to {out}; max d {max(t['d'] for t in top)}")
p.close()
