"""A/B of the headline shard balance: every rank's shard of config2(N x 10^4)
evaluated on one GPU under the cost model with an extra per-row constant
(cycles), printing each rank's evaluate time and the max over ranks.

    python tools/shard_balance.py N [per_row ...]
"""
import sys

sys.path.insert(0, ".")
from paper_2411_14458_b200 import abi, workloads, distributed as D  # noqa: E402
from paper_2411_14458_b200.planner import Planner  # noqa: E402

N = int(sys.argv[1])
extras = [float(x) for x in sys.argv[2:]] or [0.0]
topos, scens = workloads.config2(10_000 * N, seed=1)
tarr = abi.array(abi.Topology, topos)
p = Planner(0)
base = D.row_cost
for extra in extras:
    D.row_cost = lambda sc, e=extra: base(sc) + e
    shards = D.shard_by_cost(scens, N)
    ms = []
    for r in range(N):
        p.load(tarr, abi.array(abi.Scenario, [scens[i] for i in shards[r]]))
        for _ in range(5):
            p.evaluate()
        ms.append(p.timing().evaluate_ms)
    print(f"N={N} per-row +{extra:g}: max {max(ms):.3f} ms, ranks {[round(x, 3) for x in ms]}",
          flush=True)
D.row_cost = base
