"""Per-row clock64 cost of the evaluation kernels on a BASELINE workload,
aggregated by (policy, S, C, M): where the device time goes."""
import collections
import json
import sys

sys.path.insert(0, ".")
from paper_2411_14458_b200 import abi, workloads  # noqa: E402
from paper_2411_14458_b200.planner import Planner  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "config2"
topos, scens = getattr(workloads, cfg)(**({"n_rows": int(sys.argv[3])} if len(sys.argv) > 3 else {}))
p = Planner(0)
p.set_profile(True)
n = p.load(abi.array(abi.Topology, topos), abi.array(abi.Scenario, scens))
p.evaluate()
p.evaluate()
rows = p.rows()
import ctypes as C
raw = (C.c_int64 * (17 * n))()
p._check(p.lib.gpb_fetch_row_cycles(p.ctx, raw, 17 * n))
cyc = list(raw[:n])
phase = [list(raw[n + 16 * i: n + 16 * i + 16]) for i in range(n)]
t = p.timing()
agg = collections.defaultdict(lambda: [0, 0, 0, [0] * 16])
for r, c, ph in zip(rows[:n], cyc, phase):
    s = scens[r.scenario]
    S = (s.num_layers + s.layers_per_partition - 1) // s.layers_per_partition
    key = (abi.POLICY_NAMES[s.policy], S, s.pipelines_per_cell, s.num_microbatches, r.feasible)
    a = agg[key]
    a[0] += 1
    a[1] += c
    a[2] = max(a[2], c)
    if s.policy == 3:
        for k in range(16):
            a[3][k] += ph[k]
tot = sum(v[1] for v in agg.values())
by_pol = collections.Counter()
for k, v in agg.items():
    by_pol[k[0]] += v[1]
print("cycles by policy:", {k: f"{100 * v / tot:.1f}%" for k, v in by_pol.most_common()})
print(json.dumps({"evaluate_ms": t.evaluate_ms, "policy_ms": list(t.policy_ms)}))
print("policy S C M feas | rows  sum_Mcyc  share  max_kcyc")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    ph = [round(x / max(1, v[1]) * 100) for x in v[3][:4]] + [round(x / v[0]) for x in v[3][4:8]] \
        + [round(x / max(1, v[1]) * 100) for x in v[3][8:12]] \
        + [round(x / max(1, v[1]) * 100) for x in v[3][12:15]] + [round(v[3][15] / v[0])]
    print(*k, "|", v[0], round(v[1] / 1e6, 2), f"{100 * v[1] / tot:.1f}%", round(v[2] / 1e3, 1),
          "phases% casc/chain/fit/drain + per-row scans/pairs/adm/rounds + casc% setup/loads/scan/commit + drain% greedy/scan/wave + wave steps", ph)
