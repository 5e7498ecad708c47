"""Isolate the config-2 critical ATLAS row's scenario (the one that sets the
headline step) and evaluate it alone, for an ncu source-level capture.

    python tools/critical_row.py [reps=3] [scenario]

With a scenario index, skips the search pass (one process = only the
isolated evaluates, for `ncu -k regex:atlas_kernel`).
"""
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_2411_14458_b200 import abi, workloads  # noqa: E402
from paper_2411_14458_b200.planner import Planner  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
topos, scens = workloads.config2()
if len(sys.argv) > 2:
    si = int(sys.argv[2])
else:
    p = Planner(0)
    p.set_profile(True)
    n = p.load(abi.array(abi.Topology, topos), abi.array(abi.Scenario, scens))
    p.evaluate()
    raw = (C.c_int64 * (17 * n))()
    p._check(p.lib.gpb_fetch_row_cycles(p.ctx, raw, 17 * n))
    rows = p.rows()
    crit = max(range(n), key=lambda i: raw[i])
    si = rows[crit].scenario
    p.close()
    print(f"critical row {crit} scenario {si} ({raw[crit] / 1e3:.0f} kcyc)", flush=True)
sc = type(scens[si]).from_buffer_copy(scens[si])
ti = sc.topology
sc.topology = 0
q = Planner(0)
q.load(abi.array(abi.Topology, [topos[ti]]), abi.array(abi.Scenario, [sc]))
for _ in range(reps):
    q.evaluate()
t = q.timing()
print("alone: evaluate_ms", round(t.evaluate_ms, 3),
      [(b.B, b.rows, round(b.ms, 3)) for b in q.bucket_infos()])
if len(sys.argv) > 3:  # per-phase profile of the slowest row of the isolated scenario
    q.set_profile(True)
    q.load(abi.array(abi.Topology, [topos[ti]]), abi.array(abi.Scenario, [sc]))
    q.evaluate()
    q.evaluate()
    n = q.rows().__len__()
    raw = (C.c_int64 * (17 * n))()
    q._check(q.lib.gpb_fetch_row_cycles(q.ctx, raw, 17 * n))
    i = max(range(n), key=lambda k: raw[k])
    ph = list(raw[n + 16 * i: n + 16 * i + 16])
    names = ["casc", "chain", "fit", "drain", "scans", "pairs", "adm", "rounds",
             "c_setup", "c_loads", "c_scan", "c_commit", "d_greedy", "d_scan", "d_wave", "wsteps"]
    print(f"row d={i + 1}: {raw[i] / 1e3:.0f} kcyc", dict(zip(names, ph)))
