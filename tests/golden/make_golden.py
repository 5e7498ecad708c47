"""Generate the golden fixtures from the compiled reference (oracle/_ref).

Run in a container where /root/reference exists (make -C oracle builds
oracle/_ref/libgeopipe_ref.so from its sources). The fixtures freeze the
reference's own outputs — select() rows, report() utilization on run(),
extract_bubbles() lists, schedule_prefills() summaries and placements — for
seeded plan spaces, so parity tests on the GPU box do not depend on the
reference tree. Doubles are stored as float.hex() (bit-exact).

    python tests/golden/make_golden.py
"""
import ctypes as C
import hashlib
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import bindings  # noqa: E402
from paper_2411_14458_b200 import abi  # noqa: E402
from tests.instances import random_space  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def struct_dict(s):
    d = {}
    for name, ctype in s._fields_:
        v = getattr(s, name)
        if hasattr(v, "__len__") and not isinstance(v, (bytes, str)):
            v = [list(x) if hasattr(x, "__len__") else x for x in v]
        d[name] = v
    return d


def hx(x):
    return float(x).hex()


def main():
    ref = bindings.reference()
    if ref is None:
        raise SystemExit("oracle/_ref/libgeopipe_ref.so missing: make -C oracle")
    rutil = ref.lib.ref_utilization
    rutil.restype = C.c_int
    rutil.argtypes = [C.POINTER(abi.Topology), C.POINTER(abi.Scenario), C.c_int32,
                      C.c_int32, C.POINTER(C.c_double)]
    spaces = []
    for seed, n, wide in ((1234, 80, False), (99, 60, True), (7, 40, True)):
        topos, scens = random_space(seed, n, wide)
        sp = {"seed": seed, "wide": wide, "topologies": [struct_dict(t) for t in topos],
              "scenarios": [], "bubbles": [], "packs": []}
        rng = random.Random(seed)
        for i, sc in enumerate(scens):
            try:
                rows, chosen, used = ref.select(topos, sc)
            except bindings.CheckerError as e:
                sp["scenarios"].append({"scenario": struct_dict(sc), "error": e.rc})
                continue
            out_rows = []
            for r in rows:
                u = C.c_double(0.0)
                if r.feasible:
                    assert rutil(topos, C.byref(sc), r.d, 1, C.byref(u)) == 0
                out_rows.append([r.d, r.feasible, r.chosen, hx(r.pp_time_ms),
                                 hx(r.allreduce_time_ms), hx(r.total_time_ms),
                                 hx(r.throughput), list(r.partitions), hx(u.value)])
            sp["scenarios"].append({"scenario": struct_dict(sc), "chosen_d": chosen,
                                    "gpus_used": used, "rows": out_rows})
            feas = [r for r in rows if r.feasible and
                    r.d * sc.pipelines_per_cell * sc.num_layers <= 1500]
            if feas and rng.random() < 0.35:
                r = rng.choice(feas[:4])
                b = ref.bubbles(topos, sc, r.d)
                sp["bubbles"].append({"scenario": i, "d": r.d, "horizon": 0, "bubbles": b})
                pm = abi.PrefillModel.default(inference_layers=rng.choice([8, 3]))
                reqs = ref.saturating(topos, sc, r.d, pm)[:400]
                summ, pl = ref.pack(topos, sc, r.d, reqs, pm)
                digest = hashlib.sha256(json.dumps(
                    [[p.accepted, p.pipeline, p.start_ns, hx(p.ttft_overhead_ms)] for p in pl]
                ).encode()).hexdigest()
                sp["packs"].append({
                    "scenario": i, "d": r.d, "inference_layers": pm.inference_layers,
                    "requests": [[q.id, q.tokens, hx(q.arrival_ms)] for q in reqs],
                    "summary": [hx(summ.utilization_before), hx(summ.utilization_after),
                                summ.accepted, summ.rejected, summ.horizon_ns,
                                str(summ.placement_hash)],
                    "placements_sha256": digest})
        spaces.append(sp)
    with open(os.path.join(OUT, "reference_spaces.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "source": "oracle/_ref/libgeopipe_ref.so (reference src/*.cpp, unmodified)",
                   "spaces": spaces}, f, separators=(",", ":"))
    print("wrote", os.path.join(OUT, "reference_spaces.json"))


if __name__ == "__main__":
    main()
