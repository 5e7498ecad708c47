"""Freeze BASELINE config-4 packing fixtures from the REFERENCE ITSELF.

    python tests/golden/make_config4_golden.py TOP_PLANS.json [n_req=20000] [ranks...]

(config4_pack_5e4.json: GOLDEN_OUT=... with n_req=50000 and ranks 52 2 1,
then the duplicate top-1000 list dropped; it is the one in config4_pack.json.)

Inputs: the config-3 top-1000 plan list by (throughput desc, row asc) as the
GPU evaluated it (tools/dump_top_plans.py; its rows are pinned bit-exact to
the reference by tests/test_gpu_scale.py / test_gpu_config2.py). For the
chosen ranks, the reference's own schedule_prefills (oracle/_ref,
bubbletea.cpp:132-222, through build_plan + run() + build_prefill_pipelines)
packs the first n_req requests of synthetic_requests(10^6, seed 42,
horizon_ms = max makespan of the 1000, default PrefillModel) — the bench's
config-4 trace — and the summary plus a digest of every request's outcome
is written to tests/golden/config4_pack.json.

The reference's search is quadratic in the trace prefix (every request
rescans all gaps of every stage GPU of every pipeline): 2*10^4 requests take
~1 h for a D=50 plan and ~4 h for a D=200 plan on one core, which is why
these are frozen here (one process per plan) instead of recomputed on the
GPU box.
"""
import json
import os
import struct
import sys
import time
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import bindings  # noqa: E402
from paper_2411_14458_b200 import abi, workloads  # noqa: E402

OUT = os.environ.get("GOLDEN_OUT", os.path.join(ROOT, "tests", "golden", "config4_pack.json"))
N_TRACE, SEED = 1_000_000, 42


def placement_digest(pl):
    """FNV-1a over every request's (accepted, pipeline, start_ns,
    ttft_overhead_ms bits), in trace order."""
    h = 1469598103934665603
    for p in pl:
        for v in (p.accepted, p.pipeline & 0xffffffff, p.start_ns & 0xffffffffffffffff,
                  struct.unpack("<Q", struct.pack("<d", p.ttft_overhead_ms))[0]):
            for i in range(8):
                h ^= (v >> (8 * i)) & 0xff
                h = (h * 1099511628211) & 0xffffffffffffffff
    return h


def main():
    top_path = sys.argv[1]
    n_req = int(sys.argv[2]) if len(sys.argv) > 2 else 20_000
    ranks = [int(x) for x in sys.argv[3:]] or [0, 2, 52, 28, 34, 87]
    top = json.load(open(top_path))["top"]
    ref = bindings.reference()
    assert ref is not None, "oracle/_ref missing: make -C oracle"
    topos, scens = workloads.config3(1_000_000, seed=2)
    tarr = abi.array(abi.Topology, topos)
    pm = abi.PrefillModel.default()
    hmax = max(t["makespan_ns"] for t in top) / 1e6
    reqs = ref.synthetic(N_TRACE, SEED, hmax, pm)[:n_req]

    def one(rank):
        t = top[rank]
        t0 = time.time()
        summ, pl = ref.pack(tarr, scens[t["scenario"]], t["d"], reqs, pm)
        dt = time.time() - t0
        print(f"rank {rank} d {t['d']} {t['policy']}: accepted {summ.accepted} in {dt:.0f} s",
              flush=True)
        return {"rank": rank, "row": t["row"], "scenario": t["scenario"], "d": t["d"],
                "policy": t["policy"], "accepted": summ.accepted, "rejected": summ.rejected,
                "horizon_ns": summ.horizon_ns, "placement_hash": summ.placement_hash,
                "utilization_before": summ.utilization_before.hex(),
                "utilization_after": summ.utilization_after.hex(),
                "placement_digest": placement_digest(pl), "ref_seconds": dt}

    with ThreadPoolExecutor(max_workers=len(ranks)) as ex:
        plans = list(ex.map(one, ranks))
    doc = {"source": "oracle/_ref schedule_prefills (unmodified reference sources)",
           "trace": {"count": N_TRACE, "seed": SEED, "horizon_ms": hmax.hex(), "prefix": n_req},
           "top": [[t["row"], t["scenario"], t["d"], t["throughput"].hex()] for t in top],
           "plans": plans}
    with open(OUT, "w") as f:
        json.dump(doc, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
