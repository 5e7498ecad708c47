"""Per-bucket launch timeline of one gpb_evaluate on a BASELINE workload
(which bucket kernel sets the step time).

    python tools/buckets.py [config2] [reps] [flush]

flush=1 writes 256 MiB (> L2) before the last evaluate, as bench.py does.
"""
import sys

sys.path.insert(0, ".")
from paper_2411_14458_b200 import abi, workloads  # noqa: E402
from paper_2411_14458_b200.planner import Planner  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "config2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
topos, scens = getattr(workloads, cfg)()
p = Planner(0)
n = p.load(abi.array(abi.Topology, topos), abi.array(abi.Scenario, scens))
flush = len(sys.argv) > 3 and sys.argv[3] == "1"
for _ in range(reps):
    if flush:
        import torch
        buf = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()
        del buf
    p.evaluate()
t = p.timing()
print(cfg, "rows", n, "evaluate_ms", round(t.evaluate_ms, 3), "kernels_ms",
      round(t.timing_kernels_ms, 3), "select_ms", round(t.select_ms, 3))
print("policy   B  rows  maxS maxC maxM stream  start_ms   ms   end_ms")
for b in sorted(p.bucket_infos(), key=lambda b: -(b.start_ms + b.ms)):
    print(f"{abi.POLICY_NAMES[b.policy]:7s} {b.B:2d} {b.rows:5d} {b.max_s:5d} {b.max_c:4d} "
          f"{b.max_m:4d} {b.stream:6d} {b.start_ms:8.3f} {b.ms:7.3f} {b.start_ms + b.ms:7.3f}")
