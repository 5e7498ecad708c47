"""BubbleTea config-4 packing: device time of the full 10^6-request pack in
three orders (fresh, after a 10^4-request warm-up, repeated) with the SM
clock sampled, to separate state effects from box effects."""
import subprocess
import sys
import time

sys.path.insert(0, ".")
from paper_2411_14458_b200 import abi, workloads  # noqa: E402
from paper_2411_14458_b200.planner import Planner, synthetic_requests  # noqa: E402

topos, scens = workloads.config3()
p = Planner(0)
n = p.load(abi.array(abi.Topology, topos), abi.array(abi.Scenario, scens))
p.evaluate()
rows = p.rows()
feas = sorted(((r.throughput, i) for i, r in enumerate(rows[:n]) if r.feasible == 1),
              key=lambda x: (-x[0], x[1]))
top = [i for _, i in feas[:1000]]
pm = abi.PrefillModel.default()
reqs = synthetic_requests(1_000_000, 42, max(rows[i].makespan_ns for i in top) / 1e6, pm)
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                        "--format=csv,noheader", "-lms", "500"], stdout=subprocess.PIPE, text=True)
for label, warm in (("fresh", 0), ("after 1e4 warm-up", 10_000), ("repeat", 0)):
    if warm:
        p.pack_prefills(top, (abi.Request * warm).from_buffer_copy(reqs, 0), pm)
    t0 = time.perf_counter()
    summ, _ = p.pack_prefills(top, reqs, pm)
    print(f"{label}: device {p.timing().pack_ms:.0f} ms wall {1e3 * (time.perf_counter() - t0):.0f} ms "
          f"accepted {sum(s.accepted for s in summ)}", flush=True)
smi.terminate()
out = smi.communicate()[0].strip().splitlines()
print("clock samples:", len(out), out[:: max(1, len(out) // 12)])
