"""Steady-state of the bench's two-session e2e loop: per-step wall time over
K steps, and the host time of gpb_load / gpb_evaluate (launch) / fetch wait."""
import ctypes
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_2411_14458_b200 import abi, workloads  # noqa: E402
from paper_2411_14458_b200.planner import Planner  # noqa: E402

topos, scens = workloads.config2()
tarr = abi.array(abi.Topology, topos)
sarr = abi.array(abi.Scenario, scens)
ps = [Planner(0), Planner(0)]
ss = [torch.cuda.Stream(), torch.cuda.Stream()]
bufs = []
for p, s in zip(ps, ss):
    p.set_stream(s.cuda_stream)
    p.set_bucket_timing(False)
    n = p.load(tarr, sarr)
    pin = torch.empty(n * ctypes.sizeof(abi.Row), dtype=torch.uint8, pin_memory=True)
    bufs.append(((abi.Row * n).from_address(pin.data_ptr()), pin))
acc = {"load": 0.0, "launch": 0.0, "fetch": 0.0}


def run(k):
    prev = None
    for i in range(k + 1):
        if i < k:
            p, s = ps[i % 2], ss[i % 2]
            t0 = time.perf_counter()
            p.load(tarr, sarr)
            t1 = time.perf_counter()
            if prev is not None:
                s.wait_event(prev)
            p.evaluate(sync=False)
            prev = torch.cuda.Event()
            prev.record(s)
            t2 = time.perf_counter()
            acc["load"] += t1 - t0
            acc["launch"] += t2 - t1
        if i > 0:
            q = ps[(i - 1) % 2]
            t3 = time.perf_counter()
            q.lib.gpb_fetch_rows(q.ctx, bufs[(i - 1) % 2][0], n)
            acc["fetch"] += time.perf_counter() - t3
    torch.cuda.synchronize()


run(6)
for k in (10, 20, 100):
    for key in acc:
        acc[key] = 0.0
    t0 = time.perf_counter()
    run(k)
    dt = time.perf_counter() - t0
    print(f"K={k}: {1e3 * dt / k:.3f} ms/step ({n * k / dt / 1e6:.2f} M plans/s)  " +
          "  ".join(f"{a} {1e3 * v / k:.3f} ms" for a, v in acc.items()))
