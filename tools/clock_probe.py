"""Does the nvidia-smi clock sampler perturb the config-2 step? Times K
flushed evaluates with no sampler, with the sampler just started, and with
the sampler started 1 s earlier.

    python tools/clock_probe.py [K=20]
"""
import subprocess
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2411_14458_b200 import abi, workloads  # noqa: E402
from paper_2411_14458_b200.planner import Planner  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
topos, scens = workloads.config2()
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
p = Planner(0)
p.set_stream(st.cuda_stream)
p.load(abi.array(abi.Topology, topos), abi.array(abi.Scenario, scens))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    p.evaluate(sync=False)
torch.cuda.synchronize()


def timed(sync_flush=False, own=False):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(K)]
    heavy = 0.0
    for k in range(K):
        flush.fill_(k & 0xff)
        if sync_flush:
            torch.cuda.synchronize()
        ev[k][0].record(st)
        p.evaluate(sync=False)
        ev[k][1].record(st)
        torch.cuda.synchronize()
        heavy += max(b.ms for b in p.bucket_infos())
    return sum(a.elapsed_time(b) for a, b in ev) / K, heavy / K


def smi():
    return subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm",
                             "--format=csv,noheader", "-lms", "100"],
                            stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)


for rep in range(2):
    print("no sampler     ", timed())
    print("sync after flush", timed(sync_flush=True))
q = smi()
print("sampler started", timed())
q.terminate()
q.wait()
st = torch.cuda.Stream(priority=-1)
torch.cuda.set_stream(st)
p.set_stream(st.cuda_stream)
for rep in range(2):
    print("high-priority stream ", timed())
    print("high-priority stream, sync after flush", timed(sync_flush=True))
