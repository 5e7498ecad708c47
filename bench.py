#!/usr/bin/env python
"""bench.py — candidate plans evaluated/sec on B200 (BASELINE.json metric).

Workload: BASELINE config 2 — the Llama-3 70B plan search over 3 DCs
[1024, 768, 512], all four policies (paper_2411_14458_b200/workloads.py).
At N GPUs the job evaluates ONE space of N x 10^4 (scenario, D) rows
(config2(N x 10^4, seed 1); N = 1 is exactly BASELINE's 10^4 plans), split
into whole-scenario shards balanced by estimated cost, one per rank (weak
scaling: 10^4 rows per GPU). A "step" evaluates every row (one evaluate_d
each, dc_select.cpp:27-66, + utilization), selects per scenario
(dc_select.cpp:99-123) and per GPU, and all-gathers the 16-byte per-GPU
winners over NCCL (N > 1): the global winner is the whatif() choice over the
whole space.

  value  plans/s with the plan tables resident in HBM, device-timed with CUDA
         events on the launching stream (K steps, L2 flushed before each),
         max over ranks.
  e2e    the same metric through the public C ABI from pinned host buffers:
         gpb_load (host validation + flatten + H2D), gpb_evaluate,
         gpb_fetch_rows (D2H of every row); two sessions alternate so a
         step's host work overlaps the previous step's evaluate (the
         evaluates stay serialised on the device).

Extra keys of the same line: config3 (10^6 plans) and config5 (the 10^7-plan
sweep), each one space sharded by cost over the ranks (strong scaling), and
bubbletea: BASELINE config 4, 10^6 synthetic prefill requests packed into the
bubbles of the 10^3 best config-3 plans (FCFS schedule_prefills), plus the
same-sample comparison against the reference's CPU packing.

--impl reference runs the reference's own CPU implementation (the reference
sources compiled into oracle/_ref, else the C port) on the host cores over
the same workload (every row of the same space, one pass with all threads).

--gpus N without torchrun relaunches itself under torch.distributed.run with
N processes (one per GPU); under torchrun, WORLD_SIZE must equal N.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidate plans evaluated/sec"
UNIT = "plans/s"
HEADLINE = ("config2: Llama-3 70B plan search, 3 DCs [1024,768,512], 4 policies, "
            "lpp/C/tp/M/ratio/multi_conn/dc_order axes")
# BASELINE config 4 as stated: 10^6 synthetic prefill requests into the
# bubbles of the 10^3 best plans (10^9 request-plan pairs per step)
BT_PLANS, BT_REQS, BT_SEED = 1000, 1_000_000, 42
# like-for-like BubbleTea sample (GPU and the reference's CPU packing on the
# same work): every one of the 10^3 plans x the first 100 requests
BT_SAMPLE_REQS = 100
GOLDEN_C4 = os.path.join(ROOT, "tests", "golden", "config4_top.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=10_000, help="rows per GPU of the headline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-bubbletea", action="store_true")
    ap.add_argument("--no-config5", action="store_true")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------- workload

def headline_space(rows_per_gpu, world):
    """One config-2 space of rows_per_gpu * world rows and its cost shards."""
    from paper_2411_14458_b200 import distributed as D, workloads
    topos, scens = workloads.config2(rows_per_gpu * world, seed=1)
    return topos, scens, D.shard_by_cost(scens, world)


def headline_config(rows_per_gpu, world, n_scen):
    """The `config` of both arms' lines (identical by construction)."""
    return {"workload": HEADLINE, "rows": rows_per_gpu * world, "rows_per_gpu": rows_per_gpu,
            "scenarios": n_scen, "space": "workloads.config2(rows, seed=1)",
            "sharding": "whole scenarios, cost-balanced (LPT) over the ranks",
            "parallelism": f"plan-space shards x{world}"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def checker():
    from oracle import bindings
    chk = bindings.reference()
    return (chk, "reference") if chk is not None else (bindings.port(), "port")


def run_cpu(topos, scens, idx, threads):
    """Time the reference's whatif() (oracle/_ref) over scenarios `idx` with
    `threads` host threads, heaviest scenario first (ctypes releases the GIL;
    the reference core is re-entrant). Returns (seconds, kind)."""
    from paper_2411_14458_b200 import abi
    chk, kind = checker()
    tarr = abi.array(abi.Topology, topos)
    todo = sorted(idx, key=lambda i: -scens[i].num_microbatches * scens[i].d_max
                  * scens[i].pipelines_per_cell)
    lock = threading.Lock()

    def worker():
        while True:
            with lock:
                if not todo:
                    return
                i = todo.pop(0)
            if kind == "reference":
                chk.whatif_count(tarr, [scens[i]])
            else:
                chk.select(tarr, scens[i])

    t0 = time.perf_counter()
    ths = [threading.Thread(target=worker) for _ in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    return time.perf_counter() - t0, kind


def cpu_one_thread(topos, scens, stride=20):
    """The reference on one host thread over every stride-th scenario."""
    idx = list(range(0, len(scens), stride))
    n = sum(scens[i].d_max for i in idx)
    dt, kind = run_cpu(topos, scens, idx, 1)
    return {"value": n / dt, "rows": n, "seconds": dt, "kind": kind,
            "sample": f"every {stride}th scenario ({len(idx)} scenarios, {n} rows), 1 thread"}


def bt_sample_plans():
    """The 10^3 config-4 plans (config-3 top by throughput desc, row asc) as
    the GPU evaluates them, frozen beside the reference-pinned packing fixture
    (tests/golden/config4_top.json): [(row, scenario, d)] and the horizon."""
    try:
        doc = json.load(open(GOLDEN_C4))
    except (OSError, ValueError):
        return None, None
    return [(r, s, d) for r, s, d, _ in doc["top"]], float.fromhex(doc["trace"]["horizon_ms"])


def bt_cpu_same_sample(threads):
    """The reference's schedule_prefills (bubbletea.cpp:132-222) on the
    like-for-like sample: every config-4 plan x the first BT_SAMPLE_REQS
    requests of the config-4 trace, all host threads."""
    from concurrent.futures import ThreadPoolExecutor
    from paper_2411_14458_b200 import abi, workloads
    from paper_2411_14458_b200.planner import synthetic_requests
    plans, hmax = bt_sample_plans()
    if plans is None:
        return None
    chk, kind = checker()
    topos, scens = workloads.config3(1_000_000, seed=2)
    tarr = abi.array(abi.Topology, topos)
    pm = abi.PrefillModel.default()
    reqs = list(synthetic_requests(BT_REQS, BT_SEED, hmax, pm)[:BT_SAMPLE_REQS]) \
        if kind == "port" else chk.synthetic(BT_REQS, BT_SEED, hmax, pm)[:BT_SAMPLE_REQS]
    order = sorted(plans, key=lambda x: -x[2])  # largest D first
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        acc = sum(ex.map(lambda p: chk.pack(tarr, scens[p[1]], p[2], reqs, pm,
                                            placements=False)[0].accepted, order))
    dt = time.perf_counter() - t0
    pairs = len(plans) * len(reqs)
    return {"value": pairs / dt, "unit": "pairs/s", "cores": threads, "kind": kind,
            "pairs": pairs, "seconds": dt, "accepted": acc,
            "sample": f"all {len(plans)} config-4 plans x the first {len(reqs)} requests of "
                      "the config-4 trace"}


# ------------------------------------------------------------- reference arm

def impl_reference(args):
    world = int(os.environ.get("WORLD_SIZE", args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    topos, scens, _ = headline_space(args.rows, world)
    n_rows = sum(s.d_max for s in scens)
    threads = os.cpu_count() or 1
    # The reference's whatif() over every row of the space with one pool of
    # all host threads (heaviest scenario first), i.e. exactly the work of K
    # steps of our arm divided into K equal parts; one pass keeps the pool
    # saturated (per-step pools idle behind each step's heaviest scenario:
    # measured 363 vs 1017 plans/s on 16 threads), so the reference is timed
    # at its best throughput.
    for _ in range(args.warmup):  # untimed (page cache, allocator, thread pool)
        run_cpu(topos, scens, list(range(min(2, len(scens)))), threads)
    total, kind = run_cpu(topos, scens, list(range(len(scens))), threads)
    times = [total / max(1, args.steps)] * max(1, args.steps)
    value = n_rows / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * total / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": headline_config(args.rows, world, len(scens)),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"the whole space: all {n_rows} rows in one timed pass "
                                   f"({len(times)} steps' worth)", "seconds": total,
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_cpu_baseline:
        one = cpu_one_thread(topos, scens)
        line["cpu_baseline"]["value_1thread"] = one["value"]
        line["cpu_baseline"]["sample_1thread"] = one["sample"]
    if not args.no_bubbletea:
        bt = bt_cpu_same_sample(threads)
        if bt is not None:
            line["bubbletea"] = {"metric": "prefills packed/sec (request-plan pairs)",
                                 "value": bt["value"], "unit": "pairs/s", "cpu_baseline": bt}
    emit(line)
    return 0


# ------------------------------------------------------------- GPU arm

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def algorithmic_ops(scens, rows):
    """Non-redundant max-plus ops per feasible row:
    gpipe/varuna 5SM+6WM, 1f1b 4SM+6WM, atlas C(4SM+6WM) (its data-dependent
    search work is not credited). W = WAN boundaries = DC blocks - 1."""
    ops = [0, 0, 0, 0]
    for r in rows:
        if r.feasible != 1:
            continue
        s = scens[r.scenario]
        S = (s.num_layers + s.layers_per_partition - 1) // s.layers_per_partition
        M = s.num_microbatches
        W = sum(1 for p in r.partitions if p > 0) - 1
        if s.policy in (0, 2):
            ops[s.policy] += 5 * S * M + 6 * W * M
        elif s.policy == 1:
            ops[1] += 4 * S * M + 6 * W * M
        else:
            ops[3] += s.pipelines_per_cell * (4 * S * M + 6 * W * M)
    return ops


def torch_device_index():
    import torch
    return torch.cuda.current_device()


def sharded(space, rank, world):
    """This rank's cost shard of a (topos, scens) space."""
    from paper_2411_14458_b200 import distributed as D
    topos, scens = space
    shard = D.shard_by_cost(scens, world)[rank]
    return topos, [scens[i] for i in shard]


def reduce_over_ranks(vals_max, vals_sum, world):
    import torch
    import torch.distributed as dist
    mx = torch.tensor(vals_max, dtype=torch.float64, device="cuda")
    sm = torch.tensor(vals_sum, dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    return [float(x) for x in mx], [float(x) for x in sm]


def space_measure(space, rank, world, reps=3, keep_rows=False):
    """A large plan space (config 3 / config 5), this rank's cost shard
    (strong scaling): device time of the evaluate launch sequence after an L2
    flush, per-bucket device times and algorithmic ops, and the e2e load
    (host flatten + H2D) + evaluate + D2H of every row into pinned memory."""
    import torch
    from paper_2411_14458_b200 import abi
    from paper_2411_14458_b200.planner import Planner
    topos, scens = sharded(space, rank, world)
    tarr, sarr = abi.array(abi.Topology, topos), abi.array(abi.Scenario, scens)
    p = Planner(torch_device_index())
    n = p.load(tarr, sarr)
    p.evaluate()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    ev, buckets = [], None
    for _ in range(reps):
        flush.fill_(1)
        torch.cuda.synchronize()
        p.evaluate()
        ev.append(p.timing().evaluate_ms)
        if buckets is None or ev[-1] == min(ev):
            buckets = p.bucket_infos()
    del flush
    # e2e: K steps of load (host flatten + H2D) + evaluate + D2H of every row
    # into pinned memory, two sessions alternating so step k+1's host work
    # overlaps step k's evaluate (the evaluates stay serialised on the device)
    p2 = Planner(torch_device_index())
    e2e_s, out = e2e_pipelined([p, p2], tarr, sarr, n, steps=3)
    rows = (abi.Row * max(1, n)).from_buffer_copy(out) if keep_rows else None
    p2.close()
    p.close()
    e2e = [e2e_s]
    return {"rows": n, "scenarios": len(scens), "evaluate_ms": statistics.median(ev),
            "e2e_s": min(e2e), "ops": sum(b.algo_ops for b in buckets), "buckets": buckets,
            "topos": topos, "scens": scens, "row_list": rows}


def e2e_pipelined(sessions, tarr, sarr, n_rows, steps, after_fetch=None):
    """End-to-end steps through the C ABI: each step loads the space (host
    flatten + H2D), evaluates it and reads every row back (D2H into pinned
    memory). Sessions alternate on their own streams: step k+1's load runs
    while step k evaluates; step k+1's evaluate waits for step k's end event,
    so the device work per step equals the device-timed loop's. Returns
    (seconds per step, the pinned rows of the last step)."""
    import torch
    from paper_2411_14458_b200 import abi
    streams = [torch.cuda.Stream() for _ in sessions]
    host = []
    for p, st in zip(sessions, streams):
        p.set_stream(st.cuda_stream)
        p.set_bucket_timing(False)
        pinned = torch.empty(max(1, n_rows) * ctypes.sizeof(abi.Row), dtype=torch.uint8,
                             pin_memory=True)
        host.append(((abi.Row * max(1, n_rows)).from_address(pinned.data_ptr()), pinned))

    def launch(i, prev_end):
        p, st = sessions[i % 2], streams[i % 2]
        p.load(tarr, sarr)
        if prev_end is not None:
            st.wait_event(prev_end)
        p.evaluate(sync=False)
        end = torch.cuda.Event()
        end.record(st)
        return end

    def finish(i):
        p = sessions[i % 2]
        rc = p.lib.gpb_fetch_rows(p.ctx, host[i % 2][0], n_rows)
        assert rc == 0, p.lib.gpb_last_error(p.ctx)
        if after_fetch is not None:
            after_fetch(i, streams[i % 2])

    def run(k):
        prev = None
        for i in range(k):
            prev = launch(i, prev)
            if i > 0:
                finish(i - 1)
        finish(k - 1)
        torch.cuda.synchronize()

    run(2)  # untimed: prepares each session's launch sequence
    t0 = time.perf_counter()
    run(steps)
    dt = (time.perf_counter() - t0) / steps
    for p in sessions:
        p.set_stream(None)
    return dt, host[(steps - 1) % 2][0]


def bucket_rooflines(buckets, peak, top=4):
    from paper_2411_14458_b200 import abi
    out = []
    for b in sorted(buckets, key=lambda b: -b.ms)[:top]:
        ach = b.algo_ops / (b.ms * 1e-3) / 1e9 if b.ms > 0 else 0.0
        out.append({"kernel": f"{abi.POLICY_NAMES[b.policy]} B={b.B} rows={b.rows} "
                              f"S<={b.max_s} M<={b.max_m}", "ms": b.ms,
                    "achieved": ach, "frac": ach / peak if peak else None})
    return out


def bt_measure(c3, rank, world):
    """BASELINE config 4: the top-BT_PLANS plans of this rank's config-3
    shard by (throughput desc, row asc), packing BT_REQS requests each;
    device time of the packing kernel and wall time of the C-ABI call
    (timelines, H2D of the trace, D2H of the summaries). Plus the same-sample
    leg: all plans x the first BT_SAMPLE_REQS requests (the reference's CPU
    packing is timed on exactly this work)."""
    import torch
    from paper_2411_14458_b200 import abi
    from paper_2411_14458_b200.planner import Planner, synthetic_requests
    topos, scens, rows = c3["topos"], c3["scens"], c3["row_list"]
    p = Planner(torch_device_index())
    p.load(abi.array(abi.Topology, topos), abi.array(abi.Scenario, scens))
    p.evaluate()
    feas = sorted(((r.throughput, i) for i, r in enumerate(rows[:c3["rows"]])
                   if r.feasible == 1), key=lambda x: (-x[0], x[1]))
    top = [i for _, i in feas[:BT_PLANS]]
    pm = abi.PrefillModel.default()
    hmax = max(rows[i].makespan_ns for i in top) / 1e6
    reqs = synthetic_requests(BT_REQS, BT_SEED, hmax, pm)
    # same-sample leg (also the warm-up of the kernels and buffers)
    sample = (abi.Request * BT_SAMPLE_REQS).from_buffer_copy(reqs, 0)
    p.pack_prefills(top, sample, pm)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p.pack_prefills(top, sample, pm)
    same_wall = time.perf_counter() - t0
    same_dev = p.timing().pack_ms / 1e3
    t0 = time.perf_counter()
    summ, _ = p.pack_prefills(top, reqs, pm)
    wall = time.perf_counter() - t0
    dev = p.timing().pack_ms / 1e3
    p.close()
    return {"top": len(top), "n_reqs": len(reqs), "dev_s": dev, "wall_s": wall,
            "accepted": sum(s.accepted for s in summ), "horizon_ms": hmax,
            "same_dev_s": same_dev, "same_wall_s": same_wall,
            "same_pairs": len(top) * BT_SAMPLE_REQS}


def impl_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2411_14458_b200 import abi, workloads
    from paper_2411_14458_b200 import distributed as pdist
    from paper_2411_14458_b200.planner import Planner

    world, rank, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = local if world > 1 else 0
    torch.cuda.set_device(device)
    stream = torch.cuda.Stream()  # one non-default stream for every launch and event
    torch.cuda.set_stream(stream)

    topos, scens_all, shards = headline_space(args.rows, world)
    scens = [scens_all[i] for i in shards[rank]]
    grows = [pdist.global_rows(scens_all, s) for s in shards]
    tarr = abi.array(abi.Topology, topos)
    sarr = abi.array(abi.Scenario, scens)
    planner = Planner(device)
    planner.set_stream(stream.cuda_stream)
    n_rows = planner.load(tarr, sarr)
    l2_flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    best_t = torch.zeros(2, dtype=torch.int64, device="cuda")   # raw gpb_best
    gathered = torch.zeros(2 * world, dtype=torch.int64, device="cuda")
    align_t = torch.zeros(1, dtype=torch.int32, device="cuda")

    def gather_best():
        if world > 1:
            # 16-byte per-GPU winner, D2D on the stream, then one NCCL all-gather
            planner.copy_best(best_t.data_ptr())
            pdist.all_gather_best(best_t, world, gathered)

    for _ in range(args.warmup):
        planner.evaluate(sync=False)
        gather_best()
    torch.cuda.synchronize()
    rows0 = planner.rows()

    # timed region: device-resident tables
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    bucket_ms = {}
    eval_ms = 0.0
    launches = 0
    clocks = ClockSampler(device)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    for k in range(args.steps):
        l2_flush.fill_(k & 0xff)  # > L2 (126 MB): every step starts cold
        # the flush completes before the step's start event (measured: a step
        # queued right behind the 256 MiB write runs ~45 us slower while the
        # write drains; the L2 is cold either way)
        torch.cuda.synchronize()
        if world > 1:
            # align the ranks' step starts (outside the timed events): a rank
            # that started early would otherwise count its wait for the
            # slowest rank inside the winner all-gather as its own step time.
            # The host barrier brings the launches close; a one-word NCCL
            # all-reduce on the stream then aligns the devices themselves
            # (its completion, which the start event follows, is the same
            # instant on every GPU up to the collective's own skew)
            dist.barrier()
            dist.all_reduce(align_t)
        starts[k].record(stream)
        planner.evaluate(sync=False)
        gather_best()
        ends[k].record(stream)
        torch.cuda.synchronize()
        t = planner.timing()
        eval_ms += t.evaluate_ms
        launches += t.launches
        for bi, b in enumerate(planner.bucket_infos()):  # per-launch device times
            bucket_ms[bi] = bucket_ms.get(bi, 0.0) + b.ms
    torch.cuda.synchronize()
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    total_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    (total_ms,), (rows_all,) = reduce_over_ranks([total_ms], [float(n_rows)], world)
    ms_per_step = total_ms / args.steps
    value = rows_all / (ms_per_step / 1000.0)

    # e2e through the C ABI from pinned host buffers: every step loads its
    # shard (host flatten + H2D), evaluates, and reads every row back (D2H).
    # Two sessions alternate so that step k+1's host flatten and H2D overlap
    # step k's evaluate; the evaluates stay serialised on the device (step
    # k+1's launch stream waits on step k's end event).
    e2e_steps = max(3, args.steps)
    planner2 = Planner(device)

    def exchange(i, st):
        if world > 1:  # the 16-byte winners, ordered after the step's evaluate
            with torch.cuda.stream(st):
                [planner, planner2][i % 2].copy_best(best_t.data_ptr())
                pdist.all_gather_best(best_t, world, gathered)

    if world > 1:
        dist.barrier()
    e2e_s, _ = e2e_pipelined([planner, planner2], tarr, sarr, n_rows, e2e_steps,
                             after_fetch=exchange)
    assert all(bytes(a) == bytes(b) for a, b in zip(rows0, planner2.rows())), \
        "second session rows differ"
    planner2.close()
    (e2e_s,), _ = reduce_over_ranks([e2e_s], [0.0], world)
    tinfo = planner.timing()

    rows1 = planner.rows()
    assert all(bytes(a) == bytes(b) for a, b in zip(rows0, rows1)), "non-deterministic rows"

    # the global winner: per-rank (throughput, local row) -> global row
    global_winner = None
    if world > 1:
        recs = []
        for r in range(world):
            thr, lrow = pdist.decode_best(gathered[2 * r: 2 * r + 2].cpu())
            recs.append((thr, grows[r][lrow] if lrow >= 0 else -1))
        global_winner = pdist.reduce_best_global(recs)

    # roofline: the dominant kernel = the bucket launch with the longest
    # average duration (it sets the step), its algorithmic max-plus ops
    # per launch over that duration; peaks from the on-box
    # microbenchmark in the kernels' representation (int64), with the FP64
    # and int32 forms beside it
    ops = algorithmic_ops(scens, rows1)
    step_ms = eval_ms / args.steps
    peaks = {k: planner.microbench(i) for i, k in enumerate(("int64", "fp64", "int32"))}
    peak = peaks["int64"]
    achieved = sum(ops) / (step_ms * 1e-3) / 1e9 if step_ms > 0 else 0.0
    binfo = planner.bucket_infos()
    kb = max(range(len(binfo)), key=lambda i: bucket_ms.get(i, 0.0))
    kb_ms = bucket_ms.get(kb, 0.0) / args.steps
    kb_ach = binfo[kb].algo_ops / (kb_ms * 1e-3) / 1e9 if kb_ms > 0 else 0.0
    kname = {0: "flush_kernel<gpipe>", 1: "onef1b_kernel", 2: "flush_kernel<varuna>",
             3: "atlas_kernel"}[binfo[kb].policy]
    kb_name = f"{kname} B={binfo[kb].B} ({abi.POLICY_NAMES[binfo[kb].policy]} bucket, " \
              f"{binfo[kb].rows} rows)"
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r02_dominant_kernel.json")) as f:
            prof = json.load(f)
        if binfo[kb].policy == prof.get("policy", 3) and binfo[kb].B == prof.get("B", 1):
            traffic = prof["dram_read_bytes"] + prof["dram_write_bytes"]
    except (OSError, KeyError, ValueError):
        pass

    # config 3 (10^6 plans) and config 5 (10^7 plans), one space each sharded
    # by cost over the ranks
    c3 = space_measure(workloads.config3(1_000_000, seed=2), rank, world,
                       keep_rows=not args.no_bubbletea)
    (c3_ms, c3_e2e), (c3_rows, c3_ops) = reduce_over_ranks(
        [c3["evaluate_ms"], c3["e2e_s"]], [float(c3["rows"]), float(c3["ops"])], world)
    bt = None
    if not args.no_bubbletea:
        bt = bt_measure(c3, rank, world)
        (bt_dev, bt_wall, bt_sdev, bt_swall), (bt_pairs, bt_spairs, bt_acc) = reduce_over_ranks(
            [bt["dev_s"], bt["wall_s"], bt["same_dev_s"], bt["same_wall_s"]],
            [float(bt["top"] * bt["n_reqs"]), float(bt["same_pairs"]), float(bt["accepted"])],
            world)
    c5 = None
    if not args.no_config5:
        c5 = space_measure(workloads.config5(10_000_000), rank, world, reps=2)
        (c5_ms, c5_e2e), (c5_rows, c5_ops) = reduce_over_ranks(
            [c5["evaluate_ms"], c5["e2e_s"]], [float(c5["rows"]), float(c5["ops"])], world)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int64", "data": "synthetic",
            "config": headline_config(args.rows, world, len(scens_all)),
            "l2": "flushed (256 MiB write) before every timed step",
            "e2e": {"value": rows_all / e2e_s, "unit": UNIT,
                    "h2d_bytes_per_step": int(tinfo.h2d_bytes),
                    "d2h_bytes_per_step": int(tinfo.d2h_bytes),
                    "sessions": 2, "device_evaluates": "serialised", "host_buffers": "pinned"},
            "gpu_launches": launches,
            "global_best": ({"throughput": global_winner[0], "row": global_winner[1]}
                            if global_winner else None),
            "device_ms": {"evaluate": eval_ms / args.steps},
            "roofline": {"bound": "alu", "kernel": kb_name,
                         "achieved": kb_ach, "peak": peak, "unit": "Gop/s",
                         "frac": kb_ach / peak if peak else None, "traffic": traffic,
                         "launch_ms": kb_ms, "ops_per_launch": binfo[kb].algo_ops,
                         "peak_source": "on-box int64 max-plus microbenchmark (gpb_microbench)",
                         "peaks_gops": peaks,
                         "traffic_source": "profiles/r02_dominant_kernel.json (ncu --set full)",
                         "step": {"achieved": achieved, "frac": achieved / peak if peak else None,
                                  "ops_per_step": sum(ops),
                                  "ops_per_policy": {abi.POLICY_NAMES[i]: ops[i]
                                                     for i in range(4)}},
                         "note": "latency-bound sequential recurrences (the longest ATLAS row "
                                 "sets the launch); see DESIGN.md §4-5"},
            "clocks": clk,
        }
        if not args.no_cpu_baseline and world == 1:
            # the reference's whatif() over the same space, all host threads
            # and 1 thread (rank 0 at N = 1 only)
            threads = os.cpu_count() or 1
            dt, kind = run_cpu(topos, scens, list(range(len(scens))), threads)
            one = cpu_one_thread(topos, scens)
            line["cpu_baseline"] = {
                "value": n_rows / dt, "unit": UNIT, "cores": threads, "kind": kind,
                "sample": f"all {n_rows} rows of this GPU's space", "seconds": dt,
                "value_1thread": one["value"], "sample_1thread": one["sample"],
                "cpu": cpu_model()}
        for key, m, ms, e2e, nrows, nops, desc in (
                ("config3", c3, c3_ms, c3_e2e, c3_rows, c3_ops,
                 "BASELINE config 3: Llama-3.1 405B plan search, 5 DCs [600,500,400,300,200], "
                 "latency x cap x multi_conn WAN grid"),
                ("config5", c5, c5_ms if c5 else 0, c5_e2e if c5 else 0, c5_rows if c5 else 0,
                 c5_ops if c5 else 0,
                 "BASELINE config 5: full sweep, random topologies of 2-8 DCs (64-1024 GPUs "
                 "each), GPT-A/GPT-B/Llama-3 70B/Llama-3.1 405B, microbatches 4-256, all axes")):
            if m is None:
                continue
            ach = nops / (ms * 1e-3) / 1e9
            line[key] = {
                "metric": METRIC, "value": nrows / (ms * 1e-3), "unit": UNIT,
                "scaling": "strong", "workload": f"{desc}; {int(nrows)} rows, one space sharded "
                                                 f"by cost over {world} GPU(s)",
                "ms": ms, "e2e": {"value": nrows / e2e, "unit": UNIT, "seconds": e2e,
                                  "includes": "host flatten + H2D of the tables, evaluate, "
                                              "D2H of every row into pinned memory"},
                "roofline": {"bound": "alu", "achieved": ach, "peak": peak, "unit": "Gop/s",
                             "frac": ach / peak if peak else None, "ops_per_step": nops,
                             "buckets_rank0": bucket_rooflines(m["buckets"], peak)},
                "l2": "flushed (256 MiB write) before every timed evaluate"}
        if bt is not None:
            line["bubbletea"] = {
                "metric": "prefills packed/sec (request-plan pairs)", "value": bt_pairs / bt_dev,
                "unit": "pairs/s", "e2e": bt_pairs / bt_wall,
                "config": {"workload": "config4: top plans of config3 (Llama-3.1 405B, "
                           "5 DCs [600,500,400,300,200]) by throughput, one synthetic trace "
                           "(seed 42) over the largest makespan, FCFS schedule_prefills",
                           "plans_per_gpu": bt["top"], "requests": bt["n_reqs"],
                           "horizon_ms": bt["horizon_ms"]},
                "pairs_per_step": int(bt_pairs), "accepted": int(bt_acc),
                "device_s": bt_dev, "wall_s": bt_wall,
                "same_sample": {"pairs": int(bt_spairs), "value": bt_spairs / bt_sdev,
                                "e2e": bt_spairs / bt_swall, "unit": "pairs/s",
                                "sample": f"all {bt['top']} plans x the first {BT_SAMPLE_REQS} "
                                          "requests of the trace"}}
            if not args.no_cpu_baseline and world == 1:
                cb = bt_cpu_same_sample(os.cpu_count() or 1)
                if cb is not None:
                    line["bubbletea"]["cpu_baseline"] = cb
        emit(line)
    planner.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------- launcher

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn(args):
    """--gpus N outside torchrun: relaunch under torch.distributed.run with N
    processes and pass the JSON line of rank 0 through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    proc = subprocess.run(cmd, stdout=subprocess.PIPE, text=True)
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    if proc.returncode != 0 or not lines:
        sys.stderr.write(proc.stdout)
        sys.stderr.write(f"bench.py: torchrun with {args.gpus} ranks failed (rc "
                         f"{proc.returncode})\n")
        return proc.returncode or 1
    emit(json.loads(lines[-1]))
    return 0


def _stdout_for_json_only():
    """The driver reads exactly one JSON line from stdout: libraries (NCCL's
    version banner, warnings) write to fd 1 too, so fd 1 is pointed at
    stderr and the JSON goes through a private duplicate of the original."""
    global _JSON_OUT
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)


_JSON_OUT = None


def emit(line):
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    _stdout_for_json_only()
    args = parse()
    env_world = os.environ.get("WORLD_SIZE")
    if args.impl == "reference":
        return impl_reference(args)
    if env_world is None and args.gpus > 1:
        return spawn(args)
    if env_world is not None and int(env_world) != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}\n")
        return 2
    return impl_ours(args)


if __name__ == "__main__":
    sys.exit(main())
