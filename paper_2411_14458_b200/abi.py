"""ctypes mirror of include/geopipe_batch.h (the C-ABI boundary).

Plain structs only: this module has no torch dependency and is shared by the
host-side Python mirror (``paper_2411_14458_b200.planner``), the tests and
bench.py.
"""
from __future__ import annotations

import ctypes as C

GPB_OK, GPB_ERROR, GPB_CONFIG_ERROR, GPB_INFEASIBLE = 0, 1, 2, 3
GPB_MAX_DC = 8
GPB_MAX_TCP = 8

GPIPE, ONEF1B, VARUNA, ATLAS = 0, 1, 2, 3
POLICIES = {"gpipe": GPIPE, "1f1b": ONEF1B, "varuna": VARUNA, "atlas": ATLAS}
POLICY_NAMES = {v: k for k, v in POLICIES.items()}


class Topology(C.Structure):
    """ClusterTopology (reference topology.h:12-40)."""

    _fields_ = [
        ("n_dc", C.c_int32),
        ("gpu_count", C.c_int32 * GPB_MAX_DC),
        ("intra_bw", C.c_double * GPB_MAX_DC),
        ("latency_ms", (C.c_double * GPB_MAX_DC) * GPB_MAX_DC),
        ("pair_bw_cap", C.c_double),
        ("n_tcp", C.c_int32),
        ("pad_", C.c_int32),
        ("tcp_latency_ms", C.c_double * GPB_MAX_TCP),
        ("tcp_bw", C.c_double * GPB_MAX_TCP),
    ]


class Scenario(C.Structure):
    """SelectionInput + ModelSpec + ComputeProfile + SchedulerOptions
    (reference dc_select.h:18-30, workload.h:12-52, scheduler.h:11-16)."""

    _fields_ = [
        ("topology", C.c_int32),
        ("policy", C.c_int32),
        ("num_layers", C.c_int32),
        ("layers_per_partition", C.c_int32),
        ("num_microbatches", C.c_int32),
        ("bytes_per_element", C.c_int32),
        ("hidden", C.c_int64),
        ("seq_len", C.c_int64),
        ("microbatch", C.c_int64),
        ("params_per_layer", C.c_double),
        ("fwd_ms", C.c_double),
        ("bwd_ms", C.c_double),
        ("recompute_ms", C.c_double),
        ("ratio_C", C.c_double),
        ("pipelines_per_cell", C.c_int32),
        ("tp_degree", C.c_int32),
        ("d_max", C.c_int32),
        ("n_order", C.c_int32),
        ("dc_order", C.c_int32 * GPB_MAX_DC),
        ("recompute", C.c_int32),
        ("multi_conn", C.c_int32),
        ("n_connections", C.c_int32),
        ("mem_limit", C.c_int32),
    ]


class Row(C.Structure):
    """SelectionRow (reference dc_select.h:32-40) + utilization."""

    _fields_ = [
        ("pp_time_ms", C.c_double),
        ("allreduce_time_ms", C.c_double),
        ("total_time_ms", C.c_double),
        ("throughput", C.c_double),
        ("utilization", C.c_double),
        ("makespan_ns", C.c_int64),
        ("scenario", C.c_int32),
        ("d", C.c_int32),
        ("feasible", C.c_int32),
        ("chosen", C.c_int32),
        ("partitions", C.c_int16 * GPB_MAX_DC),
    ]


class ScenarioResult(C.Structure):
    _fields_ = [
        ("first_row", C.c_int64),
        ("gpus_used", C.c_int64),
        ("n_rows", C.c_int32),
        ("chosen_d", C.c_int32),
    ]


class BucketInfo(C.Structure):
    _fields_ = [("policy", C.c_int32), ("B", C.c_int32), ("rows", C.c_int32),
                ("max_s", C.c_int32), ("max_c", C.c_int32), ("max_m", C.c_int32),
                ("stream", C.c_int32), ("pad_", C.c_int32), ("start_ms", C.c_float),
                ("ms", C.c_float), ("algo_ops", C.c_double)]


class Best(C.Structure):
    _fields_ = [("throughput", C.c_double), ("row", C.c_int64)]


class Bubble(C.Structure):
    _fields_ = [
        ("gpu_id", C.c_int32),
        ("pad_", C.c_int32),
        ("start_ns", C.c_int64),
        ("end_ns", C.c_int64),
    ]


class Request(C.Structure):
    _fields_ = [("id", C.c_int32), ("tokens", C.c_int32), ("arrival_ms", C.c_double)]


class PrefillModel(C.Structure):
    """PrefillModel (reference bubbletea.h:38-58) with its defaults."""

    _fields_ = [
        ("saturation_ms", C.c_double),
        ("max_tokens", C.c_int32),
        ("inference_layers", C.c_int32),
        ("stage_bw", C.c_double),
        ("boundary_latency_ms", C.c_double),
        ("guard_ms", C.c_double),
        ("memory_budget_bytes", C.c_int64),
        ("inference_hidden", C.c_int64),
        ("inference_params_per_layer", C.c_double),
        ("bytes_per_element", C.c_int32),
        ("pad_", C.c_int32),
    ]

    @classmethod
    def default(cls, **kw) -> "PrefillModel":
        pm = cls(
            saturation_ms=300.0,
            max_tokens=8192,
            inference_layers=8,
            stage_bw=25000000.0,
            boundary_latency_ms=0.0,
            guard_ms=0.0,
            memory_budget_bytes=1073741824,
            inference_hidden=1024,
            inference_params_per_layer=0.0,
            bytes_per_element=2,
        )
        for k, v in kw.items():
            setattr(pm, k, v)
        return pm


class Placement(C.Structure):
    _fields_ = [
        ("start_ns", C.c_int64),
        ("ttft_overhead_ms", C.c_double),
        ("accepted", C.c_int32),
        ("pipeline", C.c_int32),
    ]


class PackSummary(C.Structure):
    _fields_ = [
        ("utilization_before", C.c_double),
        ("utilization_after", C.c_double),
        ("accepted", C.c_int64),
        ("rejected", C.c_int64),
        ("horizon_ns", C.c_int64),
        ("placement_hash", C.c_uint64),
    ]


class Timing(C.Structure):
    _fields_ = [
        ("evaluate_ms", C.c_float),
        ("timing_kernels_ms", C.c_float),
        ("select_ms", C.c_float),
        ("pack_ms", C.c_float),
        ("policy_ms", C.c_float * 4),
        ("launches", C.c_int32),
        ("pad_", C.c_int32),
        ("h2d_bytes", C.c_int64),
        ("d2h_bytes", C.c_int64),
    ]


class Task(C.Structure):
    """ScheduledTask (reference schedule.h:14-23)."""

    _fields_ = [
        ("gpu", C.c_int32),
        ("cell", C.c_int32),
        ("pipeline", C.c_int32),
        ("kind", C.c_int32),
        ("microbatch", C.c_int32),
        ("stage", C.c_int32),
        ("start", C.c_int64),
        ("end", C.c_int64),
    ]


# --------------------------------------------------------------- builders

def gbps(x: float) -> float:
    """gbps_to_bytes_per_ms (reference base.h:23)."""
    return x * 125000.0


def make_topology(gpu_counts, latency_ms=0.0, cap_gbps=5.0, intra_gbps=100.0,
                  latency=None) -> Topology:
    """fixtures::make_topology (reference tests/support/fixtures.h:18-36);
    `latency` optionally gives a full symmetric matrix."""
    t = Topology()
    t.n_dc = len(gpu_counts)
    for i, g in enumerate(gpu_counts):
        t.gpu_count[i] = int(g)
        t.intra_bw[i] = gbps(intra_gbps)
    for i in range(t.n_dc):
        for j in range(t.n_dc):
            if i == j:
                v = 0.0
            elif latency is not None:
                v = float(latency[i][j])
            else:
                v = float(latency_ms)
            t.latency_ms[i][j] = v
    t.pair_bw_cap = gbps(cap_gbps)
    t.n_tcp = 0
    return t


def make_scenario(topology=0, policy="atlas", num_layers=1, layers_per_partition=1,
                  num_microbatches=1, hidden=1, seq_len=1, microbatch=1,
                  bytes_per_element=2, params_per_layer=0.0, fwd_ms=1.0,
                  bwd_ms=1.0, recompute_ms=1.0, ratio_C=0.0, C=1, tp=1,
                  d_max=0, dc_order=(), recompute=True, multi_conn=True,
                  n_connections=32, mem_limit=0) -> Scenario:
    s = Scenario()
    s.topology = topology
    s.policy = POLICIES[policy] if isinstance(policy, str) else int(policy)
    s.num_layers = num_layers
    s.layers_per_partition = layers_per_partition
    s.num_microbatches = num_microbatches
    s.bytes_per_element = bytes_per_element
    s.hidden = hidden
    s.seq_len = seq_len
    s.microbatch = microbatch
    s.params_per_layer = params_per_layer
    s.fwd_ms = fwd_ms
    s.bwd_ms = bwd_ms
    s.recompute_ms = recompute_ms
    s.ratio_C = ratio_C
    s.pipelines_per_cell = C
    s.tp_degree = tp
    s.d_max = d_max
    s.n_order = len(dc_order)
    for i, d in enumerate(dc_order):
        s.dc_order[i] = int(d)
    s.recompute = int(bool(recompute))
    s.multi_conn = int(bool(multi_conn))
    s.n_connections = n_connections
    s.mem_limit = mem_limit
    return s


def array(ctype, items):
    arr = (ctype * max(1, len(items)))()
    for i, x in enumerate(items):
        arr[i] = x
    return arr
