"""Host-side Python mirror of the reference's planner interface, over the
C ABI of libgeopipe_b200.so (include/geopipe_batch.h).

Reference interface mirrored (/root/reference/proj/src):
  select(SelectionInput)            dc_select.h:57   -> Planner.select()
  whatif(vector<WhatIfScenario>)    dc_select.h:72   -> Planner.whatif()
  extract_bubbles(Timeline, horizon) bubbletea.h:81  -> Planner.bubbles()
  schedule_prefills(...)            bubbletea.h:101  -> Planner.pack_prefills()
  synthetic_requests(...)           bubbletea.h:119  -> synthetic_requests()

Errors follow the reference's exception classes (capi.cpp:19-39 maps them
to GP_CONFIG_ERROR / GP_INFEASIBLE / GP_ERROR): ConfigError,
InsufficientGpus, GeopipeError. There is no CPU fallback: constructing a
Planner without the CUDA library or without a GPU raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgeopipe_b200.so")


class GeopipeError(RuntimeError):
    rc = abi.GPB_ERROR


class ConfigError(GeopipeError):
    rc = abi.GPB_CONFIG_ERROR


class InsufficientGpus(GeopipeError):
    rc = abi.GPB_INFEASIBLE


_ERRS = {abi.GPB_ERROR: GeopipeError, abi.GPB_CONFIG_ERROR: ConfigError,
         abi.GPB_INFEASIBLE: InsufficientGpus}

_lib = None


def load_library(path: str = LIB_PATH):
    """Load the CUDA library (fails loudly when it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise GeopipeError(f"{path} is missing: build it with __graft_entry__.build()")
    lib = C.CDLL(path)
    P = C.POINTER
    sig = {
        "gpb_create": (C.c_void_p, [C.c_int]),
        "gpb_destroy": (None, [C.c_void_p]),
        "gpb_last_error": (C.c_char_p, [C.c_void_p]),
        "gpb_single_tcp_bandwidth": (C.c_double, [P(abi.Topology), C.c_double]),
        "gpb_repeated_sum_host": (C.c_double, [C.c_double, C.c_longlong]),
        "gpb_load": (C.c_int, [C.c_void_p, P(abi.Topology), C.c_int32, P(abi.Scenario),
                               C.c_int32, P(C.c_int64)]),
        "gpb_evaluate": (C.c_int, [C.c_void_p, C.c_int32]),
        "gpb_fetch_rows": (C.c_int, [C.c_void_p, P(abi.Row), C.c_int64]),
        "gpb_fetch_scenarios": (C.c_int, [C.c_void_p, P(abi.ScenarioResult), C.c_int32]),
        "gpb_fetch_best": (C.c_int, [C.c_void_p, P(abi.Best)]),
        "gpb_device_best": (C.c_void_p, [C.c_void_p]),
        "gpb_bubbles": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, P(abi.Bubble),
                                  C.c_int64, P(C.c_int64)]),
        "gpb_pack_prefills": (C.c_int, [C.c_void_p, P(C.c_int64), C.c_int32,
                                        P(abi.Request), C.c_int64, P(abi.PrefillModel),
                                        C.c_int64, P(abi.PackSummary), P(abi.Placement)]),
        "gpb_synthetic_requests": (C.c_int, [C.c_int32, C.c_uint32, C.c_double,
                                             P(abi.PrefillModel), P(abi.Request)]),
        "gpb_get_timing": (C.c_int, [C.c_void_p, P(abi.Timing)]),
        "gpb_microbench": (C.c_int, [C.c_void_p, C.c_int32, P(C.c_double)]),
        "gpb_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
        "gpb_copy_best": (C.c_int, [C.c_void_p, C.c_void_p]),
        "gpb_set_profile": (C.c_int, [C.c_void_p, C.c_int32]),
        "gpb_set_bucket_timing": (C.c_int, [C.c_void_p, C.c_int32]),
        "gpb_set_allreduce_tail": (C.c_int, [C.c_void_p, C.c_int32]),
        "gpb_timeline_arrays": (C.c_int, [C.c_void_p, C.c_int64, P(C.c_int64), P(C.c_int64),
                                          C.c_int64, P(C.c_int32), P(C.c_int64)]),
        "gpb_fetch_row_cycles": (C.c_int, [C.c_void_p, P(C.c_int64), C.c_int64]),
        "gpb_bucket_infos": (C.c_int, [C.c_void_p, P(abi.BucketInfo), C.c_int32,
                                       P(C.c_int32)]),
        "gpb_saturating_requests": (C.c_int, [C.c_void_p, C.c_int64, P(abi.PrefillModel),
                                              C.c_int64, P(abi.Request), C.c_int64,
                                              P(C.c_int64)]),
        "gpb_validate_timeline": (C.c_int, [C.c_void_p, C.c_int64, P(C.c_int64), P(C.c_int64),
                                            P(C.c_int32), P(C.c_int64)]),
        "gpb_allreduce_tail": (C.c_int, [C.c_void_p, C.c_int64, P(C.c_int64), P(C.c_int64),
                                         C.c_int32, P(C.c_int32)]),
        "gpb_group_create": (C.c_void_p, [C.c_int32, P(C.c_int32)]),
        "gpb_group_destroy": (None, [C.c_void_p]),
        "gpb_group_last_error": (C.c_char_p, [C.c_void_p]),
        "gpb_group_size": (C.c_int32, [C.c_void_p]),
        "gpb_group_load": (C.c_int, [C.c_void_p, P(abi.Topology), C.c_int32, P(abi.Scenario),
                                     C.c_int32, P(C.c_int64)]),
        "gpb_group_evaluate": (C.c_int, [C.c_void_p]),
        "gpb_group_fetch_rows": (C.c_int, [C.c_void_p, P(abi.Row), C.c_int64]),
        "gpb_group_fetch_scenarios": (C.c_int, [C.c_void_p, P(abi.ScenarioResult), C.c_int32]),
        "gpb_group_fetch_best": (C.c_int, [C.c_void_p, P(abi.Best)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols():
    return ["gpb_create", "gpb_destroy", "gpb_last_error", "gpb_single_tcp_bandwidth",
            "gpb_load", "gpb_evaluate", "gpb_fetch_rows", "gpb_fetch_scenarios",
            "gpb_fetch_best", "gpb_device_best", "gpb_bubbles", "gpb_pack_prefills",
            "gpb_synthetic_requests", "gpb_get_timing", "gpb_microbench", "gpb_set_stream",
            "gpb_copy_best", "gpb_set_profile", "gpb_fetch_row_cycles",
            "gpb_set_allreduce_tail", "gpb_timeline_arrays", "gpb_bucket_infos",
            "gpb_set_bucket_timing", "gpb_saturating_requests", "gpb_validate_timeline",
            "gpb_allreduce_tail",
            "gpb_group_create", "gpb_group_destroy",
            "gpb_group_last_error", "gpb_group_size", "gpb_group_load", "gpb_group_evaluate",
            "gpb_group_fetch_rows", "gpb_group_fetch_scenarios", "gpb_group_fetch_best"]


@dataclass
class SelectionReport:
    """SelectionReport (dc_select.h:42-46)."""
    rows: list
    chosen_d: int
    gpus_used: int


@dataclass
class WhatIfRow:
    scenario: str
    row: abi.Row
    chosen: bool


class Planner:
    """One batch context bound to one CUDA device (not thread-safe)."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        self.ctx = self.lib.gpb_create(device)
        if not self.ctx:
            raise GeopipeError(f"gpb_create({device}) failed: no usable CUDA device")
        self.device = device
        self.n_rows = 0
        self.n_scen = 0

    def close(self):
        if self.ctx:
            self.lib.gpb_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc != abi.GPB_OK:
            msg = self.lib.gpb_last_error(self.ctx).decode()
            raise _ERRS.get(rc, GeopipeError)(msg)

    # ------------------------------------------------------------- batch
    def load(self, topos, scens) -> int:
        """Upload a plan space; returns the number of (scenario, D) rows."""
        if not isinstance(topos, C.Array):
            topos = abi.array(abi.Topology, list(topos))
        scen_arr = scens if isinstance(scens, C.Array) else abi.array(abi.Scenario, list(scens))
        n_scen = len(scens)
        n = C.c_int64()
        self._check(self.lib.gpb_load(self.ctx, topos, len(topos), scen_arr, n_scen,
                                      C.byref(n)))
        self.n_rows = n.value
        self.n_scen = n_scen
        return n.value

    def evaluate(self, sync: bool = True):
        self._check(self.lib.gpb_evaluate(self.ctx, 1 if sync else 0))

    def rows(self):
        out = (abi.Row * max(1, self.n_rows))()
        self._check(self.lib.gpb_fetch_rows(self.ctx, out, self.n_rows))
        return out

    def scenario_results(self):
        out = (abi.ScenarioResult * max(1, self.n_scen))()
        self._check(self.lib.gpb_fetch_scenarios(self.ctx, out, self.n_scen))
        return out

    def best(self) -> abi.Best:
        b = abi.Best()
        self._check(self.lib.gpb_fetch_best(self.ctx, C.byref(b)))
        return b

    def set_stream(self, cuda_stream: int | None):
        self._check(self.lib.gpb_set_stream(self.ctx, cuda_stream or None))

    def set_bucket_timing(self, enable: bool):
        self._check(self.lib.gpb_set_bucket_timing(self.ctx, int(bool(enable))))

    def set_profile(self, enable: bool):
        self._check(self.lib.gpb_set_profile(self.ctx, int(bool(enable))))

    def row_cycles(self):
        out = (C.c_int64 * max(1, self.n_rows))()
        self._check(self.lib.gpb_fetch_row_cycles(self.ctx, out, self.n_rows))
        return list(out[: self.n_rows])

    def copy_best(self, dst_ptr: int):
        """D2D copy of the 16-byte gpb_best to a device address (async)."""
        self._check(self.lib.gpb_copy_best(self.ctx, dst_ptr))

    def device_best_ptr(self) -> int:
        return self.lib.gpb_device_best(self.ctx)

    def timing(self) -> abi.Timing:
        t = abi.Timing()
        self._check(self.lib.gpb_get_timing(self.ctx, C.byref(t)))
        return t

    def bucket_infos(self):
        """Per-bucket shapes and device times of the last evaluate()."""
        n = C.c_int32()
        self._check(self.lib.gpb_bucket_infos(self.ctx, None, 0, C.byref(n)))
        out = (abi.BucketInfo * max(1, n.value))()
        self._check(self.lib.gpb_bucket_infos(self.ctx, out, n.value, C.byref(n)))
        return list(out[: n.value])

    def microbench(self, kind: int = 0) -> float:
        g = C.c_double()
        self._check(self.lib.gpb_microbench(self.ctx, kind, C.byref(g)))
        return g.value

    # ------------------------------------------------- reference mirrors
    def select(self, topos, scenario) -> SelectionReport:
        """select() (dc_select.cpp:99-123) for one scenario."""
        self.load(topos, [scenario])
        self.evaluate()
        rows = list(self.rows()[: self.n_rows])
        res = self.scenario_results()[0]
        return SelectionReport(rows, res.chosen_d, res.gpus_used)

    def whatif(self, topos, named_scenarios):
        """whatif() (dc_select.cpp:125-134): rows ordered by scenario then D."""
        names = [n for n, _ in named_scenarios]
        self.load(topos, [s for _, s in named_scenarios])
        self.evaluate()
        rows = self.rows()
        return [WhatIfRow(names[r.scenario], r, bool(r.chosen)) for r in rows[: self.n_rows]]

    def bubbles(self, row: int, horizon_ns: int = 0):
        cap = 1 << 16
        while True:
            out = (abi.Bubble * cap)()
            n = C.c_int64()
            self._check(self.lib.gpb_bubbles(self.ctx, row, horizon_ns, out, cap, C.byref(n)))
            if n.value <= cap:
                return [(b.gpu_id, b.start_ns, b.end_ns) for b in out[: n.value]]
            cap = n.value

    def timeline_arrays(self, row: int):
        """(fe, ps, dims, makespan) of one row's timeline, cell 0
        ([pipeline][stage][microbatch]; dims = (Ce, S, M, D))."""
        dims = (C.c_int32 * 4)()
        mk = C.c_int64()
        self._check(self.lib.gpb_timeline_arrays(self.ctx, row, None, None, 0, dims,
                                                 C.byref(mk)))
        n = dims[0] * dims[1] * dims[2]
        fe, ps = (C.c_int64 * n)(), (C.c_int64 * n)()
        self._check(self.lib.gpb_timeline_arrays(self.ctx, row, fe, ps, n, dims, C.byref(mk)))
        return fe, ps, tuple(dims), mk.value

    def allreduce_tail(self, row: int):
        """append_allreduce (scheduler.cpp:613-650) on the device: per stage
        (start_ns, duration_ns) of the all-reduce task."""
        n = C.c_int32()
        self._check(self.lib.gpb_allreduce_tail(self.ctx, row, None, None, 0, C.byref(n)))
        st, du = (C.c_int64 * max(1, n.value))(), (C.c_int64 * max(1, n.value))()
        self._check(self.lib.gpb_allreduce_tail(self.ctx, row, st, du, n.value, C.byref(n)))
        return list(zip(st[:n.value], du[:n.value]))

    def validate(self, row: int, fe=None, ps=None):
        """validate_timeline (validate.h:77-256) on the device: (check, where)."""
        chk, where = C.c_int32(), C.c_int64()
        self._check(self.lib.gpb_validate_timeline(self.ctx, row, fe, ps, C.byref(chk),
                                                   C.byref(where)))
        return chk.value, where.value

    def saturating_requests(self, row: int, pm=None, horizon_ns: int = 0):
        """saturating_requests (bubbletea.cpp:240-267) computed on the device."""
        pm = pm or abi.PrefillModel.default()
        n = C.c_int64()
        self._check(self.lib.gpb_saturating_requests(self.ctx, row, C.byref(pm), horizon_ns,
                                                     None, 0, C.byref(n)))
        out = (abi.Request * max(1, n.value))()
        self._check(self.lib.gpb_saturating_requests(self.ctx, row, C.byref(pm), horizon_ns,
                                                     out, n.value, C.byref(n)))
        return out if n.value > 0 else (abi.Request * 0)()

    def pack_prefills(self, rows, reqs, pm=None, horizon_ns: int = 0, placements=False):
        pm = pm or abi.PrefillModel.default()
        rows_arr = (C.c_int64 * max(1, len(rows)))(*rows)
        req_arr = reqs if isinstance(reqs, C.Array) else abi.array(abi.Request, reqs)
        n_req = len(reqs)
        summ = (abi.PackSummary * max(1, len(rows)))()
        pl = (abi.Placement * max(1, len(rows) * n_req))() if placements else None
        self._check(self.lib.gpb_pack_prefills(self.ctx, rows_arr, len(rows), req_arr, n_req,
                                               C.byref(pm), horizon_ns, summ, pl))
        return list(summ[: len(rows)]), pl


class PlannerGroup:
    """One plan space sharded over several devices of one box (gpb_group_*):
    cost-balanced whole-scenario shards, one host thread per device, the
    per-device winners all-gathered over NCCL. Results are in the order of
    the whole space, identical to a single-device Planner."""

    def __init__(self, devices=None):
        self.lib = load_library()
        devs = list(devices) if devices else []
        arr = (C.c_int32 * max(1, len(devs)))(*devs)
        self.g = self.lib.gpb_group_create(len(devs), arr if devs else None)
        if not self.g:
            raise GeopipeError(f"gpb_group_create({devs or 'all'}) failed")
        self.n_rows = 0
        self.n_scen = 0

    def size(self) -> int:
        return self.lib.gpb_group_size(self.g)

    def close(self):
        if self.g:
            self.lib.gpb_group_destroy(self.g)
            self.g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc != abi.GPB_OK:
            msg = self.lib.gpb_group_last_error(self.g).decode()
            raise _ERRS.get(rc, GeopipeError)(msg)

    def load(self, topos, scens) -> int:
        if not isinstance(topos, C.Array):
            topos = abi.array(abi.Topology, list(topos))
        scen_arr = scens if isinstance(scens, C.Array) else abi.array(abi.Scenario, list(scens))
        n = C.c_int64()
        self._check(self.lib.gpb_group_load(self.g, topos, len(topos), scen_arr, len(scens),
                                            C.byref(n)))
        self.n_rows, self.n_scen = n.value, len(scens)
        return n.value

    def evaluate(self):
        self._check(self.lib.gpb_group_evaluate(self.g))

    def rows(self):
        out = (abi.Row * max(1, self.n_rows))()
        self._check(self.lib.gpb_group_fetch_rows(self.g, out, self.n_rows))
        return out

    def scenario_results(self):
        out = (abi.ScenarioResult * max(1, self.n_scen))()
        self._check(self.lib.gpb_group_fetch_scenarios(self.g, out, self.n_scen))
        return out

    def best(self) -> abi.Best:
        b = abi.Best()
        self._check(self.lib.gpb_group_fetch_best(self.g, C.byref(b)))
        return b


def synthetic_requests(count: int, seed: int, horizon_ms: float, pm=None):
    """synthetic_requests (bubbletea.cpp:269-284) on the host."""
    lib = load_library()
    pm = pm or abi.PrefillModel.default()
    out = (abi.Request * max(1, count))()
    rc = lib.gpb_synthetic_requests(count, seed, horizon_ms, C.byref(pm), out)
    if rc != abi.GPB_OK:
        raise ConfigError("synthetic_requests: bad arguments")
    return out if count > 0 else (abi.Request * 0)()
