"""TEST INFRASTRUCTURE ONLY — ctypes loaders for the checkers.

* ``port()``      -> oracle/liboracle.so, the plain-C restatement
                     (geopipe_oracle.c) of the reference hot path.
* ``reference()`` -> oracle/_ref/libgeopipe_ref.so, the unmodified reference
                     sources compiled by oracle/Makefile (absent on a box
                     where it was not built; then returns None).

Both expose the same calls over the batch ABI structs, so a test can diff
the product against either. Only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline leg import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from functools import lru_cache

from paper_2411_14458_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgeopipe_ref.so")


class CheckerError(RuntimeError):
    def __init__(self, rc, msg):
        super().__init__(f"rc={rc}: {msg}")
        self.rc = rc


class Checker:
    """Uniform wrapper; `prefix` is 'orc' (port) or 'ref' (reference)."""

    def __init__(self, path: str, prefix: str):
        self.path = path
        self.prefix = prefix
        self.lib = C.CDLL(path)
        f = self._fn
        P = C.POINTER
        self._err = f("last_error", C.c_char_p, [])
        self._single = f("single_tcp_bandwidth", C.c_double,
                         [P(abi.Topology), C.c_double])
        self._select = f("select", C.c_int, [P(abi.Topology), P(abi.Scenario), P(abi.Row),
                                             C.c_int32, P(C.c_int32), P(C.c_int32),
                                             P(C.c_int64)])
        self._bubbles = f("bubbles", C.c_int, [P(abi.Topology), P(abi.Scenario), C.c_int32,
                                               C.c_int64, P(abi.Bubble), C.c_int64,
                                               P(C.c_int64)])
        self._pack = f("pack_prefills", C.c_int,
                       [P(abi.Topology), P(abi.Scenario), C.c_int32, P(abi.Request),
                        C.c_int64, P(abi.PrefillModel), C.c_int64, P(abi.PackSummary),
                        P(abi.Placement)])
        self._sat = f("saturating_requests", C.c_int,
                      [P(abi.Topology), P(abi.Scenario), C.c_int32, P(abi.PrefillModel),
                       C.c_int64, P(abi.Request), C.c_int64, P(C.c_int64)])
        if prefix == "ref":
            self._timeline = f("timeline", C.c_int,
                               [P(abi.Topology), P(abi.Scenario), C.c_int32, C.c_int32,
                                P(abi.Task), C.c_int64, P(C.c_int64), P(C.c_int64)])
            self._synth = f("synthetic_requests", C.c_int,
                            [C.c_int32, C.c_uint32, C.c_double, P(abi.PrefillModel),
                             P(abi.Request)])
            self._whatif = f("whatif_count", C.c_int,
                             [P(abi.Topology), P(abi.Scenario), C.c_int32,
                              P(C.c_int64), P(C.c_int64)])
            self._artail = f("allreduce_tail", C.c_int,
                             [P(abi.Topology), P(abi.Scenario), C.c_int32, P(C.c_int64),
                              P(C.c_int64), C.c_int32, P(C.c_int32)])
            self._report = f("report_rows", C.c_int,
                             [P(abi.Topology), P(abi.Scenario), C.c_int32,
                              P(C.c_double), P(C.c_int64)])
        else:
            self._timeline_orc = f("timeline", C.c_int,
                                   [P(abi.Topology), P(abi.Scenario), C.c_int32,
                                    P(abi.Task), C.c_int64, P(C.c_int64), P(C.c_int64)])

    def _fn(self, name, res, args):
        fn = getattr(self.lib, f"{self.prefix}_{name}")
        fn.restype = res
        fn.argtypes = args
        return fn

    def _check(self, rc):
        if rc != 0:
            raise CheckerError(rc, self._err().decode())

    # ------------------------------------------------------------ calls
    def single_tcp_bandwidth(self, topo: abi.Topology, lat: float) -> float:
        return self._single(C.byref(topo), lat)

    def select(self, topos, sc):
        cap = 4096
        rows = (abi.Row * cap)()
        n, chosen, used = C.c_int32(), C.c_int32(), C.c_int64()
        self._check(self._select(topos, C.byref(sc), rows, cap, C.byref(n),
                                 C.byref(chosen), C.byref(used)))
        if n.value > cap:
            rows = (abi.Row * n.value)()
            self._check(self._select(topos, C.byref(sc), rows, n.value, C.byref(n),
                                     C.byref(chosen), C.byref(used)))
        return list(rows[: n.value]), chosen.value, used.value

    def timeline(self, topos, sc, d, replay=1):
        cap = 1 << 16
        while True:
            out = (abi.Task * cap)()
            n, ms = C.c_int64(), C.c_int64()
            if self.prefix == "ref":
                rc = self._timeline(topos, C.byref(sc), d, replay, out, cap,
                                    C.byref(n), C.byref(ms))
            else:
                rc = self._timeline_orc(topos, C.byref(sc), d, out, cap, C.byref(n),
                                        C.byref(ms))
            self._check(rc)
            if n.value <= cap:
                return list(out[: n.value]), ms.value
            cap = n.value

    def bubbles(self, topos, sc, d, horizon=0):
        cap = 1 << 14
        while True:
            out = (abi.Bubble * cap)()
            n = C.c_int64()
            self._check(self._bubbles(topos, C.byref(sc), d, horizon, out, cap, C.byref(n)))
            if n.value <= cap:
                return [(b.gpu_id, b.start_ns, b.end_ns) for b in out[: n.value]]
            cap = n.value

    def pack(self, topos, sc, d, reqs, pm, horizon=0, placements=True):
        n = len(reqs)
        req_arr = abi.array(abi.Request, reqs)
        summ = abi.PackSummary()
        pl = (abi.Placement * max(1, n))() if placements else None
        self._check(self._pack(topos, C.byref(sc), d, req_arr, n, C.byref(pm), horizon,
                               C.byref(summ), pl))
        return summ, (list(pl[:n]) if placements else None)

    def saturating(self, topos, sc, d, pm, horizon=0):
        cap = 1 << 14
        while True:
            out = (abi.Request * cap)()
            n = C.c_int64()
            self._check(self._sat(topos, C.byref(sc), d, C.byref(pm), horizon, out, cap,
                                  C.byref(n)))
            if n.value <= cap:
                return list(out[: n.value])
            cap = n.value

    def synthetic(self, count, seed, horizon_ms, pm):
        out = (abi.Request * max(1, count))()
        self._check(self._synth(count, seed, horizon_ms, C.byref(pm), out))
        return list(out[:count])

    def report_rows(self, topos, sc, n):
        """[(utilization, makespan_ns)] of rows d = 1..n: the reference's
        report() on run() (metrics.cpp:39-54); (0, 0) for infeasible rows.
        The port's select() rows carry the same two values."""
        if self.prefix != "ref":
            rows, _, _ = self.select(topos, sc)
            return [(r.utilization, r.makespan_ns) for r in rows[:n]]
        util = (C.c_double * max(1, n))()
        mk = (C.c_int64 * max(1, n))()
        self._check(self._report(topos, C.byref(sc), n, util, mk))
        return list(zip(util[:n], mk[:n]))

    def allreduce_tail(self, topos, sc, d):
        """[(start_ns, duration_ns)] per stage of append_allreduce
        (scheduler.cpp:613-650) on row d's schedule (reference only)."""
        cap = 512
        st, du, n = (C.c_int64 * cap)(), (C.c_int64 * cap)(), C.c_int32()
        self._check(self._artail(topos, C.byref(sc), d, st, du, cap, C.byref(n)))
        return list(zip(st[:n.value], du[:n.value]))

    def whatif_count(self, topos, scens):
        arr = abi.array(abi.Scenario, scens)
        nr, nc = C.c_int64(), C.c_int64()
        self._check(self._whatif(topos, arr, len(scens), C.byref(nr), C.byref(nc)))
        return nr.value, nc.value


@lru_cache(maxsize=None)
def port() -> Checker:
    if not os.path.exists(PORT_SO):
        raise FileNotFoundError(f"{PORT_SO} missing: run `make -C oracle`")
    return Checker(PORT_SO, "orc")


@lru_cache(maxsize=None)
def reference():
    if not os.path.exists(REF_SO):
        return None
    return Checker(REF_SO, "ref")
