"""GPU parity at BASELINE config 2's full size (the bench workload): every one
of the 10^4 (scenario, D) rows of the Llama-3 70B plan search, all four
policies, bit-exact against the reference's select() (oracle/_ref compiled
from the reference sources, else the C port), the reference's report() on
run() for utilization and makespan, plus the per-scenario choice and the
global best. The reference runs on a host thread pool (its core is
re-entrant)."""
from concurrent.futures import ThreadPoolExecutor
import os

import pytest

from paper_2411_14458_b200 import abi, workloads

pytestmark = pytest.mark.gpu


def _key(r):
    return (r.d, r.feasible, r.chosen, r.pp_time_ms, r.allreduce_time_ms, r.total_time_ms,
            r.throughput, tuple(r.partitions))


def test_config2_all_rows_bit_exact(planner, checker):
    topos, scens = workloads.config2(10_000, seed=1)
    tarr = abi.array(abi.Topology, topos)
    n = planner.load(tarr, abi.array(abi.Scenario, scens))
    assert n == 10_000
    planner.evaluate()
    rows = planner.rows()
    res = planner.scenario_results()
    order = sorted(range(len(scens)), key=lambda i: -scens[i].num_microbatches * scens[i].d_max)

    def ref_scenario(i):
        # select() rows, plus report() on run() for every row: utilization
        # (metrics.cpp:39-54) and makespan (schedule.cpp:42-44)
        return checker.select(tarr, scens[i]), checker.report_rows(tarr, scens[i],
                                                                   scens[i].d_max)

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        ref = dict(zip(order, ex.map(ref_scenario, order)))
    best = (-1.0, -1)
    for i, sc in enumerate(scens):
        (ref_rows, chosen, used), rep = ref[i]
        r0 = res[i].first_row
        assert (res[i].n_rows, res[i].chosen_d, res[i].gpus_used) == (len(ref_rows), chosen, used)
        for k, (b, (util, mk)) in enumerate(zip(ref_rows, rep)):
            a = rows[r0 + k]
            assert _key(a) == _key(b), (i, k + 1, abi.POLICY_NAMES[sc.policy], _key(a), _key(b))
            assert (a.utilization, a.makespan_ns) == (util, mk), \
                (i, k + 1, abi.POLICY_NAMES[sc.policy], a.utilization, util, a.makespan_ns, mk)
            if b.feasible == 1 and b.throughput > best[0]:
                best = (b.throughput, r0 + k)
    got = planner.best()
    assert (got.throughput, got.row) == best


def test_two_sessions_pipelined(planner):
    """The bench's e2e loop: two sessions on their own streams, session B
    loading (host flatten + H2D) while session A evaluates, B's evaluate
    ordered after A's by an event. Each step's rows must equal a
    single-session evaluation of the same space."""
    import torch
    from paper_2411_14458_b200.planner import Planner

    spaces = []
    for seed in (1, 2):
        topos, scens = workloads.config2(2_000, seed=seed)
        tarr, sarr = abi.array(abi.Topology, topos), abi.array(abi.Scenario, scens)
        planner.load(tarr, sarr)
        planner.evaluate()
        spaces.append((tarr, sarr, [bytes(r) for r in planner.rows()]))
    other = Planner(0)
    try:
        sessions = [planner, other]
        streams = [torch.cuda.Stream(), torch.cuda.Stream()]
        for p, s in zip(sessions, streams):
            p.set_stream(s.cuda_stream)
        prev, pending = None, []
        for i in range(6):
            p, s = sessions[i % 2], streams[i % 2]
            tarr, sarr, want = spaces[(i // 2) % 2]
            p.load(tarr, sarr)
            if prev is not None:
                s.wait_event(prev)
            p.evaluate(sync=False)
            prev = torch.cuda.Event()
            prev.record(s)
            pending.append((p, want))
            if len(pending) == 2:
                q, w = pending.pop(0)
                out = (abi.Row * q.n_rows)()
                assert q.lib.gpb_fetch_rows(q.ctx, out, q.n_rows) == 0
                assert [bytes(r) for r in out] == w, i
        q, w = pending.pop(0)
        assert [bytes(r) for r in q.rows()] == w
    finally:
        other.close()
        planner.set_stream(None)
