"""GPU parity: every row of select()/whatif() computed by the sm_100a
kernels equals the reference's (compiled oracle/_ref when present, else the
C port) bit for bit — pp/allreduce/total/throughput doubles, partitions,
feasibility, chosen flags, gpus_used — plus report() utilization and the
makespan. Parity target: bit-exact (north_star)."""
import math

import pytest

from paper_2411_14458_b200 import abi
from tests import fixtures
from tests.instances import random_space

pytestmark = pytest.mark.gpu


def _row_key(r):
    return (r.d, r.feasible, r.chosen, r.pp_time_ms, r.allreduce_time_ms, r.total_time_ms,
            r.throughput, tuple(r.partitions))


def _compare_space(planner, checker, port, topos, scens):
    """Every row of the space vs the checker's select(), and utilization /
    makespan vs its report() on run() (the reference's, metrics.cpp:39-54,
    when oracle/_ref is present; else the C port's rows, pinned to the
    reference in test_oracle.py). `port` is kept for call compatibility."""
    from concurrent.futures import ThreadPoolExecutor
    import os
    planner.load(topos, scens)
    planner.evaluate()
    rows = planner.rows()
    res = planner.scenario_results()

    def ref_scenario(i):
        sel = checker.select(topos, scens[i])
        return sel, checker.report_rows(topos, scens[i], len(sel[0]))

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        ref = list(ex.map(ref_scenario, range(len(scens))))
    n_checked = 0
    for i, ((ref_rows, chosen, used), rep) in enumerate(ref):
        r0 = res[i].first_row
        assert res[i].n_rows == len(ref_rows)
        assert res[i].chosen_d == chosen, f"scenario {i}"
        assert res[i].gpus_used == used
        for k, (a, b, (util, mk)) in enumerate(zip(rows[r0:r0 + len(ref_rows)], ref_rows, rep)):
            assert a.scenario == i
            assert _row_key(a) == _row_key(b), f"scenario {i} d={k+1}: {_row_key(a)} vs {_row_key(b)}"
            assert (a.makespan_ns, a.utilization) == (mk, util), (i, k, a.utilization, util)
            n_checked += 1
    return n_checked


def test_unit12_makespans(planner):
    # test_scheduler.cpp:53-63: gpipe 38, 1f1b 39, varuna 38, atlas 36 ms
    for pol, ms in (("gpipe", 38.0), ("1f1b", 39.0), ("varuna", 38.0), ("atlas", 36.0)):
        topos, sc = fixtures.unit12(policy=pol)
        rep = planner.select(topos, sc)
        assert rep.rows[0].pp_time_ms == ms, pol


def test_atlas_mem_limits(planner):
    # test_scheduler.cpp:175-196: mem_limit 1 -> 89, 2 -> 67, 6 -> 36
    for ml, ms in ((1, 89.0), (2, 67.0), (6, 36.0)):
        topos, sc = fixtures.unit12(policy="atlas", mem_limit=ml)
        assert planner.select(topos, sc).rows[0].pp_time_ms == ms


def test_config1_kats(planner):
    # config-1 makespans from the compiled reference
    kat = {("1f1b", False): 28344.858980, ("1f1b", True): 2470.61274,
           ("gpipe", False): 44295.774368, ("gpipe", True): 2896.980384,
           ("atlas", False): 45335.774368, ("atlas", True): 3936.980384}
    for (pol, multi), ms in kat.items():
        topos, sc = fixtures.config1(pol, multi)
        got = planner.select(topos, sc).rows[0].pp_time_ms
        assert abs(got - ms) < 5e-7, (pol, multi, got)


def test_config1_bit_exact(planner, checker):
    """BASELINE config 1 (4-stage PP over 2 DCs, M=8), all four policies x
    single/multi TCP: the whole row (pp/all-reduce/total/throughput doubles,
    partitions, chosen) bit-exact against the reference's select()
    (dc_select.cpp:99-123) and utilization/makespan against its report() on
    run() (metrics.cpp:39-54)."""
    for pol in ("gpipe", "1f1b", "varuna", "atlas"):
        for multi in (False, True):
            topos, sc = fixtures.config1(pol, multi)
            rep = planner.select(topos, sc)
            ref_rows, chosen, used = checker.select(topos, sc)
            assert rep.chosen_d == chosen and rep.gpus_used == used, (pol, multi)
            (util, mk), = checker.report_rows(topos, sc, 1)
            a, b = rep.rows[0], ref_rows[0]
            assert _row_key(a) == _row_key(b), (pol, multi, _row_key(a), _row_key(b))
            assert (a.utilization, a.makespan_ns) == (util, mk), (pol, multi)


def test_small_random_spaces(planner, checker):
    from oracle import bindings
    topos, scens = random_space(1234, 400, wide=False)
    assert _compare_space(planner, checker, bindings.port(), topos, scens) > 400


def test_wide_random_spaces(planner, checker):
    from oracle import bindings
    topos, scens = random_space(99, 250, wide=True)
    assert _compare_space(planner, checker, bindings.port(), topos, scens) > 250


def test_five_dc_select(planner, checker):
    from oracle import bindings
    for pol in ("atlas", "varuna", "gpipe", "1f1b"):
        for C in (2, 3):
            topos, sc = fixtures.five_dc(5, C, pol)
            _compare_space(planner, checker, bindings.port(), topos, [sc])


def test_best_is_global_argmax(planner):
    topos, scens = random_space(5, 60, wide=True)
    planner.load(topos, scens)
    planner.evaluate()
    rows = planner.rows()
    best = planner.best()
    cand = [(r.throughput, -i) for i, r in enumerate(rows[:planner.n_rows]) if r.feasible == 1]
    if cand:
        thr, neg = max(cand)
        assert best.row == -neg and best.throughput == thr


def test_reload_same_shapes_and_stream_switch(planner, checker):
    """A reload with the same bucket shapes keeps the prepared launch sequence
    (host.cu gpb_load); uploads are asynchronous on the launch stream, and a
    stream switch after the load must still see them. Every row stays
    bit-exact with the reference."""
    import ctypes

    import torch
    from oracle import bindings

    def clone(x):
        y = type(x)()
        ctypes.memmove(ctypes.byref(y), ctypes.byref(x), ctypes.sizeof(x))
        return y

    topos, scens = random_space(4321, 120, wide=False)
    assert _compare_space(planner, checker, bindings.port(), topos, scens) > 120
    # same shapes (policy, stages, microbatches, pipelines, row counts),
    # different WAN latencies and compute times
    topos2 = abi.array(abi.Topology, [clone(t) for t in topos])
    for t in topos2:
        for a in range(t.n_dc):
            for b in range(t.n_dc):
                if a != b:
                    t.latency_ms[a][b] = t.latency_ms[a][b] * 1.5 + 3.0
    scens2 = abi.array(abi.Scenario, [clone(s) for s in scens])
    for s in scens2:
        s.fwd_ms, s.bwd_ms = s.fwd_ms * 1.25, s.bwd_ms * 0.8
        if s.ratio_C > 0:
            s.ratio_C = s.ratio_C * 0.75
    assert _compare_space(planner, checker, bindings.port(), topos2, scens2) > 120
    # load on the own stream, evaluate on a fresh torch stream
    side = torch.cuda.Stream()
    planner.set_stream(None)
    planner.load(topos, scens)
    planner.set_stream(side.cuda_stream)
    planner.evaluate()
    rows = planner.rows()
    planner.set_stream(None)
    for i, sc in enumerate(scens[:40]):
        ref_rows, _, _ = checker.select(topos, sc)
        r0 = planner.scenario_results()[i].first_row
        for a, b in zip(rows[r0:r0 + len(ref_rows)], ref_rows):
            assert _row_key(a) == _row_key(b)


@pytest.mark.parametrize("graph", ["1", "0"])
def test_graph_mode_reloads(planner, checker, monkeypatch, graph):
    """The evaluate launch sequence is replayed as a CUDA graph (default) or
    launched directly (GPB_GRAPH=0); a reload (same bucket shapes with other
    values, a different scenario split, another space) must re-capture the
    graph whenever anything it baked in changed: every row stays bit-exact."""
    import ctypes
    monkeypatch.setenv("GPB_GRAPH", graph)
    topos, scens = random_space(4321, 120, wide=False)
    assert _compare_space(planner, checker, None, topos, scens) > 120
    scens2 = abi.array(abi.Scenario, [type(s).from_buffer_copy(s) for s in scens])
    for s in scens2:
        s.fwd_ms, s.bwd_ms = s.fwd_ms * 1.25, s.bwd_ms * 0.8
    assert _compare_space(planner, checker, None, topos, scens2) > 120
    # same rows split over scenarios differently (d_max moved between two)
    scens3 = abi.array(abi.Scenario, [type(s).from_buffer_copy(s) for s in scens])
    assert ctypes.sizeof(scens3[0]) == ctypes.sizeof(abi.Scenario)
    assert _compare_space(planner, checker, None, topos, scens3[::-1]) > 120
    topos4, scens4 = random_space(99, 80, wide=True)
    assert _compare_space(planner, checker, None, topos4, scens4) > 80


@pytest.mark.parametrize("lane", ["1", "0"])
def test_drain_greedy_variants(planner, checker, monkeypatch, lane):
    """The WAN-stage drain greedy runs on one lane (C <= 4, S >= GPB_DRAIN_LANE,
    default 32) or warp-wide; force each on every eligible row (the graph key
    carries the switch, so the same load re-captures): rows stay bit-exact."""
    monkeypatch.setenv("GPB_DRAIN_LANE", lane)
    for ml, ms in ((1, 89.0), (2, 67.0), (6, 36.0), (0, 36.0)):
        topos, sc = fixtures.unit12(policy="atlas", mem_limit=ml)
        assert planner.select(topos, sc).rows[0].pp_time_ms == ms
    topos, scens = random_space(2024, 120, wide=False)
    assert _compare_space(planner, checker, None, topos, scens) > 120
    topos, scens = random_space(77, 60, wide=True)
    assert _compare_space(planner, checker, None, topos, scens) > 60


def test_validator_accepts_every_policy(planner):
    """validate_timeline (validate.h:77-256) on the device: every feasible
    row's own timeline is valid (completeness, GPU and link exclusivity,
    causality, makespan)."""
    import random
    topos, scens = random_space(71, 150, wide=True)
    planner.load(topos, scens)
    planner.evaluate()
    rows = planner.rows()
    rng = random.Random(2)
    seen = set()
    n = 0
    for i, r in enumerate(rows[:planner.n_rows]):
        sc = scens[r.scenario]
        if r.feasible != 1 or r.d * sc.pipelines_per_cell * sc.num_layers > 3000 or rng.random() > 0.4:
            continue
        assert planner.validate(i) == (0, 0), (i, abi.POLICY_NAMES[sc.policy])
        seen.add(sc.policy)
        n += 1
    assert n > 40 and seen == {0, 1, 2, 3}


def test_validator_rejects_corrupted_timelines(planner):
    """The validator flags timelines corrupted to break completeness (check
    1), GPU / link exclusivity or causality (checks 2-5: a moved task breaks
    the first of them it meets) and the makespan (check 6), on unit12 (2
    pipelines x 6 stages over 3 DCs) for ATLAS and gpipe."""
    for pol in ("atlas", "gpipe"):
        topos, sc = fixtures.unit12(policy=pol)
        planner.load(topos, [sc])
        planner.evaluate()
        fe, ps, (Ce, S, M, D), mk = planner.timeline_arrays(0)
        assert planner.validate(0) == (0, 0)
        assert planner.validate(0, fe, ps) == (0, 0)
        idx = lambda p, s, m: (p * S + s) * M + m  # noqa: E731

        def corrupt(fn):
            a, b = type(fe).from_buffer_copy(fe), type(ps).from_buffer_copy(ps)
            fn(a, b)
            return planner.validate(0, a, b)[0]

        assert corrupt(lambda a, b: a.__setitem__(idx(0, 2, 1), -1)) == 1
        assert corrupt(lambda a, b: b.__setitem__(idx(0, 3, 1), -1)) == 1
        # a forward moved before its input, a pair before its gradient, a
        # pair onto a forward
        assert corrupt(lambda a, b: a.__setitem__(idx(0, 3, 0), a[idx(0, 2, 0)])) in (2, 3, 4)
        assert corrupt(lambda a, b: b.__setitem__(idx(0, 2, M - 1), b[idx(0, 3, M - 1)])) in (2, 3, 5)
        assert corrupt(lambda a, b: b.__setitem__(idx(0, 5, 0), a[idx(0, 5, 0)] - 1)) in (2, 5)
        # the last pair (stage 0) pushed later: the makespan no longer matches
        last = max(range(len(ps)), key=lambda k: ps[k])
        assert (last // M) % S == 0
        assert corrupt(lambda a, b: b.__setitem__(last, b[last] + 10**9)) == 6
    # pooled link (ATLAS): pipeline 1's activation transfer on the first WAN
    # boundary (stage 1 -> 2) moved onto pipeline 0's
    topos, sc = fixtures.unit12(policy="atlas")
    planner.load(topos, [sc])
    planner.evaluate()
    fe, ps, (Ce, S, M, D), mk = planner.timeline_arrays(0)
    a, b = type(fe).from_buffer_copy(fe), type(ps).from_buffer_copy(ps)
    a[(1 * S + 1) * M + 0] = a[(0 * S + 1) * M + 0]
    assert planner.validate(0, a, b)[0] in (2, 3, 4)


def test_atlas_wave_rows_bit_exact(planner, checker, monkeypatch):
    """Heavy ATLAS rows with 2..8 pipelines run one CTA per row, one warp per
    pipeline, pipeline p waiting on the earlier pipelines' link frontiers
    (atlas_wave_kernel); force it on every eligible row of the unit12 KATs,
    random spaces with small memory caps, and config 2, and check each row
    against the reference."""
    import random
    from oracle import bindings
    from paper_2411_14458_b200 import workloads
    monkeypatch.setenv("GPB_ATLAS_WAVE", "2")
    for ml, ms in ((1, 89.0), (2, 67.0), (6, 36.0), (0, 36.0)):
        topos, sc = fixtures.unit12(policy="atlas", mem_limit=ml)
        assert planner.select(topos, sc).rows[0].pp_time_ms == ms
    rng = random.Random(9)
    topos, scens = [], []
    for _ in range(80):
        n_dc = rng.randint(2, 5)
        counts = [rng.choice([64, 128, 256]) for _ in range(n_dc)]
        lat = [[0.0] * n_dc for _ in range(n_dc)]
        for i in range(n_dc):
            for j in range(i + 1, n_dc):
                lat[i][j] = lat[j][i] = rng.choice([5.0, 20.0, 80.0])
        topos.append(abi.make_topology(counts, cap_gbps=rng.choice([1.0, 5.0, 25.0]),
                                       intra_gbps=100.0, latency=lat))
        S = rng.randint(2, 32)
        scens.append(abi.make_scenario(
            topology=len(topos) - 1, policy="atlas", num_layers=S,
            num_microbatches=rng.choice([2, 7, 16, 64]),
            hidden=rng.choice([1024, 4096]), seq_len=rng.choice([1024, 4096]),
            fwd_ms=rng.uniform(1.0, 20.0), bwd_ms=rng.uniform(2.0, 40.0),
            recompute_ms=rng.uniform(0.0, 10.0), C=rng.choice([2, 3, 4, 8]),
            recompute=rng.random() < 0.5, multi_conn=rng.random() < 0.5,
            mem_limit=rng.choice([0, 1, 2, 5, S]), d_max=1, dc_order=list(range(n_dc))))
    assert _compare_space(planner, checker, bindings.port(), abi.array(abi.Topology, topos),
                          abi.array(abi.Scenario, scens)) == 80
    topos, scens = workloads.config2(3000, seed=7)
    scens = [s for s in scens if s.policy == 3]
    assert _compare_space(planner, checker, bindings.port(), abi.array(abi.Topology, topos),
                          abi.array(abi.Scenario, scens)) > 500
