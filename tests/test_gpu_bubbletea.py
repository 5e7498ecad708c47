"""GPU parity for bubbles (extract_bubbles, bubbletea.cpp:56-66) and BubbleTea
packing (schedule_prefills, bubbletea.cpp:132-222) against the reference:
bit-exact bubble lists, per-request placements (pipeline, start, ttft),
accepted/rejected counts, placement hash and utilization before/after."""
import random

import pytest

from paper_2411_14458_b200 import abi
from paper_2411_14458_b200.planner import synthetic_requests
from tests import fixtures
from tests.instances import random_space

pytestmark = pytest.mark.gpu


def _feasible_rows(planner, topos, scens, limit_gpus=3000):
    planner.load(topos, scens)
    planner.evaluate()
    rows = planner.rows()
    out = []
    for i, r in enumerate(rows[: planner.n_rows]):
        sc = scens[r.scenario]
        if r.feasible == 1 and r.d * sc.pipelines_per_cell * sc.num_layers <= limit_gpus:
            out.append((i, r))
    return out


@pytest.mark.parametrize("wide", [False, True])
def test_bubbles_random(planner, checker, wide):
    topos, scens = random_space(77 if wide else 78, 150, wide)
    rng = random.Random(3)
    n = 0
    for i, r in _feasible_rows(planner, topos, scens):
        if rng.random() > 0.5:
            continue
        sc = scens[r.scenario]
        for hz in (0, max(1, r.makespan_ns // 2), r.makespan_ns + 12345):
            got = planner.bubbles(i, hz)
            want = checker.bubbles(topos, sc, r.d, hz)
            assert got == want, (i, r.d, hz, abi.POLICY_NAMES[sc.policy])
            n += 1
    assert n > 30


def test_unit12_bubble_kats(planner, checker):
    # unit12 atlas 32 bubbles, varuna 54
    for pol, nb in (("atlas", 32), ("varuna", 54)):
        topos, sc = fixtures.unit12(policy=pol)
        planner.load(topos, [sc])
        planner.evaluate()
        b = planner.bubbles(0)
        assert len(b) == nb
        assert b == checker.bubbles(topos, sc, 1)


def test_acceptance_bubble_filling(planner, checker):
    # acceptance.cpp:221-252: unit12 M=5 atlas, saturating stream
    topos, sc = fixtures.unit12(M=5, policy="atlas")
    planner.load(topos, [sc])
    planner.evaluate()
    pm = abi.PrefillModel.default()
    reqs = checker.saturating(topos, sc, 1, pm)
    summ, pl = planner.pack_prefills([0], reqs, pm, placements=True)
    want, wpl = checker.pack(topos, sc, 1, reqs, pm)
    s = summ[0]
    assert (s.accepted, s.rejected, s.placement_hash, s.utilization_before,
            s.utilization_after) == (want.accepted, want.rejected, want.placement_hash,
                                     want.utilization_before, want.utilization_after)
    assert 0.37 <= s.utilization_before <= 0.53 and s.utilization_after >= 0.90
    for a, b in zip(pl[: len(reqs)], wpl):
        assert (a.accepted, a.pipeline, a.start_ns, a.ttft_overhead_ms) == \
            (b.accepted, b.pipeline, b.start_ns, b.ttft_overhead_ms)


@pytest.mark.parametrize("wide", [False, True])
def test_pack_random(planner, checker, wide):
    topos, scens = random_space(91 if wide else 92, 120, wide)
    rng = random.Random(11)
    cand = _feasible_rows(planner, topos, scens, limit_gpus=2000)
    rng.shuffle(cand)
    cand = cand[:24]
    assert cand
    for mode in ("sat", "syn"):
        pm = abi.PrefillModel.default(
            guard_ms=rng.choice([0.0, 0.5]), boundary_latency_ms=rng.choice([0.0, 1.0]),
            inference_layers=rng.choice([8, 3, 1]))
        if mode == "syn":
            hmax = max(r.makespan_ns for _, r in cand) / 1e6
            reqs = list(synthetic_requests(400, rng.randint(0, 99), hmax * 1.1, pm))
        for i, r in cand:
            sc = scens[r.scenario]
            if mode == "sat":
                reqs = checker.saturating(topos, sc, r.d, pm)
            got, gpl = planner.pack_prefills([i], reqs, pm, placements=True)
            want, wpl = checker.pack(topos, sc, r.d, reqs, pm)
            g = got[0]
            assert (g.accepted, g.rejected, g.placement_hash, g.horizon_ns) == \
                (want.accepted, want.rejected, want.placement_hash, want.horizon_ns), (mode, i)
            assert g.utilization_before == want.utilization_before
            assert g.utilization_after == want.utilization_after
            for a, b in zip(gpl[: len(reqs)], wpl):
                assert (a.accepted, a.pipeline, a.start_ns, a.ttft_overhead_ms) == \
                    (b.accepted, b.pipeline, b.start_ns, b.ttft_overhead_ms)


def test_pack_many_rows_one_call(planner, checker):
    topos, scens = random_space(5, 80, True)
    cand = _feasible_rows(planner, topos, scens, limit_gpus=2000)[:40]
    pm = abi.PrefillModel.default()
    hmax = max(r.makespan_ns for _, r in cand) / 1e6
    reqs = list(synthetic_requests(300, 42, hmax, pm))
    got, _ = planner.pack_prefills([i for i, _ in cand], reqs, pm)
    for (i, r), g in zip(cand, got):
        want, _ = checker.pack(topos, scens[r.scenario], r.d, reqs, pm, placements=False)
        assert (g.accepted, g.placement_hash, g.utilization_after) == \
            (want.accepted, want.placement_hash, want.utilization_after), i


def test_synthetic_requests_match_reference(checker):
    from oracle import bindings
    ref = bindings.reference()
    if ref is None:
        pytest.skip("compiled reference not present")
    pm = abi.PrefillModel.default()
    a = list(synthetic_requests(1000, 42, 1234.5, pm))
    b = ref.synthetic(1000, 42, 1234.5, pm)
    assert [(x.id, x.tokens, x.arrival_ms) for x in a] == [(x.id, x.tokens, x.arrival_ms) for x in b]


def test_pack_config2_top_plans_long_trace(planner, checker):
    """BubbleTea at a config-4-like shape: the best plans of the bench's
    config-2 space, one shared synthetic trace whose arrivals span the largest
    makespan, most requests rejected; summaries and placements bit-exact."""
    from paper_2411_14458_b200 import workloads
    topos, scens = workloads.config2(2_000, seed=3)
    tarr = abi.array(abi.Topology, topos)
    planner.load(tarr, abi.array(abi.Scenario, scens))
    planner.evaluate()
    rows = planner.rows()
    # the best plans with at most 8 cells (the reference's packing cost grows
    # with D^2 per request; the GPU path is D-parallel)
    feas = sorted(((r.throughput, i) for i, r in enumerate(rows[:planner.n_rows])
                   if r.feasible == 1 and r.d <= 8), key=lambda x: (-x[0], x[1]))
    pols = {}
    top = []
    for _, i in feas:  # a few plans of every policy
        pol = scens[rows[i].scenario].policy
        if pols.get(pol, 0) < 2:
            pols[pol] = pols.get(pol, 0) + 1
            top.append(i)
    pm = abi.PrefillModel.default()
    hmax = max(rows[i].makespan_ns for i in top) / 1e6
    reqs = list(synthetic_requests(4_000, 7, hmax, pm))
    got, gpl = planner.pack_prefills(top, reqs, pm, placements=True)
    n = len(reqs)
    for k, i in enumerate(top):
        sc = scens[rows[i].scenario]
        want, wpl = checker.pack(tarr, sc, rows[i].d, reqs, pm)
        g = got[k]
        assert (g.accepted, g.rejected, g.placement_hash, g.utilization_before,
                g.utilization_after) == (want.accepted, want.rejected, want.placement_hash,
                                         want.utilization_before, want.utilization_after), k
        for a, b in zip(gpl[k * n:(k + 1) * n], wpl):
            assert (a.accepted, a.pipeline, a.start_ns, a.ttft_overhead_ms) == \
                (b.accepted, b.pipeline, b.start_ns, b.ttft_overhead_ms)


def test_pack_many_cells_zero_layer_stages(planner, checker):
    """Plans with more cells than inference layers (D > 8): the trailing
    stages of every prefill pipeline carry zero layers and zero-length pieces
    (the touching-gap rule); placements bit-exact on a saturating stream and a
    synthetic trace."""
    from paper_2411_14458_b200 import workloads
    topos, scens = workloads.config2(3_000, seed=5)
    tarr = abi.array(abi.Topology, topos)
    planner.load(tarr, abi.array(abi.Scenario, scens))
    planner.evaluate()
    rows = planner.rows()
    cand = sorted(((r.throughput, i) for i, r in enumerate(rows[:planner.n_rows])
                   if r.feasible == 1 and 9 <= r.d <= 70), key=lambda x: (-x[0], x[1]))
    top = [i for _, i in cand[:3]]
    assert top
    for guard in (0.0, 0.5):
        pm = abi.PrefillModel.default(guard_ms=guard)
        hmax = max(rows[i].makespan_ns for i in top) / 1e6
        reqs = list(synthetic_requests(300, 11, hmax, pm))
        got, gpl = planner.pack_prefills(top, reqs, pm, placements=True)
        n = len(reqs)
        for k, i in enumerate(top):
            sc = scens[rows[i].scenario]
            want, wpl = checker.pack(tarr, sc, rows[i].d, reqs, pm)
            g = got[k]
            assert (g.accepted, g.placement_hash, g.utilization_after) == \
                (want.accepted, want.placement_hash, want.utilization_after), (k, guard)
            for a, b in zip(gpl[k * n:(k + 1) * n], wpl):
                assert (a.accepted, a.pipeline, a.start_ns) == (b.accepted, b.pipeline, b.start_ns)
        sat = checker.saturating(tarr, scens[rows[top[0]].scenario], rows[top[0]].d, pm)[:400]
        got, _ = planner.pack_prefills([top[0]], sat, pm)
        want, _ = checker.pack(tarr, scens[rows[top[0]].scenario], rows[top[0]].d, sat, pm,
                               placements=False)
        assert (got[0].accepted, got[0].placement_hash) == (want.accepted, want.placement_hash)


@pytest.mark.parametrize("wide", [False, True])
def test_saturating_requests_on_device(planner, checker, wide):
    """saturating_requests (bubbletea.cpp:240-267) computed on the device from
    the timeline's gap lists: the same requests (ids, arrival doubles, token
    counts) as the reference, at the makespan and at other horizons."""
    topos, scens = random_space(55 if wide else 56, 120, wide)
    rng = random.Random(4)
    pm = abi.PrefillModel.default()
    n = 0
    for i, r in _feasible_rows(planner, topos, scens, limit_gpus=2500):
        if rng.random() > 0.3:
            continue
        sc = scens[r.scenario]
        for hz in (0, max(1, r.makespan_ns // 3), r.makespan_ns + 7_000_001):
            got = [(q.id, q.arrival_ms, q.tokens) for q in planner.saturating_requests(i, pm, hz)]
            want = [(q.id, q.arrival_ms, q.tokens) for q in checker.saturating(topos, sc, r.d, pm, hz)]
            assert got == want, (i, r.d, hz, abi.POLICY_NAMES[sc.policy], len(got), len(want))
            n += 1
    assert n > 20
    # unit12 at M=5 (acceptance.cpp:221-252's stream)
    topos, sc = fixtures.unit12(M=5, policy="atlas")
    planner.load(topos, [sc])
    planner.evaluate()
    got = [(q.id, q.arrival_ms, q.tokens) for q in planner.saturating_requests(0, pm)]
    assert got == [(q.id, q.arrival_ms, q.tokens) for q in checker.saturating(topos, sc, 1, pm)]
    assert len(got) > 10


def test_allreduce_tail_on_device(planner, checker):
    """append_allreduce (scheduler.cpp:613-650) computed on the device: every
    stage's all-reduce start (the last backward end over all replicas) and
    duration equal the reference's on random spaces of every policy."""
    if not hasattr(checker, "allreduce_tail"):
        pytest.skip("needs the compiled reference (oracle/_ref)")
    for wide in (False, True):
        topos, scens = random_space(61 if wide else 62, 100, wide)
        rng = random.Random(6)
        n = 0
        for i, r in _feasible_rows(planner, topos, scens, limit_gpus=3000):
            if rng.random() > 0.3:
                continue
            sc = scens[r.scenario]
            assert planner.allreduce_tail(i) == checker.allreduce_tail(topos, sc, r.d), \
                (i, r.d, abi.POLICY_NAMES[sc.policy])
            n += 1
        assert n > 10
