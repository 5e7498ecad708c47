"""CPU: the C oracle (oracle/geopipe_oracle.c) pinned against the
reference's golden vectors and known-answer tests, and against fixtures
frozen from the compiled reference (tests/golden/)."""
import math

import pytest

from oracle import bindings
from paper_2411_14458_b200 import abi
from tests import fixtures, golden_io


@pytest.fixture(scope="module")
def port():
    return bindings.port()


def _ms(port, topos, sc):
    rows, _, _ = port.select(topos, sc)
    return rows[0].pp_time_ms


def test_unit12_makespans(port):
    # test_scheduler.cpp:53-63
    for pol, ms in (("gpipe", 38.0), ("1f1b", 39.0), ("varuna", 38.0), ("atlas", 36.0)):
        topos, sc = fixtures.unit12(policy=pol)
        assert _ms(port, topos, sc) == ms


def test_atlas_mem_limits(port):
    # test_scheduler.cpp:175-196
    for ml, ms in ((1, 89.0), (2, 67.0), (6, 36.0)):
        topos, sc = fixtures.unit12(policy="atlas", mem_limit=ml)
        assert _ms(port, topos, sc) == ms


def test_two_stage_hand_checkable(port):
    # test_scheduler.cpp:154-173: 9 ms without recompute, 12 ms with
    topo = abi.make_topology([2], 0.0, 5.0)
    for pol in ("gpipe", "1f1b", "varuna", "atlas"):
        for rec, ms in ((False, 9.0), (True, 12.0)):
            sc = abi.make_scenario(policy=pol, num_layers=2, hidden=1000, seq_len=625,
                                   num_microbatches=2, fwd_ms=1.0, bwd_ms=2.0, recompute_ms=1.0,
                                   dc_order=[0], d_max=1, recompute=rec)
            assert _ms(port, abi.array(abi.Topology, [topo]), sc) == ms


def test_no_wan_compute_bound(port):
    # test_engine.cpp:87-99: 27 ms for all policies
    topo = abi.make_topology([12], 0.0, 5.0)
    for pol in ("gpipe", "1f1b", "varuna", "atlas"):
        sc = abi.make_scenario(policy=pol, num_layers=6, hidden=1000, seq_len=625,
                               num_microbatches=4, C=2, dc_order=[0], d_max=1)
        assert _ms(port, abi.array(abi.Topology, [topo]), sc) == 27.0


def test_atlas_rank1_start_and_pooling(port):
    # test_scheduler.cpp:80-106: rank 1 starts at 4 ms; pooled 1 ms vs 2 ms
    topos, sc = fixtures.unit12(policy="atlas")
    tasks, ms = port.timeline(topos, sc, 1)
    f0 = [t for t in tasks if t.kind == 0 and t.stage == 0 and t.microbatch == 0]
    starts = sorted((t.pipeline, t.start) for t in f0)
    assert starts == [(0, 0), (1, 4_000_000)]


def test_single_conn_much_slower(port):
    # test_scheduler.cpp:214-226
    topos, sc = fixtures.wan12(policy="gpipe", multi_conn=True)
    fast = _ms(port, topos, sc)
    topos, sc = fixtures.wan12(policy="gpipe", multi_conn=False)
    assert _ms(port, topos, sc) > 5.0 * fast


def test_config1_kats(port):
    # SURVEY.md §8(c), from the compiled reference
    kat = {("1f1b", False): 28344.858980, ("1f1b", True): 2470.61274,
           ("gpipe", False): 44295.774368, ("gpipe", True): 2896.980384,
           ("atlas", False): 45335.774368, ("atlas", True): 3936.980384}
    for (pol, multi), ms in kat.items():
        topos, sc = fixtures.config1(pol, multi)
        assert abs(_ms(port, topos, sc) - ms) < 5e-7


def test_unit12_utilization_and_bubbles(port):
    # atlas util 1/3, 32 bubbles (gpu4 windows); varuna 54
    topos, sc = fixtures.unit12(policy="atlas")
    rows, _, _ = port.select(topos, sc)
    assert rows[0].utilization == 0.33333333333333331
    b = port.bubbles(topos, sc, 1)
    assert len(b) == 32
    assert [x for x in b if x[0] == 4] == [(4, 0, 3_000_000), (4, 7_000_000, 18_000_000),
                                           (4, 26_000_000, 36_000_000)]
    topos, sc = fixtures.unit12(policy="varuna")
    rows, _, _ = port.select(topos, sc)
    assert rows[0].utilization == 0.31578947368421056
    assert len(port.bubbles(topos, sc, 1)) == 54


def test_tcp_table_bit_exact(port):
    # acceptance criterion 2 / test_comm_model.cpp:24-31, 63-69
    t = abi.make_topology([1], 0.0, 5.0)
    for lat, mbps in ((10, 1220), (20, 600), (30, 396), (40, 293)):
        assert port.single_tcp_bandwidth(t, lat) == mbps * 125.0
    assert port.single_tcp_bandwidth(t, 80.0) == 36625.0 * 40.0 / 80.0
    assert port.single_tcp_bandwidth(t, 0.1) == 1220 * 125.0


def test_bubble_filling_acceptance(port):
    # acceptance.cpp:221-252: util 0.3846 -> 0.9986
    topos, sc = fixtures.unit12(M=5, policy="atlas")
    pm = abi.PrefillModel.default()
    reqs = port.saturating(topos, sc, 1, pm)
    s, _ = port.pack(topos, sc, 1, reqs, pm)
    assert 0.37 <= s.utilization_before <= 0.53 and s.utilization_after >= 0.90
    assert s.accepted == 32


def test_prefill_overhead():
    # acceptance criterion 9: 32 boundaries ~85.90 ms
    bytes_ = 1 * 8192 * 4096 * 2
    ms32 = 32 * (0.0 + bytes_ / 25000000.0)
    assert 84.0 <= ms32 <= 88.0


@pytest.fixture(scope="module")
def golden():
    return golden_io.load()


def test_golden_rows(port, golden):
    n = 0
    for sp, topos, scens in golden:
        for entry, sc in zip(sp["scenarios"], scens):
            if "error" in entry:
                with pytest.raises(bindings.CheckerError):
                    port.select(topos, sc)
                continue
            rows, chosen, used = port.select(topos, sc)
            assert chosen == entry["chosen_d"] and used == entry["gpus_used"]
            for r, g in zip(rows, entry["rows"]):
                d, feas, ch, pp, ar, tot, thr, parts, util = g
                assert (r.d, r.feasible, r.chosen) == (d, feas, ch)
                assert r.pp_time_ms == golden_io.unhex(pp)
                assert r.allreduce_time_ms == golden_io.unhex(ar)
                assert r.total_time_ms == golden_io.unhex(tot)
                assert r.throughput == golden_io.unhex(thr)
                assert list(r.partitions) == parts
                if feas:
                    assert r.utilization == golden_io.unhex(util)
                n += 1
    assert n > 400


def test_golden_bubbles_and_packs(port, golden):
    import hashlib
    import json
    nb = npk = 0
    for sp, topos, scens in golden:
        for b in sp["bubbles"]:
            got = port.bubbles(topos, scens[b["scenario"]], b["d"], b["horizon"])
            assert [list(x) for x in got] == b["bubbles"]
            nb += 1
        for pk in sp["packs"]:
            pm = abi.PrefillModel.default(inference_layers=pk["inference_layers"])
            reqs = [abi.Request(id=i, tokens=t, arrival_ms=golden_io.unhex(a))
                    for i, t, a in pk["requests"]]
            s, pl = port.pack(topos, scens[pk["scenario"]], pk["d"], reqs, pm)
            ub, ua, acc, rej, hz, h = pk["summary"]
            assert (s.accepted, s.rejected, s.horizon_ns, str(s.placement_hash)) == (acc, rej, hz, h)
            assert s.utilization_before == golden_io.unhex(ub)
            assert s.utilization_after == golden_io.unhex(ua)
            dig = hashlib.sha256(json.dumps(
                [[p.accepted, p.pipeline, p.start_ns, float(p.ttft_overhead_ms).hex()] for p in pl]
            ).encode()).hexdigest()
            assert dig == pk["placements_sha256"]
            npk += 1
    assert nb > 10 and npk > 10


def test_port_vs_compiled_reference():
    ref = bindings.reference()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    from tests.instances import random_space
    port = bindings.port()
    topos, scens = random_space(2024, 60, True)
    for sc in scens:
        try:
            a = port.select(topos, sc)
        except bindings.CheckerError as e:
            with pytest.raises(bindings.CheckerError):
                ref.select(topos, sc)
            continue
        b = ref.select(topos, sc)
        assert a[1:] == b[1:]
        for x, y in zip(a[0], b[0]):
            assert (x.pp_time_ms, x.throughput, x.chosen, list(x.partitions)) == \
                (y.pp_time_ms, y.throughput, y.chosen, list(y.partitions))
