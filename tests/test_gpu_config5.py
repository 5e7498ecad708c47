"""GPU parity on BASELINE config 5's shapes (workloads.config5): random
topologies of 2-8 DCs, GPT-A/GPT-B/70B/405B, microbatches 4-256, every
policy — all rows bit-exact with the reference (oracle/_ref), plus the
largest ATLAS cell the sweep holds (405B at one layer per stage: 126 stages,
8 DCs, 4 pipelines, 256 microbatches)."""
import pytest

from paper_2411_14458_b200 import abi, workloads
from tests.test_gpu_rows import _compare_space

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [11, 12])
def test_config5_sample_bit_exact(planner, checker, seed):
    from oracle import bindings
    topos, scens = workloads.config5(1500, seed=seed, max_rows_per_scenario=3)
    topos = abi.array(abi.Topology, topos)
    assert {t.n_dc for t in topos} >= {2, 8}
    assert max(s.num_microbatches for s in scens) == 256
    assert _compare_space(planner, checker, bindings.port(), topos, scens) == 1500


def test_config5_largest_atlas_cell(planner, checker):
    from oracle import bindings
    n = 8
    lat = [[0.0 if i == j else 10.0 * (1 + abs(i - j)) for j in range(n)] for i in range(n)]
    topo = abi.make_topology([1024, 896, 768, 640, 512, 384, 256, 128], cap_gbps=5.0, latency=lat)
    scens = []
    for pol in ("atlas", "gpipe", "1f1b", "varuna"):
        for multi in (0, 1):
            scens.append(abi.make_scenario(
                topology=0, policy=pol, num_layers=126, layers_per_partition=1,
                num_microbatches=256, hidden=16384, seq_len=8192, ratio_C=2.0, C=4, tp=1,
                d_max=2, dc_order=list(range(n)), multi_conn=multi))
    topos = abi.array(abi.Topology, [topo])
    assert _compare_space(planner, checker, bindings.port(), topos, scens) == 2 * len(scens)


def test_grouped_rows_bit_exact(planner, checker, monkeypatch):
    """Large spaces evaluate shallow gpipe/varuna/1f1b rows several per warp
    (flush_group_kernel / onef1b_group_kernel, S <= 8 / 16); force it on a
    small space and check every row against the reference."""
    from oracle import bindings
    monkeypatch.setenv("GPB_GROUP_FLUSH_MIN_ROWS", "0")
    topos, scens = workloads.config5(4000, seed=21, max_rows_per_scenario=4)
    scens = [s for s in scens if s.policy in (0, 1, 2)]
    topos = abi.array(abi.Topology, topos)
    scens = abi.array(abi.Scenario, scens)
    assert sum(1 for s in scens if -(-s.num_layers // s.layers_per_partition) <= 8) > 50
    assert _compare_space(planner, checker, bindings.port(), topos, scens) > 1500


def test_atlas_seq_rows_bit_exact(planner, checker, monkeypatch):
    """Large spaces run ATLAS rows of shallow pipelines (S <= 16) one per
    thread (atlas_seq_kernel); force it on small spaces — config-5 shapes,
    the unit12 KATs with memory caps, random caps/latencies — and check every
    row against the reference (select() + report() on run())."""
    import random
    from oracle import bindings
    from tests import fixtures
    monkeypatch.setenv("GPB_GROUP_FLUSH_MIN_ROWS", "0")
    monkeypatch.setenv("GPB_ATLAS_SEQ", "2")
    for ml, ms in ((1, 89.0), (2, 67.0), (6, 36.0), (0, 36.0)):
        topos, sc = fixtures.unit12(policy="atlas", mem_limit=ml)
        assert planner.select(topos, sc).rows[0].pp_time_ms == ms
    topos, scens = workloads.config5(3000, seed=31, max_rows_per_scenario=3)
    scens = [s for s in scens if s.policy == 3
             and -(-s.num_layers // s.layers_per_partition) <= 16]
    assert len(scens) > 100
    topos = abi.array(abi.Topology, topos)
    assert _compare_space(planner, checker, bindings.port(), topos,
                          abi.array(abi.Scenario, scens)) > 300
    rng = random.Random(8)
    topos, scens = [], []
    for _ in range(120):
        n_dc = rng.randint(2, 6)
        counts = [rng.choice([64, 128, 256]) for _ in range(n_dc)]
        lat = [[0.0] * n_dc for _ in range(n_dc)]
        for i in range(n_dc):
            for j in range(i + 1, n_dc):
                lat[i][j] = lat[j][i] = rng.choice([0.0, 5.0, 20.0, 80.0])
        topos.append(abi.make_topology(counts, cap_gbps=rng.choice([1.0, 5.0, 25.0]),
                                       intra_gbps=100.0, latency=lat))
        S = rng.randint(2, 16)
        scens.append(abi.make_scenario(
            topology=len(topos) - 1, policy="atlas", num_layers=S,
            num_microbatches=rng.choice([1, 3, 8, 33, 64]),
            hidden=rng.choice([512, 4096]), seq_len=rng.choice([512, 4096]),
            fwd_ms=rng.uniform(0.5, 20.0), bwd_ms=rng.uniform(1.0, 40.0),
            recompute_ms=rng.uniform(0.0, 10.0), C=rng.choice([1, 2, 3, 4, 6]),
            recompute=rng.random() < 0.5, multi_conn=rng.random() < 0.5,
            mem_limit=rng.choice([0, 1, 2, 3, S]), d_max=rng.choice([1, 2]),
            dc_order=list(range(n_dc))))
    assert _compare_space(planner, checker, bindings.port(), abi.array(abi.Topology, topos),
                          abi.array(abi.Scenario, scens)) >= 120
