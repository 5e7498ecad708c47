"""Host-side plan-space generators for the BASELINE configs (no GPU): exact
row counts, the axes each config states, shards that cover
a space exactly once, and the reference's own d_max default."""
import pytest

from paper_2411_14458_b200 import workloads


def _n_dc(t):
    return t.n_dc


@pytest.mark.parametrize("n_rows", [1, 999, 10_000])
def test_config2_rows_exact(n_rows):
    topos, scens = workloads.config2(n_rows)
    assert workloads.count_rows(scens) == n_rows
    assert {t.n_dc for t in topos} == {3}
    assert {s.num_layers for s in scens} == {80}


def test_config3_shards_cover_space():
    full_t, full_s = workloads.config3(20_000)
    assert workloads.count_rows(full_s) == 20_000
    parts = [workloads.config3(20_000, shard=r, n_shards=3) for r in range(3)]
    assert sum(workloads.count_rows(s) for _, s in parts) == 20_000
    assert sum(len(s) for _, s in parts) == len(full_s)
    assert {t.n_dc for t in full_t} == {5}


def test_config5_axes_and_shards():
    topos, scens = workloads.config5(200_000, seed=5)
    assert workloads.count_rows(scens) == 200_000
    assert {t.n_dc for t in topos} == set(range(2, 9))
    assert {s.num_microbatches for s in scens} == {4, 8, 16, 32, 64, 128, 256}
    assert {s.num_layers for s in scens} == {m[1] for m in workloads.CONFIG5_MODELS}
    for t in topos[:200]:
        counts = [t.gpu_count[i] for i in range(t.n_dc)]
        assert all(c % 64 == 0 and 64 <= c <= 1024 for c in counts)
        for i in range(t.n_dc):
            for j in range(t.n_dc):
                assert t.latency_ms[i][j] == t.latency_ms[j][i]
    for s, t in zip(scens[:500], [topos[s.topology] for s in scens[:500]]):
        P = -(-s.num_layers // s.layers_per_partition)
        dflt = max(1, sum(t.gpu_count[i] for i in range(t.n_dc)) //
                   (s.pipelines_per_cell * P * s.tp_degree))
        assert s.d_max <= dflt  # dc_select.cpp:20-25 (only the last scenario is clipped)
        assert sorted(s.dc_order[i] for i in range(s.n_order)) == list(range(t.n_dc))
    parts = [workloads.config5(200_000, seed=5, shard=r, n_shards=4) for r in range(4)]
    assert sum(workloads.count_rows(s) for _, s in parts) == 200_000


def test_config5_capped_sample():
    topos, scens = workloads.config5(1500, seed=11, max_rows_per_scenario=3)
    assert workloads.count_rows(scens) == 1500
    assert max(s.d_max for s in scens) <= 3
