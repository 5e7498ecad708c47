"""GPU parity beyond config 2's shapes: a stratified sample of BASELINE config
3 (Llama-3.1 405B over 5 DCs, 10^6 rows evaluated in one launch sequence) and
random ATLAS stress shapes (up to 126 stages = 4 stages per lane, 256
microbatches, 8 pipelines, small memory caps), every sampled row bit-exact
against the reference's select(), utilization and makespan against its
report() on run()."""
from concurrent.futures import ThreadPoolExecutor
import os
import random

import pytest

from paper_2411_14458_b200 import abi, workloads

pytestmark = pytest.mark.gpu


def _key(r):
    return (r.d, r.feasible, r.chosen, r.pp_time_ms, r.allreduce_time_ms, r.total_time_ms,
            r.throughput, tuple(r.partitions))


def _check_sample(planner, checker, topos, scens, idx):
    tarr = abi.array(abi.Topology, topos)
    rows = planner.rows()
    res = planner.scenario_results()
    def ref_scenario(i):
        sel = checker.select(tarr, scens[i])
        return sel, checker.report_rows(tarr, scens[i], len(sel[0]))

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        ref = list(ex.map(ref_scenario, idx))
    n = 0
    for i, ((ref_rows, chosen, used), rep) in zip(idx, ref):
        r0 = res[i].first_row
        assert (res[i].n_rows, res[i].chosen_d, res[i].gpus_used) == (len(ref_rows), chosen, used), i
        for k, (b, (util, mk)) in enumerate(zip(ref_rows, rep)):
            a = rows[r0 + k]
            assert _key(a) == _key(b), (i, k + 1, abi.POLICY_NAMES[scens[i].policy])
            # report() on run(): utilization and makespan (metrics.cpp:39-54)
            assert (a.utilization, a.makespan_ns) == (util, mk), (i, k + 1)
            n += 1
    return n


def test_config3_sample_bit_exact(planner, checker):
    topos, scens = workloads.config3(1_000_000, seed=2)
    assert planner.load(abi.array(abi.Topology, topos), abi.array(abi.Scenario, scens)) == 1_000_000
    planner.evaluate()
    rng = random.Random(17)
    by_pol = {}
    for i, sc in enumerate(scens):
        by_pol.setdefault(sc.policy, []).append(i)
    idx = []
    for pol, lst in sorted(by_pol.items()):  # stratified by policy
        idx += rng.sample(lst, 40)
    assert _check_sample(planner, checker, topos, scens, idx) > 160


def test_atlas_stress_shapes(planner, checker):
    rng = random.Random(5)
    topos, scens = [], []
    for _ in range(48):
        n_dc = rng.randint(2, 5)
        counts = [rng.choice([64, 128, 256, 512]) for _ in range(n_dc)]
        lat = [[0.0] * n_dc for _ in range(n_dc)]
        for i in range(n_dc):
            for j in range(i + 1, n_dc):
                lat[i][j] = lat[j][i] = rng.choice([5.0, 20.0, 40.0, 80.0])
        topos.append(abi.make_topology(counts, cap_gbps=rng.choice([1.0, 5.0, 25.0]),
                                       intra_gbps=100.0, latency=lat))
        S = rng.choice([33, 64, 97, 126])
        M = rng.choice([16, 64, 128, 256])
        C = rng.choice([1, 2, 4, 8])
        scens.append(abi.make_scenario(
            topology=len(topos) - 1, policy="atlas", num_layers=S, num_microbatches=M,
            hidden=rng.choice([1024, 4096]), seq_len=rng.choice([1024, 4096]),
            fwd_ms=rng.uniform(1.0, 20.0), bwd_ms=rng.uniform(2.0, 40.0),
            recompute_ms=rng.uniform(0.0, 10.0), C=C, recompute=rng.random() < 0.5,
            multi_conn=rng.random() < 0.5, mem_limit=rng.choice([0, 1, 2, 8, S]),
            d_max=1, dc_order=list(range(n_dc))))
    planner.load(abi.array(abi.Topology, topos), abi.array(abi.Scenario, scens))
    planner.evaluate()
    assert _check_sample(planner, checker, topos, scens, list(range(len(scens)))) == len(scens)
