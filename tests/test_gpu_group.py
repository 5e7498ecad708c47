"""GPU: one plan space sharded over several devices through the C ABI
(gpb_group_*) gives exactly the single-device answer: every
row (bytes), every scenario's choice, and the global winner (whatif() over
the whole space, dc_select.cpp:125-134). On a one-GPU box the group is two
or three contexts on device 0 (winners exchanged through the host); with two
or more GPUs the NCCL all-gather path runs too."""
import pytest

from paper_2411_14458_b200 import abi, workloads
from paper_2411_14458_b200.planner import PlannerGroup
from tests.instances import random_space

pytestmark = pytest.mark.gpu


def _single(planner, topos, scens):
    planner.load(topos, scens)
    planner.evaluate()
    rows = [bytes(r) for r in planner.rows()[: planner.n_rows]]
    res = [bytes(r) for r in planner.scenario_results()[: planner.n_scen]]
    b = planner.best()
    return rows, res, (b.throughput, b.row)


def _group(devices, topos, scens):
    g = PlannerGroup(devices)
    try:
        g.load(topos, scens)
        g.evaluate()
        rows = [bytes(r) for r in g.rows()[: g.n_rows]]
        res = [bytes(r) for r in g.scenario_results()[: g.n_scen]]
        b = g.best()
        return rows, res, (b.throughput, b.row)
    finally:
        g.close()


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0]])
def test_group_same_device_matches_single(planner, devices):
    for space in (random_space(31, 150, wide=True), workloads.config2(10_000, seed=3)):
        topos = abi.array(abi.Topology, space[0])
        scens = abi.array(abi.Scenario, space[1])
        assert _group(devices, topos, scens) == _single(planner, topos, scens)


def test_group_errors_match_single(planner):
    topos, scens = random_space(32, 20, wide=False)
    scens = abi.array(abi.Scenario, scens)
    scens[7].pipelines_per_cell = 0
    g = PlannerGroup([0, 0])
    try:
        with pytest.raises(Exception) as eg:
            g.load(topos, scens)
    finally:
        g.close()
    with pytest.raises(Exception) as es:
        planner.load(topos, scens)
    assert (type(eg.value), str(eg.value)) == (type(es.value), str(es.value))


def test_group_all_devices_nccl(planner):
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("one GPU: the NCCL exchange needs two devices")
    topos, scens = workloads.config2(20_000, seed=4)
    topos, scens = abi.array(abi.Topology, topos), abi.array(abi.Scenario, scens)
    assert _group(list(range(n)), topos, scens) == _single(planner, topos, scens)
