"""CPU (gloo, world_size 2): the plan-space sharding and the best-plan
all-gather used by bench.py at N>1 (the only collective on the path)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_14458_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, recs, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        thr, row = recs[rank]
        local = D.encode_best(thr, row)
        q.put((rank, D.global_best(local, world)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("recs,want", [
    ([(1.5, 10), (2.5, 3)], (1, 2.5, 3)),
    ([(2.5, 7), (2.5, 3)], (0, 2.5, 7)),      # tie: lower rank wins
    ([(0.0, -1), (0.5, 0)], (1, 0.5, 0)),     # rank 0 has no feasible plan
    ([(0.0, -1), (0.0, -1)], (-1, 0.0, -1)),
])
def test_global_best_gloo(recs, want):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, recs, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, res in got:
        assert res == want, (rank, res)


def test_shards_cover_exactly():
    for n in (0, 1, 7, 197, 1000):
        for world in (1, 2, 3, 4, 8):
            spans = [D.shard_scenarios(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b


def test_encode_roundtrip():
    for thr, row in ((0.0, -1), (1.2345678901234567, 99), (1e-300, 2 ** 40)):
        assert D.decode_best(D.encode_best(thr, row)) == (thr, row)


def _shard_worker(rank, world, port, q):
    """One rank of a sharded whatif: evaluate this rank's cost shard with the
    C port (oracle: select() per scenario, dc_select.cpp:99-123), map the
    local winner to its global row, all-gather the 16-byte winners."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import bindings
    from paper_2411_14458_b200 import abi
    from tests.instances import random_space
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        topos, scens = random_space(2024, 60, wide=True)
        for s in scens:  # resolve d_max like the workloads generators do
            s.d_max = len(bindings.port().select(topos, s)[0])
        shard = D.shard_by_cost(scens, world)[rank]
        grows = D.global_rows(scens, shard)
        chk = bindings.port()
        rows = [r for i in shard for r in chk.select(topos, scens[i])[0]]
        best = (0.0, -1)
        for k, r in enumerate(rows):
            if r.feasible == 1 and (best[1] < 0 or r.throughput > best[0]):
                best = (r.throughput, k)
        local = D.encode_best(best[0], grows[best[1]] if best[1] >= 0 else -1)
        out = D.all_gather_best(local, world)
        recs = [D.decode_best(out[2 * r: 2 * r + 2]) for r in range(world)]
        q.put((rank, D.reduce_best_global(recs), len(rows)))
    finally:
        dist.destroy_process_group()


def test_sharded_whatif_gloo():
    """World size 2: cost-balanced shards of one plan space, each evaluated
    on its own rank; the merged winner equals one whatif() over the whole
    space (max throughput, first row on ties)."""
    from oracle import bindings
    from tests.instances import random_space
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    topos, scens = random_space(2024, 60, wide=True)
    chk = bindings.port()
    rows = [r for s in scens for r in chk.select(topos, s)[0]]
    want = (0.0, -1)
    for k, r in enumerate(rows):
        if r.feasible == 1 and (want[1] < 0 or r.throughput > want[0]):
            want = (r.throughput, k)
    assert want[1] >= 0
    assert sum(n for _, _, n in got) == len(rows)
    for rank, res, _ in got:
        assert res == want, (rank, res, want)


def test_shard_by_cost_balanced():
    from paper_2411_14458_b200 import workloads
    topos, scens = workloads.config2(20_000, seed=1)
    for world in (1, 2, 4, 8):
        shards = D.shard_by_cost(scens, world)
        assert sorted(i for s in shards for i in s) == list(range(len(scens)))
        loads = [sum(D.row_cost(scens[i]) * scens[i].d_max for i in s) for s in shards]
        assert max(loads) <= 1.05 * (sum(loads) / world) + max(
            D.row_cost(s) * s.d_max for s in scens)
        rows = [D.global_rows(scens, s) for s in shards]
        assert sorted(r for x in rows for r in x) == list(range(sum(s.d_max for s in scens)))
