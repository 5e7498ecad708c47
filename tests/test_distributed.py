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
