"""Plan-space sharding across GPUs and the global best-plan exchange.

Plans are independent ("Per-D evaluations are independent"), so
N ranks (one process per GPU, torch.distributed) each evaluate their own
shard of the plan space with no data-path collective. The only exchange is
the K7 step of SURVEY.md §2: every rank contributes its 16-byte gpb_best
record (throughput, row) and one all-gather (NCCL over NVLink on GPUs, gloo
in the CPU tests) gives every rank the same global winner, keyed by
(throughput desc, rank asc, row asc) — the sequential order of a whatif()
over the concatenated shards.
"""
from __future__ import annotations

import struct

import torch
import torch.distributed as dist


def shard_scenarios(n_scen: int, rank: int, world: int):
    """Contiguous scenario ranges: rank r owns [lo, hi). Keeping a
    scenario's D rows on one rank keeps select()'s per-scenario argmax
    local."""
    base, extra = divmod(n_scen, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def decode_best(raw: torch.Tensor):
    """A gpb_best record (double throughput, int64 row) from 2 int64 words."""
    words = [int(x) for x in raw.tolist()]
    thr = struct.unpack("<d", struct.pack("<q", words[0]))[0]
    return thr, words[1]


def encode_best(thr: float, row: int, device="cpu") -> torch.Tensor:
    w0 = struct.unpack("<q", struct.pack("<d", thr))[0]
    return torch.tensor([w0, row], dtype=torch.int64, device=device)


def reduce_best(records):
    """records: list of (throughput, row) per rank -> (rank, throughput, row)
    of the global best; rows < 0 mean 'no feasible plan'."""
    best = None
    for rank, (thr, row) in enumerate(records):
        if row < 0:
            continue
        key = (-thr, rank, row)
        if best is None or key < best[0]:
            best = (key, rank, thr, row)
    if best is None:
        return -1, 0.0, -1
    return best[1], best[2], best[3]


def all_gather_best(local: torch.Tensor, world: int, out: torch.Tensor | None = None):
    """All-gather of the 16-byte per-rank winners (one collective)."""
    if out is None:
        out = torch.empty(2 * world, dtype=torch.int64, device=local.device)
    dist.all_gather_into_tensor(out, local)
    return out


def global_best(local: torch.Tensor, world: int):
    gathered = all_gather_best(local, world)
    recs = [decode_best(gathered[2 * r: 2 * r + 2].cpu()) for r in range(world)]
    return reduce_best(recs)
