"""Plan-space sharding across GPUs and the global best-plan exchange.

Plans are independent ("Per-D evaluations are independent"), so
N ranks (one process per GPU, torch.distributed) each evaluate their own
shard of the plan space with no data-path collective. The only exchange is
the K7 step of SURVEY.md §2: every rank contributes its 16-byte gpb_best
record (throughput, row) and one all-gather (NCCL over NVLink on GPUs, gloo
in the CPU tests) gives every rank the same global winner.

Shards: whole scenarios (select()'s per-scenario argmax
stays local), dealt by estimated cost — the same per-row cost model the
library buckets by (ATLAS ~ C*M*(2000*C + 250*S), flush/1F1B ~ 20*M*S cycles)
times the scenario's row count — longest first onto the least-loaded rank
(LPT). Each rank keeps its scenarios in space order, so mapping a rank's
local winner row back to its global row index and keying the winners by
(throughput desc, global row asc) reproduces exactly the choice of one
whatif() over the whole space (first maximum in row order).
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


def row_cost(sc) -> float:
    """Estimated cycles of one row of scenario `sc` (host.cu's bucket model)."""
    S = -(-sc.num_layers // sc.layers_per_partition)
    C, M = sc.pipelines_per_cell, sc.num_microbatches
    if sc.policy == 3:
        return float(C * M * (2000 * C + 250 * S))
    return float(20 * M * S)


def shard_by_cost(scens, world: int):
    """Cost-balanced scenario shards: list of `world` index lists, each in
    space order. Scenario i carries d_max(i) rows (scens must have d_max
    resolved, as the workloads generators set it)."""
    order = sorted(range(len(scens)), key=lambda i: (-row_cost(scens[i]) * scens[i].d_max, i))
    load = [0.0] * world
    out = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        load[r] += row_cost(scens[i]) * scens[i].d_max
        out[r].append(i)
    for lst in out:
        lst.sort()
    return out


def global_rows(scens, shard):
    """Global row index of every local row of a shard (rows of a scenario are
    D = 1..d_max, scenarios in space order)."""
    first = [0] * (len(scens) + 1)
    for i, sc in enumerate(scens):
        first[i + 1] = first[i] + sc.d_max
    out = []
    for i in shard:
        out.extend(range(first[i], first[i + 1]))
    return out


def reduce_best_global(records):
    """records: (throughput, global row) per rank (row < 0: none) -> the
    global best (throughput, row): max throughput, lowest row on ties."""
    best = (0.0, -1)
    for thr, row in records:
        if row < 0:
            continue
        if best[1] < 0 or thr > best[0] or (thr == best[0] and row < best[1]):
            best = (thr, row)
    return best


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
