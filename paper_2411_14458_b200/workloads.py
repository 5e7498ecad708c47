"""Synthetic plan spaces for the BASELINE.json configs.

The reference defines no plan-space generator; these restate the configs'
axes literally. Scenario draws use Python's MT19937 (``random.Random(seed)``)
index picks; every scenario expands to all of its D rows (D = 1..d_max,
dc_select.cpp:99-104) and the last scenario's d_max is clipped so a space has
exactly the requested number of rows.
"""
from __future__ import annotations

import itertools
import random

from . import abi

POLICY_LIST = ["gpipe", "1f1b", "varuna", "atlas"]


def _d_max_default(counts, C, P, tp):
    return max(1, sum(counts) // (C * P * tp))


def config1(policy="1f1b", multi_conn=True):
    """Config 1: 4-stage PP over 2 DCs, 8 microbatches, 96 MiB activations,
    15/30/15 ms compute, 40 ms WAN, 5 Gbps cap (single plan)."""
    topo = abi.make_topology([2, 2], 40.0, 5.0)
    sc = abi.make_scenario(policy=policy, num_layers=4, hidden=8192, seq_len=6144,
                           num_microbatches=8, fwd_ms=15.0, bwd_ms=30.0, recompute_ms=15.0,
                           C=1, dc_order=[0, 1], d_max=1, multi_conn=multi_conn)
    return [topo], [sc]


def config2(n_rows=10_000, seed=1):
    """Config 2: Llama-3 70B plan search over 3 DCs [1024, 768, 512]."""
    lat_axis = [10.0, 20.0, 30.0, 40.0, 60.0, 80.0]
    lpp_axis = [1, 2, 4, 5, 8, 10, 16, 20]
    C_axis = [1, 2, 3, 4]
    tp_axis = [1, 2, 4, 8]
    M_axis = [4, 8, 16, 32, 64]
    ratio_axis = [1.0, 2.0, 3.0]
    orders = list(itertools.permutations(range(3)))
    counts = [1024, 768, 512]
    rng = random.Random(seed)
    topos, scens, rows = [], [], 0
    while rows < n_rows:
        pick = lambda axis: axis[rng.randrange(len(axis))]  # noqa: E731
        lat = [[0.0] * 3 for _ in range(3)]
        for i, j in ((0, 1), (0, 2), (1, 2)):
            lat[i][j] = lat[j][i] = pick(lat_axis)
        topos.append(abi.make_topology(counts, cap_gbps=5.0, intra_gbps=100.0, latency=lat))
        lpp, C, tp, M = pick(lpp_axis), pick(C_axis), pick(tp_axis), pick(M_axis)
        ratio, pol, multi, order = pick(ratio_axis), pick(POLICY_LIST), pick([0, 1]), pick(orders)
        P = (80 + lpp - 1) // lpp
        d_max = _d_max_default(counts, C, P, tp)
        if rows + d_max > n_rows:
            d_max = n_rows - rows
        scens.append(abi.make_scenario(
            topology=len(topos) - 1, policy=pol, num_layers=80, layers_per_partition=lpp,
            num_microbatches=M, hidden=8192, seq_len=8192, ratio_C=ratio, C=C, tp=tp,
            d_max=d_max, dc_order=list(order), multi_conn=multi))
        rows += d_max
    return topos, scens


def config3(n_rows=1_000_000, seed=2, shard=0, n_shards=1):
    """Config 3: Llama-3.1 405B over DC-set-2 [600, 500, 400, 300, 200] with a
    latency x cap x multi_conn WAN grid; `shard` selects every n_shards-th
    scenario (plans are independent)."""
    lat_axis = [5.0, 10.0, 20.0, 40.0, 80.0, 160.0]
    cap_axis = [1.0, 2.5, 5.0, 10.0, 25.0]
    lpp_axis = [1, 2, 3, 6, 7, 9, 14, 18]
    C_axis = [1, 2, 3, 4]
    tp_axis = [1, 2, 4, 8]
    M_axis = [4, 8, 16, 32, 64]
    ratio_axis = [1.0, 2.0, 3.0]
    counts = [600, 500, 400, 300, 200]
    orders = list(itertools.permutations(range(5)))
    rng = random.Random(seed)
    topos, scens, rows, k = [], [], 0, 0
    while rows < n_rows:
        pick = lambda axis: axis[rng.randrange(len(axis))]  # noqa: E731
        lat = [[0.0] * 5 for _ in range(5)]
        for i in range(5):
            for j in range(i + 1, 5):
                lat[i][j] = lat[j][i] = pick(lat_axis)
        cap = pick(cap_axis)
        lpp, C, tp, M = pick(lpp_axis), pick(C_axis), pick(tp_axis), pick(M_axis)
        ratio, pol, multi, order = pick(ratio_axis), pick(POLICY_LIST), pick([0, 1]), pick(orders)
        P = (126 + lpp - 1) // lpp
        d_max = _d_max_default(counts, C, P, tp)
        if rows + d_max > n_rows:
            d_max = n_rows - rows
        rows += d_max
        mine = k % n_shards == shard
        k += 1
        if not mine:
            continue
        topos.append(abi.make_topology(counts, cap_gbps=cap, intra_gbps=100.0, latency=lat))
        scens.append(abi.make_scenario(
            topology=len(topos) - 1, policy=pol, num_layers=126, layers_per_partition=lpp,
            num_microbatches=M, hidden=16384, seq_len=8192, ratio_C=ratio, C=C, tp=tp,
            d_max=d_max, dc_order=list(order), multi_conn=multi))
    return topos, scens


# (name, layers, hidden, seq_len): GPT-A / GPT-B are the paper's baseline
# models (L,H = 4K,4K and 6K,8K; their layer counts are not
# given there: 24 and 48 here), Llama-3 70B and Llama-3.1 405B as above.
CONFIG5_MODELS = [("gpt-a", 24, 4096, 4096), ("gpt-b", 48, 8192, 6144),
                  ("llama3-70b", 80, 8192, 8192), ("llama3.1-405b", 126, 16384, 8192)]


def config5(n_rows=10_000_000, seed=5, shard=0, n_shards=1, max_rows_per_scenario=0):
    """Config 5: the full sweep — random topologies of 2-8 DCs with
    64..1024 GPUs each (step 64), the four models, microbatches 4-256, and
    every other axis of config 3; `shard` selects every n_shards-th scenario.
    `max_rows_per_scenario` > 0 caps each scenario's D range (parity samples)."""
    lat_axis = [5.0, 10.0, 20.0, 40.0, 80.0, 160.0]
    cap_axis = [1.0, 2.5, 5.0, 10.0, 25.0]
    lpp_axis = [1, 2, 3, 4, 6, 8, 12, 16]
    C_axis = [1, 2, 3, 4]
    tp_axis = [1, 2, 4, 8]
    M_axis = [4, 8, 16, 32, 64, 128, 256]
    ratio_axis = [1.0, 2.0, 3.0]
    rng = random.Random(seed)
    topos, scens, rows, k = [], [], 0, 0
    while rows < n_rows:
        pick = lambda axis: axis[rng.randrange(len(axis))]  # noqa: E731
        n_dc = 2 + rng.randrange(7)
        counts = [64 * (1 + rng.randrange(16)) for _ in range(n_dc)]
        lat = [[0.0] * n_dc for _ in range(n_dc)]
        for i in range(n_dc):
            for j in range(i + 1, n_dc):
                lat[i][j] = lat[j][i] = pick(lat_axis)
        cap = pick(cap_axis)
        _, layers, hidden, seq = pick(CONFIG5_MODELS)
        lpp, C, tp, M = pick(lpp_axis), pick(C_axis), pick(tp_axis), pick(M_axis)
        ratio, pol, multi = pick(ratio_axis), pick(POLICY_LIST), pick([0, 1])
        order = list(range(n_dc))
        rng.shuffle(order)
        P = (layers + lpp - 1) // lpp
        d_max = _d_max_default(counts, C, P, tp)
        if max_rows_per_scenario > 0:
            d_max = min(d_max, max_rows_per_scenario)
        if rows + d_max > n_rows:
            d_max = n_rows - rows
        rows += d_max
        mine = k % n_shards == shard
        k += 1
        if not mine:
            continue
        topos.append(abi.make_topology(counts, cap_gbps=cap, intra_gbps=100.0, latency=lat))
        scens.append(abi.make_scenario(
            topology=len(topos) - 1, policy=pol, num_layers=layers, layers_per_partition=lpp,
            num_microbatches=M, hidden=hidden, seq_len=seq, ratio_C=ratio, C=C, tp=tp,
            d_max=d_max, dc_order=order, multi_conn=multi))
    return topos, scens


def count_rows(scens):
    return sum(s.d_max for s in scens)
