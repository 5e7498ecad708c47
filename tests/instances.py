"""Seeded random plan spaces for parity tests.

Small instances follow the reference's own generator
(tests/support/instances.h:34-88: <=4 stages, <=3 pipelines, <=6
microbatches, latencies {0,5,10,40}, caps {1,2,5,10} Gbps); `wide=True`
widens every axis toward the BASELINE configs (more DCs, stages,
microbatches, TP, layer grouping, ratio-derived profiles, single TCP).
"""
from __future__ import annotations

import random

from paper_2411_14458_b200 import abi


def random_space(seed: int, n_scen: int, wide: bool = False):
    rng = random.Random(seed)
    topos, scens = [], []
    for _ in range(n_scen):
        if wide:
            n_dc = rng.randint(1, 5)
            counts = [rng.choice([2, 4, 6, 8, 12, 16, 24, 32, 48, 64]) for _ in range(n_dc)]
            lats = [0.0, 5.0, 10.0, 12.5, 20.0, 25.0, 40.0, 60.0, 80.0]
            lat = [[0.0] * n_dc for _ in range(n_dc)]
            for i in range(n_dc):
                for j in range(i + 1, n_dc):
                    lat[i][j] = lat[j][i] = rng.choice(lats)
            t = abi.make_topology(counts, cap_gbps=rng.choice([1.0, 2.5, 5.0, 10.0, 25.0]),
                                  intra_gbps=rng.choice([50.0, 100.0, 400.0]), latency=lat)
            S = rng.randint(1, 40)
            lpp = rng.choice([1, 1, 2, 3])
            layers = S * lpp - rng.randint(0, lpp - 1)
            M = rng.choice([1, 2, 3, 4, 5, 8, 12, 16, 24, 32])
            C = rng.randint(1, 4)
            tp = rng.choice([1, 1, 2])
            order = list(range(n_dc))
            if rng.random() < 0.5:
                rng.shuffle(order)
            elif rng.random() < 0.5:
                order = []
            hidden = rng.choice([256, 1024, 4096, 8192])
            seq = rng.choice([128, 1024, 4096, 8192])
            ratio = rng.choice([0.0, 0.0, 0.5, 1.0, 2.0, 3.0])
            f = rng.uniform(0.3, 30.0)
            sc = abi.make_scenario(
                topology=len(topos), policy=rng.choice(["gpipe", "1f1b", "varuna", "atlas"]),
                num_layers=layers, layers_per_partition=lpp, num_microbatches=M,
                hidden=hidden, seq_len=seq, fwd_ms=f, bwd_ms=f * rng.uniform(1.0, 2.5),
                recompute_ms=rng.choice([f, 0.0, f * 0.5]), ratio_C=ratio, C=C, tp=tp,
                dc_order=order, recompute=rng.random() < 0.7,
                multi_conn=rng.random() < 0.6,
                mem_limit=rng.choice([0, 0, 0, 1, 2, M, max(1, M // 2 + 1)]),
                d_max=rng.choice([0, 0, 0, 3]))
        else:
            S = rng.randint(1, 4)
            C = rng.randint(1, 3)
            D = rng.randint(1, 2)
            M = rng.randint(1, 6)
            dc_of = [0] * S
            for s in range(1, S):
                dc_of[s] = min(dc_of[s - 1] + rng.randint(0, 1), 2)
            n_dc = dc_of[-1] + 1
            counts = [0] * n_dc
            for d in dc_of:
                counts[d] += D * C
            t = abi.make_topology(counts, rng.choice([0.0, 5.0, 10.0, 40.0]),
                                  rng.choice([1.0, 2.0, 5.0, 10.0]))
            f = rng.uniform(0.3, 3.0)
            sc = abi.make_scenario(
                topology=len(topos), policy=rng.choice(["gpipe", "1f1b", "varuna", "atlas"]),
                num_layers=S, num_microbatches=M, hidden=256 << rng.randint(0, 3),
                seq_len=128 << rng.randint(0, 3), fwd_ms=f, bwd_ms=f * rng.uniform(1.0, 2.5),
                recompute_ms=f, C=C, dc_order=list(range(n_dc)),
                recompute=rng.random() < 0.5, multi_conn=rng.random() < 0.5,
                mem_limit=rng.choice([0, M, max(1, M // 2 + 1)]))
        topos.append(t)
        scens.append(sc)
    return abi.array(abi.Topology, topos), scens
