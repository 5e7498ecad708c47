"""Fixture builders restating the reference's tests/support/fixtures.h
(make_topology :18-36, unit12 :44-62, five_dc :71-89, growth :95-105,
wan12 :113-131) and the BASELINE config-1 plan."""
from paper_2411_14458_b200 import abi


def unit12(M=4, policy="atlas", C=2, **kw):
    topo = abi.make_topology([4, 4, 4], 0.0, 5.0)
    sc = abi.make_scenario(policy=policy, num_layers=6, hidden=1000, seq_len=625,
                           num_microbatches=M, fwd_ms=1.0, bwd_ms=1.0, recompute_ms=1.0,
                           C=C, dc_order=[0, 1, 2], d_max=1, **kw)
    return abi.array(abi.Topology, [topo]), sc


def wan12(policy="gpipe", **kw):
    topo = abi.make_topology([6, 3, 3], 40.0, 5.0)
    sc = abi.make_scenario(policy=policy, num_layers=4, hidden=8192, seq_len=6144,
                           num_microbatches=4, fwd_ms=15.0, bwd_ms=30.0, recompute_ms=15.0,
                           C=3, dc_order=[0, 1, 2], d_max=1, **kw)
    return abi.array(abi.Topology, [topo]), sc


def five_dc(num_dcs=5, C=3, policy="atlas"):
    topo = abi.make_topology([600] * num_dcs, 20.0, 5.0)
    sc = abi.make_scenario(policy=policy, num_layers=60, hidden=6144, seq_len=4608,
                           num_microbatches=5, fwd_ms=10.0, bwd_ms=20.0, recompute_ms=10.0,
                           C=C)
    return abi.array(abi.Topology, [topo]), sc


def growth(dc1_gpus, C=2, policy="atlas"):
    counts = [600] if dc1_gpus <= 0 else [600, dc1_gpus]
    topo = abi.make_topology(counts, 40.0, 5.0)
    sc = abi.make_scenario(policy=policy, num_layers=60, hidden=6144, seq_len=2048,
                           num_microbatches=6, fwd_ms=10.0, bwd_ms=20.0, recompute_ms=10.0,
                           C=C)
    return abi.array(abi.Topology, [topo]), sc


def config1(policy="1f1b", multi_conn=True):
    """BASELINE config 1: 4-stage PP over 2 DCs, M=8, 96 MiB activations,
    15/30/15 ms, 40 ms WAN at a 5 Gbps cap."""
    topo = abi.make_topology([2, 2], 40.0, 5.0)
    sc = abi.make_scenario(policy=policy, num_layers=4, hidden=8192, seq_len=6144,
                           num_microbatches=8, fwd_ms=15.0, bwd_ms=30.0, recompute_ms=15.0,
                           C=1, tp=1, dc_order=[0, 1], d_max=1, multi_conn=multi_conn)
    return abi.array(abi.Topology, [topo]), sc
