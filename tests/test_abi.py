"""CPU: the C-ABI library loads and exports every entry point declared in
include/*.h; host-side pieces (libm bandwidth table, exact repeated sum,
request generator) agree with the reference; no silent CPU fallback."""
import ctypes as C
import glob
import os
import random
import re

import pytest

from paper_2411_14458_b200 import abi
from paper_2411_14458_b200 import planner as pl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b((?:gpb|gp)_[a-z_0-9]+)\s*\(", text):
            syms.add(m.group(1))
    return sorted(syms)


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(pl.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_repeated_sum_matches_sequential():
    lib = pl.load_library()
    rng = random.Random(0)
    cases = [(1 / 3, 12), (0.31578947368421056, 19), (0.1, 1000), (0.7, 2304)]
    for _ in range(3000):
        u = rng.choice([rng.random(), 1 - rng.random() * 1e-6, rng.random() * 1e-3,
                        (rng.randint(1, 1000)) / rng.randint(1, 1000)])
        cases.append((min(u, 1.0), rng.randint(1, 5000)))
    for u, G in cases:
        s = 0.0
        for _ in range(G):
            s += u
        assert lib.gpb_repeated_sum_host(u, G) == s, (u, G)


def test_single_tcp_bandwidth_matches_checkers():
    from oracle import bindings
    lib = pl.load_library()
    t = abi.make_topology([1], 0.0, 5.0)
    chk = bindings.reference() or bindings.port()
    for lat in [0.1, 9.99, 10, 12, 12.5, 17.3, 20, 25, 29.9, 30, 35, 40, 41, 80, 400]:
        assert lib.gpb_single_tcp_bandwidth(C.byref(t), lat) == chk.single_tcp_bandwidth(t, lat)


def test_synthetic_requests_match_reference():
    from oracle import bindings
    ref = bindings.reference()
    if ref is None:
        pytest.skip("compiled reference not built")
    pm = abi.PrefillModel.default()
    for seed, n, h in ((42, 500, 1000.0), (7, 50, 0.0), (1, 1, 5.5)):
        a = list(pl.synthetic_requests(n, seed, h, pm))
        b = ref.synthetic(n, seed, h, pm)
        assert [(x.id, x.tokens, x.arrival_ms) for x in a] == \
            [(x.id, x.tokens, x.arrival_ms) for x in b]


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pl.GeopipeError):
        pl.Planner(0)
