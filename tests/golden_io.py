"""Loader for tests/golden/reference_spaces.json (see make_golden.py)."""
import json
import os

from paper_2411_14458_b200 import abi

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_spaces.json")


def _fill(struct, d):
    for name, ctype in struct._fields_:
        v = d[name]
        if isinstance(v, list):
            arr = getattr(struct, name)
            for i, x in enumerate(v):
                if isinstance(x, list):
                    for j, y in enumerate(x):
                        arr[i][j] = y
                else:
                    arr[i] = x
        else:
            setattr(struct, name, v)
    return struct


def load():
    with open(PATH) as f:
        doc = json.load(f)
    spaces = []
    for sp in doc["spaces"]:
        topos = abi.array(abi.Topology, [_fill(abi.Topology(), t) for t in sp["topologies"]])
        scens = [_fill(abi.Scenario(), s["scenario"]) for s in sp["scenarios"]]
        spaces.append((sp, topos, scens))
    return spaces


def unhex(x):
    return float.fromhex(x)
