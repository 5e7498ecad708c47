import sys
sys.path.insert(0, ".")
from paper_2411_14458_b200 import abi
from paper_2411_14458_b200.planner import Planner
from oracle import bindings
from tests import fixtures
chk = bindings.reference() or bindings.port()
p = Planner(0)
for pol in ("gpipe", "atlas"):
    topos, sc = fixtures.unit12(policy=pol)
    p.load(topos, [sc]); p.evaluate()
    pm = abi.PrefillModel.default()
    reqs = chk.saturating(topos, sc, 1, pm)
    got, gpl = p.pack_prefills([0], reqs, pm, placements=True)
    want, wpl = chk.pack(topos, sc, 1, reqs, pm)
    print(pol, len(reqs), "got acc", got[0].accepted, "want", want.accepted)
    nbad = 0
    for i, (a, b) in enumerate(zip(gpl[:len(reqs)], wpl)):
        if (a.accepted, a.pipeline, a.start_ns) != (b.accepted, b.pipeline, b.start_ns):
            print(" req", i, reqs[i].arrival_ms, reqs[i].tokens, "got", (a.accepted, a.pipeline, a.start_ns), "want", (b.accepted, b.pipeline, b.start_ns))
            nbad += 1
            if nbad > 6: break
