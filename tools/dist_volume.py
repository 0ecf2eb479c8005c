"""Exchange volume of the distributed factorization, emulated with G virtual
ranks on one GPU (paper_1510_07363_b200.dist.VirtualGroup): per rank, the
collective calls and the bytes all-gathered per factorization, plus a check
that every rank's Ã b equals the single-GPU one bit for bit.
    python tools/dist_volume.py cfg2 2 4 8"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import make_problem  # noqa: E402
from paper_1510_07363_b200 import lorasp as L  # noqa: E402
from paper_1510_07363_b200.dist import VirtualGroup, factor_virtual  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
worlds = [int(a) for a in sys.argv[2:]] or [2, 4, 8]
p = make_problem(cfg)
h1 = L.analyze_problem(p)
h1.factor(p.values)
x1 = np.zeros(p.n)
h1.apply(p.b, x1)
fb = h1.stats()["factor_bytes"]
h1.close()
out = {"config": cfg, "n": p.n, "factor_bytes": fb, "worlds": {}}
for G in worlds:
    hs = [L.analyze_problem(p) for _ in range(G)]
    errs = factor_virtual(hs, p.values, VirtualGroup(G))
    assert errs == [None] * G, errs
    st = hs[0].stats()
    same = True
    for h in hs:
        x = np.zeros(p.n)
        h.apply(p.b, x)
        same &= bool(np.array_equal(x, x1))
    out["worlds"][G] = {"collective_calls": st["dist_exchange_calls"],
                        "allgather_bytes_per_rank": st["dist_allgather_bytes"],
                        "allgather_over_factor_bytes": st["dist_allgather_bytes"] / fb,
                        "bit_identical_to_1gpu": same}
    for h in hs:
        h.close()
print(json.dumps(out))
