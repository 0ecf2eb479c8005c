"""Exchange volume of the distributed factorization and apply, emulated with G
virtual ranks on one GPU (paper_1510_07363_b200.dist.VirtualGroup): per rank,
the bytes the neighbour push sends per factorization (blocks only to their
reader ranks; records stay local) against the single-GPU factor bytes, the
vector bytes of one distributed apply, and a check that every rank's Ã b equals
the single-GPU one bit for bit (reference without the split apply, which the
distributed apply does not use).
    python tools/dist_volume.py cfg2 2 4 8"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import make_problem  # noqa: E402
from paper_1510_07363_b200 import lorasp as L  # noqa: E402
from paper_1510_07363_b200.dist import VirtualGroup, factor_virtual, run_virtual  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
worlds = [int(a) for a in sys.argv[2:]] or [2, 4, 8]
p = make_problem(cfg)
os.environ["LORASP_NO_SPLIT_APPLY"] = "1"
h1 = L.analyze_problem(p)
del os.environ["LORASP_NO_SPLIT_APPLY"]
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

    def apply(r, h):
        x = np.zeros(p.n)
        h.apply(p.b, x)
        return x

    xs, errs = run_virtual(hs, apply)
    assert errs == [None] * G, errs
    sts = [h.stats() for h in hs]
    push = [st["dist_allgather_bytes"] for st in sts]
    out["worlds"][G] = {"collective_calls": sts[0]["dist_exchange_calls"],
                        "push_bytes_per_rank": push,
                        "push_max_over_factor_bytes": max(push) / fb,
                        "apply_vector_bytes_per_rank": [st["dist_apply_bytes"] for st in sts],
                        "apply_calls": sts[0]["dist_apply_calls"],
                        "bit_identical_to_1gpu": all(bool(np.array_equal(x, x1)) for x in xs)}
    for h in hs:
        h.close()
print(json.dumps(out))
