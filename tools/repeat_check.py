"""Bitwise repeatability stress: N re-factorizations (rank-predicted sweep and
recorded graph) + applies + Krylov solves must reproduce the first result.
    python tools/repeat_check.py cfg2 20"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from synth import make_problem  # noqa: E402
from paper_1510_07363_b200 import lorasp as L  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
p = make_problem(cfg)
h = L.analyze_problem(p)
vals = torch.tensor(p.values, device="cuda")
b = torch.tensor(p.b, device="cuda")
ref = None
bad = 0
for k in range(reps):
    h.factor(vals)
    x = torch.empty_like(b)
    h.apply(b, x)
    xk = torch.zeros_like(b)
    rc, it, rr = h.krylov(b, xk, 1e-10, method=L.LORASP_CG if p.symmetric else L.LORASP_GMRES)
    cur = (x.cpu().numpy(), xk.cpu().numpy(), it)
    if ref is None:
        ref = cur
    elif not (np.array_equal(cur[0], ref[0]) and np.array_equal(cur[1], ref[1]) and cur[2] == ref[2]):
        bad += 1
print(cfg, "reps", reps, "mismatches", bad, "graph", h.stats()["factor_graph"])
