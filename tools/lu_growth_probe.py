"""Largest no-pivot LU multiplier max|l_ij| seen by the LU-path pivot kernels, and
whether the handle switched to partial pivoting (stats lu_max_multiplier /
lu_partial_pivoting), on the LU-path workloads.   python tools/lu_growth_probe.py"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import make_problem  # noqa: E402
from synth.problems import _grid_coords, grid_vcp  # noqa: E402
from paper_1510_07363_b200 import lorasp as L  # noqa: E402

out = []
for name, kw in [("cfg5", {}), ("adv32", {"R": 1.0}), ("adv32", {"R": 1024.0})]:
    p = make_problem(name, **kw)
    h = L.analyze_problem(p)
    h.factor(p.values)
    st = h.stats()
    out.append({"config": name, **kw, "lu_max_multiplier": st["lu_max_multiplier"],
                "lu_partial_pivoting": st["lu_partial_pivoting"]})
    h.close()
for N, eps in [(16, 1e-3), (32, 1e-4)]:
    rp, ci, va = grid_vcp((N, N, N), 3)
    n = N ** 3
    h = L.Handle(n, rp, ci, _grid_coords((N, N, N)), depth=int(round(np.log2(n / 64))), eps=eps, flags=0)
    h.factor(va)
    st = h.stats()
    out.append({"config": f"vcp3 {N}^3 eps {eps}", "lu_max_multiplier": st["lu_max_multiplier"],
                "lu_partial_pivoting": st["lu_partial_pivoting"], "switches": st["lu_pivot_switches"]})
    h.close()
print(json.dumps(out, indent=1))
