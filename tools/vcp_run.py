"""The paper's VCP cases (Eq. VCP, P:l.685-694) on the GPU: factor + Krylov.
    python tools/vcp_run.py N eps"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth.problems import _grid_coords, grid_vcp  # noqa: E402
from paper_1510_07363_b200 import lorasp as L  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-3
dims = (N, N, N)
out = []
for case in (1, 2, 3):
    rp, ci, va = grid_vcp(dims, case)
    n = N ** 3
    depth = max(1, int(round(np.log2(n / 64))))
    sym = case != 3
    res = {"case": case, "n": n, "path": "SPD/PCG" if sym else "LU/GMRES"}
    try:
        h = L.Handle(n, rp, ci, _grid_coords(dims), depth=depth, eps=eps, flags=L.LORASP_SPD if sym else 0)
        h.factor(va)
        h.factor(va)
        b = np.sin(np.arange(n) * 0.1)
        x = np.zeros(n)
        rc, it, rr = h.krylov(b, x, 1e-10, method=L.LORASP_CG if sym else L.LORASP_GMRES, max_it=500)
        res.update(status=rc, iters=it, relres=rr, factor_ms=h.stats()["t_factor_host_ms"])
        h.close()
    except Exception as e:  # noqa: BLE001
        res.update(error=str(e)[:200])
    out.append(res)
print(json.dumps(out))
