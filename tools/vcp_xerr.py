"""x = Ã b of the GPU against the C++ oracle on the paper's VCP cases at 16^3
(the quantity tests/test_gpu_vcp.py bounds): python tools/vcp_xerr.py [eps]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import cpp_oracle as CO  # noqa: E402
from synth.problems import _grid_coords, grid_vcp  # noqa: E402
from paper_1510_07363_b200 import lorasp as L  # noqa: E402

eps = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-3
N = 16
dims = (N, N, N)
for case in (1, 2, 3):
    rp, ci, va = grid_vcp(dims, case)
    n = N ** 3
    depth = int(round(np.log2(n / 64)))
    xy = _grid_coords(dims)
    sym = case != 3
    h = L.Handle(n, rp, ci, xy, depth=depth, eps=eps, flags=L.LORASP_SPD if sym else 0)
    h.factor(va)
    f = CO.factorize(n, rp, ci, va, xy, depth, eps)
    b = np.sin(np.arange(n) * 0.1)
    x = np.zeros(n)
    h.apply(b, x)
    xo = CO.solve(f, b)
    nd = sum(int(np.sum(h.ranks(i) != f.ranks(i))) for i in range(1, depth + 1))
    print(f"case {case} eps {eps:g}: |x - xo| / |xo| = {np.linalg.norm(x - xo) / np.linalg.norm(xo):.3e}, "
          f"nodes with a different rank {nd}", flush=True)
    h.close()
