"""Profile one eigen-solve through the C-ABI hook: python tools/eig_one.py m [m ...] [--rank-frac f]
(LORASP_EIG_PROFILE=1 prints the per-phase cycle counts)."""
import sys
import time
import numpy as np
sys.path.insert(0, '.')
from paper_1510_07363_b200 import lorasp as L
args = [a for a in sys.argv[1:] if not a.startswith('--')]
frac = None
for a in sys.argv[1:]:
    if a.startswith('--rank-frac='):
        frac = float(a.split('=')[1])
rng = np.random.default_rng(0)
for m in [int(a) for a in args] or [128]:
    decay = 0.85 if frac is None else 1e-2 ** (1.0 / (frac * m))
    M = rng.standard_normal((2 * m, m)) @ np.diag(decay ** np.arange(m))
    G = M.T @ M
    eps = 1e-3 if frac is None else 1e-2
    L.test_eig(G, eps)
    t0 = time.perf_counter()
    sig, V, r, st = L.test_eig(G, eps)
    print("ok", m, r, st, f"{1e3 * (time.perf_counter() - t0):.2f} ms (hook wall, incl. alloc/copies)")
