"""Phase cycles of the small eigen-solvers (k_eig_warp m <= 32, k_tridiag_reg +
k_eig_t m <= 128) on one Gram matrix with a graded spectrum (kept rank ~ f m):
python tools/eig_small_profile.py m..."""
import os
import sys

import numpy as np

os.environ["LORASP_EIG_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_07363_b200 import lorasp as L  # noqa: E402

eps, f = 1e-3, float(os.environ.get("RANK_FRAC", "0.5"))
for m in [int(a) for a in sys.argv[1:]] or [24]:
    rng = np.random.default_rng(m)
    Q1, _ = np.linalg.qr(rng.standard_normal((2 * m, m)))
    Q2, _ = np.linalg.qr(rng.standard_normal((m, m)))
    M = Q1 @ np.diag(eps ** (np.arange(m) / (f * m))) @ Q2.T
    for rep in range(2):
        sig, V, r, st = L.test_eig(M.T @ M, eps)
    print(f"m={m} r={r} status={st}", flush=True)
