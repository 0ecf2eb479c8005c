"""Phase timings (clock64 cycles) of the compress eigen-solver on one Gram matrix
through the C-ABI hook lorasp_test_eig with LORASP_EIG_PROFILE=1 (printed by the
library on stderr): tridiagonalisation, lambda_0, the other eigenvalues, inverse
iteration, MGS, back-transformation.  Spectrum sigma_k = 0.8^k (rank ~31 at
eps = 1e-3), m in argv (default 128)."""
import os
import sys

import numpy as np

os.environ["LORASP_EIG_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_07363_b200 import lorasp as L  # noqa: E402

for m in [int(a) for a in sys.argv[1:]] or [128]:
    rng = np.random.default_rng(m)
    Q1, _ = np.linalg.qr(rng.standard_normal((2 * m, m)))
    Q2, _ = np.linalg.qr(rng.standard_normal((m, m)))
    M = Q1 @ np.diag(0.8 ** np.arange(m)) @ Q2.T
    sig, V, r, st = L.test_eig(M.T @ M, 1e-3)
    print(f"m={m} r={r} status={st} sigma0={sig[0]:.3f}", flush=True)
