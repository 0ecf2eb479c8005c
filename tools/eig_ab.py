"""A/B numerics of the eigen-solver between two builds of liblorasp.so:
    python tools/eig_ab.py [path/to/liblorasp.so]
Prints, per m, the kept-subspace error |V V^T - P_r| of the clustered /
degenerate spectrum (tests/test_gpu_eig.py) and of the graded stack, and the
orthonormality |V^T V - I|."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_07363_b200 import lorasp as L  # noqa: E402

L.load(sys.argv[1] if len(sys.argv) > 1 else None)
for m in [128, 129, 160, 200, 256, 300, 312, 400, 500]:
    rng = np.random.default_rng(7)
    s = np.concatenate([np.full(m // 4, 3.0), np.full(m // 4, 1.0), np.zeros(m - 2 * (m // 4))])
    Q1, _ = np.linalg.qr(rng.standard_normal((2 * m, m)))
    Q2, _ = np.linalg.qr(rng.standard_normal((m, m)))
    M = (Q1 * s) @ Q2.T
    sig, V, r, st = L.test_eig(M.T @ M, 0.2)
    _, _, Vt = np.linalg.svd(M)
    Pr = Vt[:r].T @ Vt[:r]
    e1 = np.max(np.abs(V @ V.T - Pr))
    o1 = np.max(np.abs(V.T @ V - np.eye(r)))
    rng = np.random.default_rng(m)
    Q1, _ = np.linalg.qr(rng.standard_normal((2 * m, m)))
    Q2, _ = np.linalg.qr(rng.standard_normal((m, m)))
    M = Q1 @ np.diag(1e-3 ** (np.arange(m) / (0.5 * m))) @ Q2.T
    sig, V, r2, st2 = L.test_eig(M.T @ M, 1e-2)
    _, sv, Vt = np.linalg.svd(M)
    Pr = Vt[:r2].T @ Vt[:r2]
    e2 = np.max(np.abs(V @ V.T - Pr))
    o2 = np.max(np.abs(V.T @ V - np.eye(r2)))
    print(f"m={m:4d} degenerate r={r} st={st} subspace {e1:.2e} orth {o1:.2e} | graded r={r2} st={st2} "
          f"subspace {e2:.2e} orth {o2:.2e} sig {np.max(np.abs(sig[:r2] - sv[:r2])) / sv[0]:.2e}", flush=True)
