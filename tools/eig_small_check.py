"""k_eig_small (m <= 64) against numpy and the production path through
lorasp_test_eig: ranks, sigma, subspace V_r V_r^T, timing (LORASP_EIG_PROFILE)."""
import os
import sys
import subprocess

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(small):
    env = dict(os.environ, LORASP_EIG_PROFILE="1")
    if small:
        env["LORASP_EIG_SMALL"] = "1"
    code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
from paper_1510_07363_b200 import lorasp as L
out = {}
for m in [5, 16, 24, 32, 33, 40, 48, 64]:
    rng = np.random.default_rng(m)
    Q1, _ = np.linalg.qr(rng.standard_normal((2 * m, m)))
    Q2, _ = np.linalg.qr(rng.standard_normal((m, m)))
    M = Q1 @ np.diag(0.8 ** np.arange(m)) @ Q2.T
    G = M.T @ M
    for rep in range(2):
        sig, V, r, st = L.test_eig(G, 1e-3)
    s = np.linalg.svd(M, compute_uv=False)
    _, _, Vt = np.linalg.svd(M)
    Vr = Vt[:r].T
    P1 = V[:, :r] @ V[:, :r].T; P2 = Vr @ Vr.T
    print(f"m={m} r={r} st={st} sigerr={np.max(np.abs(sig[:r]-s[:r]))/s[0]:.2e} proj={np.linalg.norm(P1-P2):.2e} orth={np.linalg.norm(V[:, :r].T@V[:, :r]-np.eye(r)):.2e}", flush=True)
'''
    return subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)


for small in (False, True):
    p = run(small)
    print("=== small" if small else "=== production")
    print("\n".join(l for l in (p.stdout + p.stderr).splitlines() if not l.strip().startswith("warp")))
