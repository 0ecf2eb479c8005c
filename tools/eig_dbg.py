import sys, numpy as np
sys.path.insert(0,'.')
from paper_1510_07363_b200 import lorasp as L
rng = np.random.default_rng(0)
for m in [1, 2, 5, 33, 128]:
    M = rng.standard_normal((2*m, m)) @ np.diag(0.7**np.arange(m))
    sig, V, r, st = L.test_eig(M.T@M, 1e-2)
    so = np.linalg.svd(M, compute_uv=False)
    print(m, "st", st, "r", r, "sig", sig[:4], "ref", so[:4])
