import sys, numpy as np
sys.path.insert(0,'.')
from paper_1510_07363_b200 import lorasp as L
rng = np.random.default_rng(0)
for m in [int(a) for a in sys.argv[1:]] or [128]:
    M = rng.standard_normal((2*m, m)) @ np.diag(0.85**np.arange(m))
    sig, V, r, st = L.test_eig(M.T @ M, 1e-3)
    print("ok", m, r, st)
