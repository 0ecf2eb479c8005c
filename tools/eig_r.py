import sys, numpy as np
sys.path.insert(0, '.')
from paper_1510_07363_b200 import lorasp as L
m, r_target, eps = int(sys.argv[1]), int(sys.argv[2]), 1e-3
rng = np.random.default_rng(1)
decay = eps ** (1.0 / r_target)
M = rng.standard_normal((2 * m, m)) @ np.diag(decay ** np.arange(m))
G = M.T @ M
for _ in range(2):
    sig, V, r, st = L.test_eig(G, eps)
print("ok", m, r)
