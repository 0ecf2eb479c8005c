import sys, os, time, numpy as np, torch, ctypes
sys.path.insert(0,'.')
from paper_1510_07363_b200 import lorasp as L
rng = np.random.default_rng(0)
for m in [16, 25, 40, 64, 100, 128]:
    M = rng.standard_normal((2*m, m)) @ np.diag(0.8**np.arange(m))
    G = M.T @ M
    L.test_eig(G, 1e-3)
    torch.cuda.synchronize(); t=time.perf_counter()
    for _ in range(5): sig, V, r, st = L.test_eig(G, 1e-3)
    dt=(time.perf_counter()-t)/5
    print(os.environ.get("LORASP_EIG_GENERIC","warp/reg"), m, r, "wall ms (incl. mallocs)", round(dt*1e3,3))
