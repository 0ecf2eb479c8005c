import sys, numpy as np
sys.path.insert(0,'.')
from paper_1510_07363_b200 import lorasp as L
rng = np.random.default_rng(0)
for m in [8, 32, 64, 128, 150]:
    M = rng.standard_normal((2*m, m)) @ np.diag(0.7**np.arange(m))
    G = M.T @ M
    sig, V, r, st = L.test_eig(G, 1e-2)
    so = np.linalg.svd(M, compute_uv=False)
    ro = int((so >= 1e-2*so[0]).sum())
    _, _, Vt = np.linalg.svd(M)
    P1 = V @ V.T; P2 = Vt[:ro].T @ Vt[:ro]
    print(m, "st", st, "r", r, ro, "sig err", np.abs(sig[:m]-so[:m]).max()/so[0], "proj err", np.abs(P1-P2).max() if r==ro else None, "orth", np.abs(V.T@V-np.eye(r)).max())
    # pivot
    Sx = rng.standard_normal((m, m)); S = Sx@Sx.T + m*np.eye(m)
    rr = max(1, m//3); Vq,_ = np.linalg.qr(rng.standard_normal((m, rr)))
    n = m+rr; K = np.zeros((n,n)); K[:m,:m]=S; K[m:,:m]=Vq.T; K[:m,m:]=Vq
    Li, st = L.test_pivot(K, m, rr)
    Lf = np.linalg.inv(Li); D = np.diag([1]*m+[-1]*rr)
    print("  pivot st", st, "recon", np.abs(Lf@D@Lf.T - K).max()/np.abs(K).max(), "upper zero", np.abs(np.triu(Li,1)).max())
