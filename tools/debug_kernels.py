import sys, numpy as np
sys.path.insert(0,'.')
from paper_1510_07363_b200 import lorasp as L
rng = np.random.default_rng(0)
def check(M, eps, tag):
    m = M.shape[1]
    G = M.T @ M
    sig, V, r, st = L.test_eig(G, eps)
    so = np.linalg.svd(M, compute_uv=False)
    so = np.concatenate([so, np.zeros(m - so.size)])
    ro = int((so >= eps*so[0]).sum())
    w, Q = np.linalg.eigh(G); Q = Q[:, ::-1]
    P2 = Q[:, :ro] @ Q[:, :ro].T
    pe = np.abs(V @ V.T - P2).max() if r == ro else None
    k = min(r+1, m)
    print(f"{tag:28s} m={m:4d} st={st} r={r} ro={ro} sigerr={np.abs(sig[:k]-so[:k]).max()/so[0]:.2e} proj={pe if pe is None else f'{pe:.2e}'} orth={np.abs(V.T@V-np.eye(r)).max():.2e}")
for m in [1, 2, 3, 8, 32, 64, 128, 150, 200, 300]:
    M = rng.standard_normal((2*m, m)) @ np.diag(0.7**np.arange(m))
    check(M, 1e-2, "decay0.7 eps1e-2")
for m in [64, 128]:
    M = rng.standard_normal((m//2, m))          # rank deficient (R < m)
    check(M, 1e-3, "rankdef eps1e-3")
    U,_ = np.linalg.qr(rng.standard_normal((m, m))); W,_ = np.linalg.qr(rng.standard_normal((m,m)))
    s = np.concatenate([np.ones(5), 1e-4*np.ones(5), 10.0**-np.arange(6, 6+m-10)])
    check(U @ np.diag(s) @ W.T, 1e-3, "clusters eps1e-3")
    s = 10.0**(-6*np.arange(m)/m)
    check(U @ np.diag(s) @ W.T, 1e-3, "slow decay eps1e-3")
# pivot kernel, small and large n (large path is exercised through the factor tests)
for m, rr in [(100, 40), (150, 10)]:
    Sx = rng.standard_normal((m, m)); S = Sx@Sx.T + m*np.eye(m)
    Vq,_ = np.linalg.qr(rng.standard_normal((m, rr)))
    n = m+rr; K = np.zeros((n,n)); K[:m,:m]=S; K[m:,:m]=Vq.T; K[:m,m:]=Vq
    Li, st = L.test_pivot(K, m, rr)
    Lf = np.linalg.inv(Li); D = np.diag([1]*m+[-1]*rr)
    print("pivot n", n, "st", st, "recon", np.abs(Lf@D@Lf.T - K).max()/np.abs(K).max())
for m, rr in [(1, 0), (5, 3), (16, 0), (17, 4), (100, 28), (128, 32), (140, 20), (120, 40)]:
    Sx = rng.standard_normal((m, m)); S = Sx@Sx.T + m*np.eye(m)
    n = m+rr; K = np.zeros((n,n)); K[:m,:m]=S
    if rr:
        Vq,_ = np.linalg.qr(rng.standard_normal((m, rr)))
        K[m:,:m]=Vq.T; K[:m,m:]=Vq
    Li, st = L.test_pivot(K, m, rr)
    Lf = np.linalg.inv(Li); D = np.diag([1]*m+[-1]*rr)
    print("pivot_blk n", n, "st", st, "recon", np.abs(Lf@D@Lf.T - K).max()/np.abs(K).max(), "upper", np.abs(np.triu(Li,1)).max())
