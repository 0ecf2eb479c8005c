import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from synth import make_problem, csr_to_dense
from oracle import lorasp_oracle as O
from paper_1510_07363_b200 import lorasp as L
for dims, depth, eps in [((16,16),4,0.0), ((32,32),6,0.0), ((32,32),6,1e-2)]:
    p = make_problem("cfg1", dims=dims, depth=depth)
    h = L.analyze_problem(p, eps=eps)
    t=time.time(); h.factor(torch.tensor(p.values, device="cuda")); torch.cuda.synchronize(); tf=time.time()-t
    b = torch.tensor(p.b, device="cuda"); x = torch.empty_like(b)
    h.apply(b, x); x = x.cpu().numpy()
    f = O.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, depth, eps)
    xo = O.solve(f, p.b)
    print(dims, eps, "tf", round(tf,4), "relerr vs oracle", np.linalg.norm(x-xo)/np.linalg.norm(xo), flush=True)
    for i in range(depth, 0, -1):
        g = h.ranks(i); o = [f.rank.get((i,c),0) for c in range(2**(i-1))]
        print("  level", i, "gpu", list(g)[:12], "oracle", o[:12], "eq", list(g)==o)
    print(h.stats())
