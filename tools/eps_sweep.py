"""Stand-alone direct-solver mode (x = Ã b, no Krylov) over a sequence of eps:
relative error against a reference solution and relative residual, with the
factorization time and the auxiliary-variable count — the paper's accuracy
study (P:l.641-649: error and residual proportional to eps).
    python tools/eps_sweep.py [cfg] [--frobenius] [eps ...]
--frobenius: the Frobenius truncation rule Eq. curOff6 (P:l.756-761, f2) instead of
Eq. cutOff1, with the paper's elasticity sequence eps = 1024e-7 ... 1e-7 by default;
each point also runs PCG to 1e-10 (iterations), as the paper's Table stiffness."""
import json
import os
import sys
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from synth import make_problem  # noqa: E402
from paper_1510_07363_b200 import lorasp as L  # noqa: E402

args = sys.argv[1:]
frob = "--frobenius" in args
args = [a for a in args if a != "--frobenius"]
cfg = args[0] if args else "cfg2"
eps_list = [float(a) for a in args[1:]] or (
    [1024e-7, 256e-7, 64e-7, 16e-7, 4e-7, 1e-7] if frob else [1e-1, 1e-2, 1e-3, 1e-4, 1e-5, 1e-6])
p = make_problem(cfg)
A = sp.csr_matrix((p.values, p.col_idx, p.row_ptr), shape=(p.n, p.n)).tocsc()
xs = spla.spsolve(A, p.b)                       # reference (sparse direct, host)
rows = []
for eps in eps_list:
    flags = (L.LORASP_SPD if p.symmetric else 0) | (L.LORASP_FROBENIUS if frob else 0)
    h = L.analyze_problem(p, eps=eps, flags=flags)
    vals = torch.tensor(p.values, device="cuda")
    h.factor(vals)
    h.factor(vals)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h.factor(vals)
    torch.cuda.synchronize()
    tf = time.perf_counter() - t0
    b = torch.tensor(p.b, device="cuda")
    x = torch.empty_like(b)
    h.apply(b, x)
    xv = x.cpu().numpy()
    xk = torch.zeros_like(b)
    rc, it, rr = h.krylov(b, xk, 1e-10, method=L.LORASP_CG if p.symmetric else L.LORASP_GMRES)
    rows.append({"eps": eps, "rel_error": float(np.linalg.norm(xv - xs) / np.linalg.norm(xs)),
                 "rel_residual": float(np.linalg.norm(p.b - A @ xv) / np.linalg.norm(p.b)),
                 "factor_ms": 1e3 * tf, "aux_vars": h.stats()["aux_vars"], "krylov_iters": it,
                 "krylov_status": rc})
    h.close()
print(json.dumps({"config": cfg, "n": p.n, "rule": "frobenius (Eq. curOff6)" if frob else "relative sigma (Eq. cutOff1)",
                  "sweep": rows}))
