"""Write the full-size oracle goldens tests/golden/fullsize_<cfg>.npz.

Calls ONLY oracle/ (the C++17 LAPACK-free oracle, oracle/cpp_oracle.py) and the
seeded generators in synth/ -- never the CUDA path.  For each BASELINE config
(cfg2 256^2, cfg3 64^3, cfg4 128^3, cfg5 1024^2) at its full size and eps:

  ranks        int16, every node's retained rank, level-major (i = 1..l, c = 0..2^(i-1)-1)
  near_*       nodes whose oracle sigma_r or sigma_{r+1} lies within 1e-9 (relative
               to sigma_0) of the threshold, with that gap (north_star rank exception,
               reading Z22: a rank mismatch is excused iff gap <= 1e-12)
  order_crc    crc32 of each level's processing order (int64 cluster ids)
  x_idx/x_val  x = Ã b (Alg. 2-4) at 16384 seeded sample indices
  x_norm       ||x||_2;  x_proj = W x for 8 seeded Gaussian rows W (default_rng(1510))
  kry_*        PCG (cfg2-4) / GMRES(50) (cfg5) from x0 = 0 to 1e-10: iterations,
               true relative residual, converged flag; paper residual Eq. GMRES_residual
  meta         json: config, n, depth, eps, oracle source sha256, threads, seconds

Usage: python tools/make_goldens.py cfg3 [cfg4 ...]   (threads: ORACLE_THREADS, default nproc)
"""
import hashlib
import json
import os
import sys
import time
import zlib

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import cpp_oracle as CO  # noqa: E402
from synth import make_problem  # noqa: E402

NSAMPLE = 16384
NPROJ = 8


def sample_indices(n):
    rng = np.random.default_rng(7363)
    return np.sort(rng.choice(n, size=min(n, NSAMPLE), replace=False)).astype(np.int64)


def projection_rows(n):
    return np.random.default_rng(1510).standard_normal((NPROJ, n))


def make(name):
    p = make_problem(name)
    t0 = time.time()
    f = CO.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, p.depth, p.eps)
    t_factor = time.time() - t0
    ranks, near_l, near_c, near_gap, crcs = [], [], [], [], []
    for i in range(1, p.depth + 1):
        r = f.ranks(i)
        ranks.append(r.astype(np.int16))
        seq, _ = f.level_order(i)
        crcs.append(zlib.crc32(np.ascontiguousarray(seq, dtype=np.int64).tobytes()))
        for c in range(r.size):
            s = f.sigma_of(i, c)
            if s.size == 0 or s[0] <= 0:
                continue
            gaps = [abs(s[k] / s[0] - p.eps) for k in (r[c] - 1, r[c]) if 0 <= k < s.size]
            if gaps and min(gaps) <= 1e-9:
                near_l.append(i), near_c.append(c), near_gap.append(min(gaps))
    t1 = time.time()
    x = CO.solve(f, p.b)
    t_solve = time.time() - t1
    t2 = time.time()
    kr = CO.krylov(f, p.row_ptr, p.col_idx, p.values, p.b, method=p.solver, tol=1e-10, restart=50, maxit=500)
    t_kry = time.time() - t2
    paper_res = CO.paper_preconditioned_residual(f, p.row_ptr, p.col_idx, p.values, p.b, kr.x)
    idx = sample_indices(p.n)
    sha = hashlib.sha256(open(CO.SRC, "rb").read()).hexdigest()
    meta = {"config": name, "n": p.n, "depth": p.depth, "eps": p.eps, "solver": p.solver,
            "oracle": "oracle/cpp/lorasp_oracle.cpp", "oracle_sha256": sha, "threads": f.threads,
            "t_factor_s": t_factor, "t_solve_s": t_solve, "t_krylov_s": t_kry, "info": f.info(),
            "rank_sum": int(sum(int(r.astype(np.int64).sum()) for r in ranks))}
    out = os.path.join(ROOT, "tests", "golden", f"fullsize_{name}.npz")
    np.savez_compressed(
        out, ranks=np.concatenate(ranks), near_level=np.array(near_l, np.int32), near_c=np.array(near_c, np.int64),
        near_gap=np.array(near_gap), order_crc=np.array(crcs, np.int64), x_idx=idx, x_val=x[idx],
        x_norm=np.array(np.linalg.norm(x)), x_proj=projection_rows(p.n) @ x, kry_iters=np.array(kr.iters),
        kry_relres=np.array(kr.relres), kry_converged=np.array(kr.converged), paper_residual=np.array(paper_res),
        meta=np.array(json.dumps(meta)))
    f.close()
    print(json.dumps(meta), "iters", kr.iters, "relres", kr.relres, "near", len(near_l), flush=True)


if __name__ == "__main__":
    for name in sys.argv[1:] or ["cfg2", "cfg3", "cfg5", "cfg4"]:
        make(name)
