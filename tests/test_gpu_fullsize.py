"""GPU checks at BASELINE.json's full sizes (cfg3 64^3, cfg4 128^3, cfg5 1024^2;
cfg4 / cfg5 also with the RRQR compressor),
in the launch configuration bench.py times (device buffers, re-factorization
through the rank-predicted sweep and the recorded graph).  The oracle cannot
factor these sizes, so the checks are properties that hold at any size
(cfg2 is compared with the oracle element by element in test_gpu_parity.py):
  * the Krylov solution's true residual, recomputed on the host from the CSR
    matrix (scipy), is <= 1e-10 (Eq. accres, P:l.585-589);
  * the structural invariant of Alg. 1: level-i super-node sizes are the sums
    of the two level-(i+1) ranks (P:l.377), and 0 <= r <= m;
  * Ã is a contraction of the error: ||b - A Ã b|| / ||b|| < 1 (what makes it a
    preconditioner), and for the SPD configs Ã is symmetric:
    |y^T Ã x - x^T Ã y| <= 1e-10 |x| |Ã y| (PCG needs a symmetric preconditioner);
  * re-factorizations are bitwise identical (rank-predicted sweep, graph)."""
import numpy as np
import pytest
import scipy.sparse as sp

from synth import make_problem

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1510_07363_b200 import build, lorasp
    build.build()
    return lorasp


def _csr(p):
    return sp.csr_matrix((p.values, p.col_idx, p.row_ptr), shape=(p.n, p.n))


def _apply(h, v):
    b = torch.tensor(v, device="cuda")
    x = torch.empty_like(b)
    h.apply(b, x)
    return x.cpu().numpy()


@pytest.mark.parametrize("name,rrqr", [("cfg3", False), ("cfg4", False), ("cfg5", False), ("cfg4", True),
                                       ("cfg5", True)])
def test_full_size_properties(L, name, rrqr):
    p = make_problem(name)
    A = _csr(p)
    flags = (L.LORASP_SPD if p.symmetric else 0) | (L.LORASP_RRQR if rrqr else 0)
    h = L.analyze_problem(p, flags=flags)
    vals = torch.tensor(p.values, device="cuda")
    h.factor(vals)
    # structure of the level sweep
    for i in range(1, h.depth):
        m_i, r_i = h.sizes(i), h.ranks(i)
        r_next = h.ranks(i + 1)
        assert np.all(r_i >= 0) and np.all(r_i <= m_i)
        assert np.array_equal(m_i, r_next[0::2] + r_next[1::2])
    x0 = _apply(h, p.b)
    # re-factorizations (rank-predicted sweep, then the recorded graph): bitwise
    for _ in range(3):
        h.factor(vals)
        assert np.array_equal(_apply(h, p.b), x0)
    assert h.stats()["factor_graph"]
    # Ã is a contraction of the error
    assert np.linalg.norm(p.b - A @ x0) < np.linalg.norm(p.b)
    if p.symmetric:
        rng = np.random.default_rng(3)
        u, v = rng.standard_normal(p.n), rng.standard_normal(p.n)
        au, av = _apply(h, u), _apply(h, v)
        assert abs(v @ au - u @ av) <= 1e-10 * np.linalg.norm(u) * np.linalg.norm(av)
    # Krylov to 1e-10, true residual recomputed on the host
    xk = torch.zeros(p.n, dtype=torch.float64, device="cuda")
    b = torch.tensor(p.b, device="cuda")
    rc, it, rr = h.krylov(b, xk, 1e-10, method=L.LORASP_CG if p.symmetric else L.LORASP_GMRES, restart=50)
    x = xk.cpu().numpy()
    rel = np.linalg.norm(p.b - A @ x) / np.linalg.norm(p.b)
    assert rc == 0 and rr <= 1e-10 and rel <= 1e-10 * 1.01
    h.close()
