"""The paper's variable-coefficient Poisson cases (Eq. VCP, P:l.685-694; SURVEY
8(f) f3): case 1 phi ~ unif(0,1), case 2 phi = 1/unif(0,1) (SPD path, PCG) and
the indefinite case 3 phi ~ unif(-1,1) (general LU path, GMRES(50)), 16^3,
eps = 1e-3, against the oracle: ranks identical up to the 1e-12 threshold
window, x = Ã b within 1e-9 (1e-6 for the indefinite case: no-pivot vs
partial-pivot LU of indefinite pivots), Krylov iterations within +-1, true
residual <= 1e-10.  Readings F3: Dirichlet boundary, arithmetic face means."""
import numpy as np
import pytest

from oracle import lorasp_oracle as O
from synth.problems import _grid_coords, grid_vcp

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1510_07363_b200 import build, lorasp
    build.build()
    return lorasp


@pytest.mark.parametrize("case", [1, 2, 3])
def test_vcp_cases_match_oracle(L, case):
    dims = (16, 16, 16)
    rp, ci, va = grid_vcp(dims, case)
    n, depth, eps = 4096, 6, 1e-3
    xy = _grid_coords(dims)
    sym = case != 3
    h = L.Handle(n, rp, ci, xy, depth=depth, eps=eps, flags=L.LORASP_SPD if sym else 0)
    h.factor(va)
    f = O.factorize(n, rp, ci, va, xy, depth, eps)
    for i in range(1, depth + 1):
        g = h.ranks(i)
        for c in range(2 ** (i - 1)):
            ro = f.rank.get((i, c), 0)
            if g[c] != ro:
                sig = f.sigma[(i, c)]
                assert any(abs(sig[k] / sig[0] - eps) <= 1e-12 for k in (ro - 1, ro) if 0 <= k < sig.size)
    b = np.sin(np.arange(n) * 0.1)
    x = np.zeros(n)
    h.apply(b, x)
    xo = O.solve(f, b)
    # indefinite case 3: the GPU's fused pivots use no-pivot LU, the oracle partial
    # pivoting; on indefinite pivots the element growth differs, so the two agree to
    # ~1e-7 (measured 1.3e-7), not 1e-9
    tol = 1e-9 if sym else 1e-6
    assert np.linalg.norm(x - xo) <= tol * np.linalg.norm(xo)
    xk = np.zeros(n)
    rc, it, rr = h.krylov(b, xk, 1e-10, method=L.LORASP_CG if sym else L.LORASP_GMRES, restart=50)
    mv = lambda v: O.spmv(rp, ci, va, v)
    kry = O.pcg if sym else O.gmres
    ro = kry(mv, lambda v: O.solve(f, v), b, tol=1e-10)
    assert rc == 0 and rr <= 1e-10 and abs(it - ro.iters) <= 1, (it, ro.iters)
    h.close()
