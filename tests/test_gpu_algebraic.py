"""GPU parity with the algebraic partitioner (LORASP_ALGEBRAIC):
nested partitionings from the graph of A alone, on grids with the coordinates
withheld and on an unstructured k-nearest-neighbour graph Laplacian.  Against
the oracle's partition="algebraic" mode: eps = 0 exact (dense solve), ranks
identical up to the 1e-12 threshold window, x = Ã b within 1e-9, Krylov to
1e-10."""
import numpy as np
import pytest

from oracle import lorasp_oracle as O
from synth import csr_to_dense, make_problem
from synth.problems import random_knn_laplacian

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1510_07363_b200 import build, lorasp
    build.build()
    return lorasp


def _cases():
    out = []
    p = make_problem("cfg1", dims=(32, 32), kind="varcoef")
    out.append(("grid2d", p.n, p.row_ptr, p.col_idx, p.values, 6, True))
    p = make_problem("cfg3", dims=(10, 10, 10))
    out.append(("grid3d", p.n, p.row_ptr, p.col_idx, p.values, 5, True))
    rp, ci, va = random_knn_laplacian(2000, seed=11)
    out.append(("knn", 2000, rp, ci, va, 5, True))
    p = make_problem("cfg5", dims=(32, 32))
    out.append(("upwind", p.n, p.row_ptr, p.col_idx, p.values, 5, False))
    return out


@pytest.mark.parametrize("case", range(4))
@pytest.mark.parametrize("eps", [0.0, 1e-2])
def test_algebraic_partition_parity(L, case, eps):
    name, n, rp, ci, va, depth, sym = _cases()[case]
    flags = (L.LORASP_SPD if sym else 0) | L.LORASP_ALGEBRAIC
    h = L.Handle(n, rp, ci, np.zeros((n, 1)), depth=depth, eps=eps, flags=flags)
    h.factor(va)
    b = np.sin(np.arange(n) * 0.37) + 0.1
    x = np.zeros(n)
    h.apply(b, x)
    f = O.factorize(n, rp, ci, va, np.zeros((n, 1)), depth, eps, partition="algebraic")
    if eps == 0.0:
        xe = np.linalg.solve(csr_to_dense(n, rp, ci, va), b)
        assert np.linalg.norm(x - xe) <= 1e-10 * np.linalg.norm(xe)
    else:
        for i in range(1, depth + 1):
            g = h.ranks(i)
            for c in range(2 ** (i - 1)):
                ro = f.rank.get((i, c), 0)
                if g[c] != ro:
                    sig = f.sigma[(i, c)]
                    assert any(abs(sig[k] / sig[0] - eps) <= 1e-12 for k in (ro - 1, ro) if 0 <= k < sig.size)
        xo = O.solve(f, b)
        assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)
        xk = np.zeros(n)
        rc, it, rr = h.krylov(b, xk, 1e-10, method=L.LORASP_CG if sym else L.LORASP_GMRES)
        assert rc == 0 and rr <= 1e-10
    h.close()
