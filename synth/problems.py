"""Synthetic problem generators for the five BASELINE.json configs.

Recipe:
  * interior grid points x = ((i+1)h, (j+1)h[, (k+1)h]), h = 1/(N+1) with N the
    largest grid dimension; dof index q = i + Nx*j (+ Nx*Ny*k), x fastest;
  * Dirichlet-0 boundary: neighbours outside the grid are dropped;
  * stencils are unit-scaled (h^2 folded into the matrix): 2D 5-point diag 4 /
    off -1, 3D 7-point diag 6 / off -1 (Eq. Pois);
  * cfg4 variable coefficient (Eq. VCP, with BASELINE's
    log-uniform law): phi_q = 10^(-3 + 6 u'_q), face coefficient
    a = 2 phi_p phi_q / (phi_p + phi_q) (harmonic mean), boundary face a = phi_p,
    A_pp = sum of the 6 face coefficients, A_pq = -a;
  * cfg5 first-order upwind convection-diffusion -Lap u + beta.grad u,
    beta = (50, 30) (PAPER.md l.803-814 family, BASELINE cfg5):
    A_qq = 4 + h (50 + 30), west -1 - 50 h, south -1 - 30 h, east/north -1;
  * right-hand side b_q = 2 u_q - 1 with u_q the splitmix64 stream (seed 1510)
    at index q, top 53 bits * 2^-53 (uniform[-1, 1)).

Everything is vectorised numpy; CSR is int64 row_ptr / col_idx (sorted per
row) and float64 values.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional, Sequence

import numpy as np

RHS_SEED = 1510
COEF_SEED = 7363

_M64 = (1 << 64) - 1


def splitmix64_uniform(seed: int, n: int, start: int = 0) -> np.ndarray:
    """u_q in [0,1) for q = start..start+n-1 from the splitmix64 stream.

    z = seed + (q+1) * 0x9E3779B97F4A7C15; z = (z ^ z>>30) * 0xBF58476D1CE4E5B9;
    z = (z ^ z>>27) * 0x94D049BB133111EB; z ^= z>>31; u = (z >> 11) * 2^-53.
    """
    q = np.arange(start, start + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & _M64) + (q + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def rhs_uniform(n: int, seed: int = RHS_SEED) -> np.ndarray:
    """b_q = 2 u_q - 1 (uniform[-1, 1)), seeded."""
    return 2.0 * splitmix64_uniform(seed, n) - 1.0


@dataclasses.dataclass
class Problem:
    name: str
    n: int
    dim: int
    row_ptr: np.ndarray      # int64 [n+1]
    col_idx: np.ndarray      # int64 [nnz]
    values: np.ndarray       # float64 [nnz]
    coords: np.ndarray       # float64 [n, dim] row-major
    b: np.ndarray            # float64 [n]
    leaf: int = 64           # target dofs per leaf red cluster
    depth: int = 0           # H-tree depth l
    eps: float = 1e-2
    solver: str = "cg"       # "cg" | "gmres"
    symmetric: bool = True

    @property
    def nnz(self) -> int:
        return int(self.col_idx.shape[0])


def _grid_coords(dims: Sequence[int]) -> np.ndarray:
    h = 1.0 / (max(dims) + 1)
    axes = [(np.arange(d, dtype=np.float64) + 1.0) * h for d in dims]
    mesh = np.meshgrid(*axes, indexing="ij")          # mesh[a][i0, i1, ...]
    # dof index q = i + Nx*j (+ Nx*Ny*k): x fastest -> flatten in Fortran order
    return np.stack([m.reshape(-1, order="F") for m in mesh], axis=1).copy()


def _assemble(n: int, rows: list, cols: list, vals: list):
    r = np.concatenate(rows); c = np.concatenate(cols); v = np.concatenate(vals)
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(row_ptr, r + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    return row_ptr, c.astype(np.int64), v.astype(np.float64)


def _neighbour_pairs(dims: Sequence[int]):
    """Yield (axis, lo_index_array, hi_index_array) for every grid face."""
    dims = list(dims)
    n = int(np.prod(dims))
    idx = np.arange(n, dtype=np.int64).reshape(dims[::-1])  # [..., j, i] (C order, x fastest)
    for a in range(len(dims)):
        ax = len(dims) - 1 - a                              # numpy axis of grid axis a
        lo = np.take(idx, np.arange(dims[a] - 1), axis=ax).reshape(-1)
        hi = np.take(idx, np.arange(1, dims[a]), axis=ax).reshape(-1)
        yield a, lo, hi


def grid_poisson(dims: Sequence[int]):
    """Unit-scaled 5-point (2D) / 7-point (3D) Dirichlet Laplacian: diag 2d, off -1."""
    n = int(np.prod(dims)); d = len(dims)
    rows = [np.arange(n, dtype=np.int64)]; cols = [np.arange(n, dtype=np.int64)]
    vals = [np.full(n, 2.0 * d)]
    for _, lo, hi in _neighbour_pairs(dims):
        rows += [lo, hi]; cols += [hi, lo]; vals += [np.full(lo.size, -1.0)] * 2
    return _assemble(n, rows, cols, vals)


def grid_varcoef(dims: Sequence[int], seed: int = COEF_SEED):
    """7-point (or 5-point) variable-coefficient diffusion, harmonic faces.

    phi_q = 10^(-3 + 6 u'_q); interior face a = 2 phi_p phi_q / (phi_p + phi_q);
    every boundary face of cell p contributes a = phi_p to A_pp (Dirichlet);
    A_pq = -a.  phi == 1 reproduces grid_poisson exactly.
    """
    n = int(np.prod(dims)); d = len(dims)
    phi = 10.0 ** (-3.0 + 6.0 * splitmix64_uniform(seed, n))
    return _varcoef_from_phi(dims, phi)


def _varcoef_from_phi(dims, phi):
    n = int(np.prod(dims)); d = len(dims)
    diag = np.zeros(n)
    rows = []; cols = []; vals = []
    nface = np.zeros(n)
    for _, lo, hi in _neighbour_pairs(dims):
        a = 2.0 * phi[lo] * phi[hi] / (phi[lo] + phi[hi])
        np.add.at(diag, lo, a); np.add.at(diag, hi, a)
        np.add.at(nface, lo, 1.0); np.add.at(nface, hi, 1.0)
        rows += [lo, hi]; cols += [hi, lo]; vals += [-a, -a]
    diag += (2.0 * d - nface) * phi                       # boundary faces: a = phi_p
    rows.append(np.arange(n, dtype=np.int64)); cols.append(np.arange(n, dtype=np.int64))
    vals.append(diag)
    return _assemble(n, rows, cols, vals)


def grid_upwind(dims: Sequence[int], beta: Sequence[float] = (50.0, 30.0)):
    """First-order upwind -Lap u + beta.grad u, unit-scaled (h folded), beta > 0.

    A_qq = 2d + h*sum(beta); upwind (west/south) neighbour -1 - h*beta_a;
    downwind neighbour -1.  Nonsymmetric M-matrix.
    """
    n = int(np.prod(dims)); d = len(dims)
    h = 1.0 / (max(dims) + 1)
    rows = [np.arange(n, dtype=np.int64)]; cols = [np.arange(n, dtype=np.int64)]
    vals = [np.full(n, 2.0 * d + h * float(sum(beta[:d])))]
    for a, lo, hi in _neighbour_pairs(dims):
        # row hi has its west/south (upwind) neighbour lo; row lo has east/north hi
        rows += [hi, lo]; cols += [lo, hi]
        vals += [np.full(lo.size, -1.0 - h * beta[a]), np.full(lo.size, -1.0)]
    return _assemble(n, rows, cols, vals)


def grid_advdiff(dims: Sequence[int], sigma: float = 1.0, R: float = 1.0):
    """The paper's advection-diffusion benchmark (P:l.803-815, Eq. advdiff):
    sigma T + R (1,...,1).grad T - Lap T = g on the unit cube, Dirichlet,
    central differences on the N^d interior grid, h = 1/(N+1), scaled by h^2:
    A_qq = 2d + sigma h^2; the +a / -a neighbours -1 + R h / 2 / -1 - R h / 2
    (symmetric diffusion + skew-symmetric advection, P:l.817)."""
    n = int(np.prod(dims)); d = len(dims)
    h = 1.0 / (max(dims) + 1)
    rows = [np.arange(n, dtype=np.int64)]; cols = [np.arange(n, dtype=np.int64)]
    vals = [np.full(n, 2.0 * d + sigma * h * h)]
    for _, lo, hi in _neighbour_pairs(dims):
        # row lo: its +a neighbour is hi; row hi: its -a neighbour is lo
        rows += [lo, hi]; cols += [hi, lo]
        vals += [np.full(lo.size, -1.0 + 0.5 * R * h), np.full(lo.size, -1.0 - 0.5 * R * h)]
    return _assemble(n, rows, cols, vals)


def grid_vcp(dims: Sequence[int], case: int = 1, seed: int = COEF_SEED):
    """The paper's variable-coefficient Poisson benchmark -div(phi grad T) (Eq. VCP,
    P:l.685-694) with per-point phi: case 1 unif(0,1), case 2 1/unif(0,1), case 3
    unif(-1,1) (indefinite).  Readings (F3): Dirichlet instead of the
    paper's periodic boundary (which leaves a constant null space for cases 1-2),
    face coefficient = arithmetic mean of the two cell values (a harmonic mean is
    undefined across a sign change), boundary faces phi_p."""
    n = int(np.prod(dims)); d = len(dims)
    u = splitmix64_uniform(seed + 100 * case, n)
    phi = {1: u, 2: 1.0 / np.maximum(u, 1e-300), 3: 2.0 * u - 1.0}[case]
    diag = np.zeros(n)
    rows = []; cols = []; vals = []
    nface = np.zeros(n)
    for _, lo, hi in _neighbour_pairs(dims):
        a = 0.5 * (phi[lo] + phi[hi])
        np.add.at(diag, lo, a); np.add.at(diag, hi, a)
        np.add.at(nface, lo, 1.0); np.add.at(nface, hi, 1.0)
        rows += [lo, hi]; cols += [hi, lo]; vals += [-a, -a]
    diag += (2.0 * d - nface) * phi
    rows.append(np.arange(n, dtype=np.int64)); cols.append(np.arange(n, dtype=np.int64))
    vals.append(diag)
    return _assemble(n, rows, cols, vals)


def random_knn_laplacian(n: int, k: int = 6, seed: int = COEF_SEED, shift: float = 0.5):
    """An unstructured SPD test matrix for the algebraic partitioner (f4): points
    from the seeded splitmix64 stream in the unit square, each joined to its k
    nearest neighbours (symmetrised), graph Laplacian with unit weights plus
    shift * I.  The coordinates are NOT passed to the solver."""
    u = splitmix64_uniform(seed, 2 * n).reshape(n, 2)
    d2 = ((u[:, None, :] - u[None, :, :]) ** 2).sum(-1)
    np.fill_diagonal(d2, np.inf)
    nb = np.argsort(d2, axis=1, kind="stable")[:, :k]
    pairs = set()
    for i in range(n):
        for j in nb[i]:
            a, b = (i, int(j)) if i < j else (int(j), i)
            pairs.add((a, b))
    pairs = sorted(pairs)
    lo = np.array([a for a, _ in pairs], dtype=np.int64)
    hi = np.array([b for _, b in pairs], dtype=np.int64)
    deg = np.bincount(lo, minlength=n) + np.bincount(hi, minlength=n)
    rows = [np.arange(n, dtype=np.int64), lo, hi]
    cols = [np.arange(n, dtype=np.int64), hi, lo]
    vals = [deg.astype(np.float64) + shift, -np.ones(lo.size), -np.ones(lo.size)]
    return _assemble(n, rows, cols, vals)


def _depth_for(n: int, leaf: int) -> int:
    return max(1, int(round(math.log2(n / leaf))))


# BASELINE.json configs[0..4] (cfg1..cfg5)
CONFIGS = {
    "cfg1": dict(kind="poisson", dims=(32, 32), leaf=16, depth=6, eps=1e-2, solver="cg"),
    "cfg2": dict(kind="poisson", dims=(256, 256), leaf=64, depth=10, eps=1e-3, solver="cg"),
    "cfg3": dict(kind="poisson", dims=(64, 64, 64), leaf=64, depth=12, eps=1e-2, solver="cg"),
    "cfg4": dict(kind="varcoef", dims=(128, 128, 128), leaf=64, depth=15, eps=1e-2, solver="cg"),
    "cfg5": dict(kind="upwind", dims=(1024, 1024), leaf=64, depth=14, eps=1e-3, solver="gmres"),
    # second LU-path workload: the paper's 3D advection-diffusion,
    # 32^3, sigma = 1, eps = 1e-1 (P:l.821-823); R via make_problem(..., R=...)
    "adv32": dict(kind="advdiff", dims=(32, 32, 32), leaf=64, depth=9, eps=1e-1, solver="gmres"),
}


def make_problem(name: str = "cfg1", dims: Optional[Sequence[int]] = None,
                 kind: Optional[str] = None, leaf: Optional[int] = None,
                 depth: Optional[int] = None, eps: Optional[float] = None,
                 rhs_seed: int = RHS_SEED, sigma: float = 1.0, R: float = 1.0) -> Problem:
    """Build a config by name, optionally overriding grid dims / kind / leaf / depth / eps."""
    base = dict(CONFIGS.get(name, CONFIGS["cfg1"]))
    if dims is not None:
        base["dims"] = tuple(dims)
        base["depth"] = None
    if kind is not None:
        base["kind"] = kind
    if leaf is not None:
        base["leaf"] = leaf
        base["depth"] = None if depth is None else depth
    if depth is not None:
        base["depth"] = depth
    if eps is not None:
        base["eps"] = eps
    dims = tuple(base["dims"]); n = int(np.prod(dims))
    k = base["kind"]
    if k == "poisson":
        rp, ci, va = grid_poisson(dims); sym = True
    elif k == "varcoef":
        rp, ci, va = grid_varcoef(dims); sym = True
    elif k == "upwind":
        rp, ci, va = grid_upwind(dims); sym = False
    elif k == "advdiff":
        rp, ci, va = grid_advdiff(dims, sigma, R); sym = False
    else:
        raise ValueError(f"unknown problem kind {k}")
    dep = base["depth"] if base.get("depth") else _depth_for(n, base["leaf"])
    solver = base.get("solver", "cg" if sym else "gmres")
    return Problem(name=name, n=n, dim=len(dims), row_ptr=rp, col_idx=ci, values=va,
                   coords=_grid_coords(dims), b=rhs_uniform(n, rhs_seed),
                   leaf=base["leaf"], depth=int(dep), eps=float(base["eps"]),
                   solver=solver, symmetric=sym)


def csr_to_dense(n, row_ptr, col_idx, values) -> np.ndarray:
    A = np.zeros((n, n))
    for i in range(n):
        s, e = row_ptr[i], row_ptr[i + 1]
        A[i, col_idx[s:e]] += values[s:e]
    return A


def csr_matvec(row_ptr, col_idx, values, x) -> np.ndarray:
    n = row_ptr.shape[0] - 1
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    return np.bincount(rows, weights=values * x[col_idx], minlength=n)
