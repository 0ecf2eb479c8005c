"""Structure pins: bisection tree, quotient graphs, distance-2 colouring, and
the synthetic generators (closed forms / brute force, no GPU)."""
import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import shortest_path

from oracle import lorasp_oracle as O
from synth import csr_to_dense, make_problem, splitmix64_uniform
from synth.problems import _varcoef_from_phi, grid_poisson


def test_splitmix64_reference_values():
    # splitmix64 with state seed + (q+1)*golden: q=0, seed=0 -> z = 0x9E3779B97F4A7C15
    # mixed: 0xE220A8397B1DCDAF (the well-known first output of splitmix64(0))
    u = splitmix64_uniform(0, 1)[0]
    assert u == (0xE220A8397B1DCDAF >> 11) * 2.0 ** -53


def test_generators_closed_forms():
    p = make_problem("cfg1", dims=(5, 4))
    A = csr_to_dense(p.n, p.row_ptr, p.col_idx, p.values)
    q = 1 + 5 * 1                      # interior point (1,1): row (-1,-1,4,-1,-1)
    assert A[q, q] == 4 and A[q, q - 1] == -1 and A[q, q + 1] == -1
    assert A[q, q - 5] == -1 and A[q, q + 5] == -1 and np.count_nonzero(A[q]) == 5
    assert np.array_equal(A, A.T)
    # varcoef with phi == 1 reproduces the Poisson matrix exactly (reading Z19)
    dims = (4, 3, 5)
    rp, ci, va = _varcoef_from_phi(dims, np.ones(60))
    rp2, ci2, va2 = grid_poisson(dims)
    assert np.array_equal(rp, rp2) and np.array_equal(ci, ci2) and np.allclose(va, va2, rtol=0, atol=0)
    # upwind: nonsymmetric, west/south carry -1 - h*beta
    u = make_problem("cfg5", dims=(8, 8))
    U = csr_to_dense(u.n, u.row_ptr, u.col_idx, u.values)
    h = 1.0 / 9
    q = 3 + 8 * 3
    assert U[q, q] == pytest.approx(4 + 80 * h)
    assert U[q, q - 1] == pytest.approx(-1 - 50 * h) and U[q, q - 8] == pytest.approx(-1 - 30 * h)
    assert U[q, q + 1] == -1 and U[q, q + 8] == -1
    # nnz of the BASELINE configs
    assert make_problem("cfg2").nnz == 326656


@pytest.mark.parametrize("dims,depth", [((32, 32), 6), ((256, 256), 10), ((64, 64, 64), 12), ((24, 16), 4)])
def test_bisection_tree_boxes(dims, depth):
    p = make_problem("cfg1", dims=dims, depth=depth)
    t = O.bisection_tree(p.coords, depth)
    n = p.n
    for k in range(depth + 1):
        cl = t.clusters[k]
        assert len(cl) == 2 ** k
        assert np.array_equal(np.sort(np.concatenate(cl)), np.arange(n))
        if k < depth:
            for c in range(2 ** k):   # nestedness (Def. nested partitionings l.214-216)
                u = np.union1d(t.clusters[k + 1][2 * c], t.clusters[k + 1][2 * c + 1])
                assert np.array_equal(u, cl[c])
    # leaves of a power-of-two grid are exact boxes of equal size
    sizes = {len(c) for c in t.clusters[depth]}
    assert sizes == {n // 2 ** depth}
    ijk = np.round(p.coords * (max(dims) + 1)).astype(int) - 1
    for mem in t.clusters[depth][:16]:
        box = ijk[mem]
        ext = box.max(0) - box.min(0) + 1
        assert np.prod(ext) == len(mem)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_lattice_colouring_is_distance2(name):
    p = make_problem(name)
    t = O.bisection_tree(p.coords, p.depth)
    rows = np.repeat(np.arange(p.n), np.diff(p.row_ptr))
    for k in range(1, p.depth):
        cl = t.leaf_of >> (p.depth - k)
        adj = O.quotient_graph(p.row_ptr, p.col_idx, cl, 2 ** k)
        N1, N2 = O.distance_sets(adj)
        col = O.colour_level(t, k, p.dim, N1, N2)
        # brute force with scipy BFS: same colour => distance >= 3
        G = sp.coo_matrix((np.ones(rows.size), (cl[rows], cl[p.col_idx])), shape=(2 ** k, 2 ** k))
        D = shortest_path(G.tocsr(), unweighted=True, directed=False)
        col = np.array(col)
        same = col[:, None] == col[None, :]
        np.fill_diagonal(same, False)
        assert np.all(D[same] >= 3)
        # the lattice rule was accepted (<= 2d+1 colours) and is balanced
        assert col.max() < 2 * p.dim + 1
        if 2 ** k >= 64:
            cnt = np.bincount(col)
            assert cnt.max() - cnt.min() <= max(2, 2 ** k // 20)


def test_greedy_fallback_on_ring():
    # 1D ring of 4 clusters: lattice colours g mod 3 = 0,1,2,0 put the adjacent
    # clusters 0 and 3 together -> the greedy distance-2 fallback must be used
    from conftest import ring_problem
    rp, ci, va, xy = ring_problem(64)
    t = O.bisection_tree(xy, 3)
    cl = t.leaf_of >> 1
    adj = O.quotient_graph(rp, ci, cl, 4)
    N1, N2 = O.distance_sets(adj)
    col = O.colour_level(t, 2, 1, N1, N2)
    assert len(set(col)) == 4          # every pair of the 4-ring is within distance 2


def test_waves_conflict_free_footprints():
    """Distance-2 colouring => the closed neighbourhoods B1(c) of same-coloured
    clusters are disjoint, so the blocks one wave reads/writes are disjoint
    (SURVEY §8.0 item 1).  Brute force on the cfg2 leaf level."""
    p = make_problem("cfg2")
    t = O.bisection_tree(p.coords, p.depth)
    k = p.depth - 1
    cl = t.leaf_of >> 1
    adj = O.quotient_graph(p.row_ptr, p.col_idx, cl, 2 ** k)
    N1, N2 = O.distance_sets(adj)
    col = O.colour_level(t, k, p.dim, N1, N2)
    for colour in set(col):
        seen = set()
        for c in range(2 ** k):
            if col[c] != colour:
                continue
            ball = {c} | N1[c]
            assert not (ball & seen)
            seen |= ball


def test_synth_advdiff_structure():
    """Eq. advdiff discretisation (P:l.811-817): symmetric part = the 7-point
    Laplacian + sigma h^2 I, skew part = R h/2 on each +axis neighbour."""
    from synth import csr_to_dense, make_problem
    from synth.problems import grid_poisson
    dims = (5, 4, 3)
    for sigma, R in ((0.0, 1.0), (1.0, 300.0)):
        p = make_problem("adv32", dims=dims, sigma=sigma, R=R)
        A = csr_to_dense(p.n, p.row_ptr, p.col_idx, p.values)
        h = 1.0 / (max(dims) + 1)
        Lp = csr_to_dense(p.n, *grid_poisson(dims))
        assert np.allclose((A + A.T) / 2, Lp + sigma * h * h * np.eye(p.n), rtol=0, atol=1e-14)
        K = (A - A.T) / 2
        # +x neighbour of dof 0 is dof 1 (x fastest): K[0, 1] = R h / 2
        assert K[0, 1] == pytest.approx(0.5 * R * h) and K[1, 0] == pytest.approx(-0.5 * R * h)
        assert K[0, dims[0]] == pytest.approx(0.5 * R * h)           # +y
        assert K[0, dims[0] * dims[1]] == pytest.approx(0.5 * R * h)  # +z
        assert np.count_nonzero(np.abs(K) > 1e-15) == 2 * sum(
            (dims[a] - 1) * int(np.prod(dims)) // dims[a] for a in range(3))


def test_algebraic_bisection_pins():
    """Reading F4 on graphs whose BFS level structure is known: a path splits into
    its two contiguous halves; on a grid every child of a connected cluster is
    connected (a BFS prefix is) and the sizes are floor / ceil halves."""
    n = 37
    rows = np.arange(n - 1)
    A = sp.coo_matrix((np.ones(2 * (n - 1)), (np.r_[rows, rows + 1], np.r_[rows + 1, rows])), shape=(n, n))
    A = (A + sp.eye(n)).tocsr()
    A.sort_indices()
    t = O.bisection_tree_algebraic(A.indptr, A.indices, 2)
    # BFS from vertex 0 reaches n-1 last; BFS from n-1 orders n-1, n-2, ..., 0
    assert list(t.clusters[1][0]) == list(range(19, 37)) and list(t.clusters[1][1]) == list(range(0, 19))
    p = make_problem("cfg1", dims=(12, 10))
    t = O.bisection_tree_algebraic(p.row_ptr, p.col_idx, 4)
    G = sp.csr_matrix((np.ones(p.col_idx.size), p.col_idx, p.row_ptr))
    for k in range(1, 5):
        for c, mem in enumerate(t.clusters[k]):
            par = t.clusters[k - 1][c // 2]
            assert mem.size in (par.size // 2, par.size - par.size // 2)
            sub = G[mem][:, mem]
            ncomp, _ = sp.csgraph.connected_components(sub, directed=False)
            parent_conn = sp.csgraph.connected_components(G[par][:, par], directed=False)[0] == 1
            if parent_conn and c % 2 == 0:
                assert ncomp == 1
    assert sorted(np.concatenate(t.clusters[4]).tolist()) == list(range(p.n))
