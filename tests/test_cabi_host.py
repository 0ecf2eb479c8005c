"""C-ABI library on the CPU box: it loads, exports every symbol include/lorasp.h
declares, and its host-only analyze phase (no device work) agrees with the
oracle's tree / colouring / order.  No compute calls are made here."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT, ring_problem
from oracle import lorasp_oracle as O
from synth import make_problem


@pytest.fixture(scope="module")
def L():
    from paper_1510_07363_b200 import build, lorasp
    build.build()
    return lorasp


def test_exports_every_declared_symbol(L):
    lib = L.load()
    hdr = open(os.path.join(ROOT, "include", "lorasp.h")).read()
    declared = set(re.findall(r"^(?:int|void|const char \*)\s*(lorasp_[a-z_]+)\s*\(", hdr, re.M))
    assert declared == set(L.SYMBOLS)
    for s in declared:
        assert hasattr(lib, s), s


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_analyze_order_matches_oracle(L, name):
    p = make_problem(name)
    h = L.analyze_problem(p)
    t = O.bisection_tree(p.coords, p.depth)
    for i in range(1, p.depth + 1):
        order, wave = h.level_order(i)
        k = i - 1
        cl = t.leaf_of >> (p.depth - k)
        N1, N2 = O.distance_sets(O.quotient_graph(p.row_ptr, p.col_idx, cl, 2 ** k))
        col = O.colour_level(t, k, p.dim, N1, N2)
        assert list(order) == sorted(range(2 ** k), key=lambda c: (col[c], c))
        # waves = colour classes, in order
        assert all(wave[order[a]] <= wave[order[a + 1]] for a in range(2 ** k - 1))
        for a in range(2 ** k):
            for b in range(2 ** k):
                if wave[a] == wave[b]:
                    assert col[a] == col[b]
    st = h.stats()
    assert st["max_edge_distance"] <= 2        # Theorem P:l.515-521 on the symbolic replay
    want = {"cfg1": 22, "cfg2": 42, "cfg3": 70}[name]
    assert st["waves"] == want
    h.close()


def test_analyze_natural_order_one_node_per_wave(L):
    rp, ci, va, xy = ring_problem(64)
    h = L.Handle(64, rp, ci, xy, depth=3, eps=1e-8, flags=L.LORASP_SPD | L.LORASP_ORDER_NATURAL)
    order, wave = h.level_order(3)
    assert list(order) == [0, 1, 2, 3] and list(wave) == [0, 1, 2, 3]
    h.close()


def test_analyze_rejects_bad_input(L):
    n = 4
    rp = np.array([0, 2, 3, 4, 5], dtype=np.int64)
    ci = np.array([0, 1, 1, 2, 3], dtype=np.int64)      # (0,1) without (1,0)
    xy = np.arange(4.0).reshape(-1, 1)
    with pytest.raises(L.LoraspError) as e:
        L.Handle(n, rp, ci, xy, depth=1, eps=0.1)
    assert e.value.code == -2
    p = make_problem("cfg1")
    with pytest.raises(L.LoraspError) as e:
        L.Handle(p.n, p.row_ptr, p.col_idx, p.coords, depth=11, eps=0.1)   # 2^11 > n
    assert e.value.code == -1
    with pytest.raises(L.LoraspError) as e:
        L.Handle(p.n, p.row_ptr, p.col_idx, p.coords, depth=6, eps=1.5)            # eps outside [0, 1]
    assert e.value.code == -1


def test_analyze_general_path_orders_match_spd(L):
    # the LU path (flags without LORASP_SPD) replays the same symbolic structure
    p = make_problem("cfg5", dims=(64, 64), depth=7)
    h1 = L.Handle(p.n, p.row_ptr, p.col_idx, p.coords, depth=7, eps=1e-3, flags=0)
    h2 = L.Handle(p.n, p.row_ptr, p.col_idx, p.coords, depth=7, eps=1e-3, flags=L.LORASP_SPD)
    for i in range(1, 8):
        assert np.array_equal(h1.level_order(i)[0], h2.level_order(i)[0])
    assert h1.stats()["waves"] == h2.stats()["waves"]
    h1.close(); h2.close()


def test_apply_before_factor_is_state_error(L):
    p = make_problem("cfg1")
    h = L.analyze_problem(p)
    with pytest.raises(L.LoraspError) as e:
        h.apply(p.b, np.zeros(p.n))
    assert e.value.code == -8
    h.close()


def _alg_problems():
    from synth.problems import random_knn_laplacian
    out = []
    for name, dims in (("cfg1", (32, 32)), ("cfg3", (8, 8, 8))):
        p = make_problem(name, dims=dims)
        out.append((p.n, p.row_ptr, p.col_idx, p.depth))
    rp, ci, _ = random_knn_laplacian(1500)
    out.append((1500, rp, ci, 5))
    return out


@pytest.mark.parametrize("case", range(3))
def test_analyze_order_matches_oracle_algebraic(L, case):
    """LORASP_ALGEBRAIC (f4): the C++ BFS bisection + colouring equal the oracle's."""
    n, rp, ci, depth = _alg_problems()[case]
    h = L.Handle(n, rp, ci, np.zeros((n, 1)), depth=depth, eps=1e-2,
                 flags=L.LORASP_SPD | L.LORASP_ALGEBRAIC)
    t = O.bisection_tree_algebraic(rp, ci, depth)
    for i in range(1, depth + 1):
        order, wave = h.level_order(i)
        k = i - 1
        cl = t.leaf_of >> (depth - k)
        N1, N2 = O.distance_sets(O.quotient_graph(rp, ci, cl, 2 ** k))
        col = O.colour_level(t, k, 1, N1, N2)
        assert list(order) == sorted(range(2 ** k), key=lambda c: (col[c], c))
    st = h.stats()
    assert st["max_edge_distance"] <= 2
    h.close()
