"""FactorStats (P:l.527-558 Lemma/Theorem symbols d_i, kappa_1,
kappa_2, alpha; P:l.729-733 the compression ratio) reported by lorasp_get_stats
against the C++ oracle's own symbolic replay and ranks.

- per-node edge counts (lorasp_get_node_counts): the partners (distance-2,
  kappa_2 edges) and the uneliminated neighbours at elimination (distance-1,
  kappa_1 edges) equal the oracle's counts node for node (integers, exact);
- per level: kappa1 / kappa2 = the maxima of those counts, d_max = max
  super-node size, compression_ratio = <rank>_l / <size>_l over the compressed
  super-nodes (reading F9), recomputed here from the ORACLE's ranks (super-node
  sizes at level i < l are the two children's ranks; leaf sizes from the
  partition) to 1e-12, and inside [0, 1] (S:l.303 invariant);
- alpha_hat = max over i < l of (d_i / d_l)^(1/(l-i)) (S:l.344)."""
import numpy as np
import pytest

from oracle import cpp_oracle as CO
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


@pytest.mark.parametrize("name,dims,kind,eps", [
    ("2d", (64, 64), "poisson", 1e-3), ("3d", (16, 16, 16), "varcoef", 1e-3), ("lu", (32, 32), "upwind", 1e-3)])
def test_factorstats_match_oracle(L, name, dims, kind, eps):
    p = make_problem("cfg1", dims=dims, kind=kind)
    h = L.analyze_problem(p, eps=eps)
    h.factor(p.values)
    f = CO.factorize(p.n, p.row_ptr, p.col_idx, p.values, p.coords, p.depth, eps)
    st = h.stats()
    lv = {e["level"]: e for e in st["levels"]}
    l = p.depth
    # super-node sizes: leaf = the merged pair of leaf clusters, else the
    # children's retained ranks (Alg. 1 MergeRedNodes, P:l.295-313)
    leaf_sizes = h.sizes(l)
    assert leaf_sizes.sum() == p.n
    k1_all = k2_all = 0
    d = {}
    for i in range(l, 0, -1):
        gp, gn = h.node_counts(i)
        op, on = f.node_counts(i)
        assert np.array_equal(gp, op) and np.array_equal(gn, on), i
        r = f.ranks(i)
        sz = leaf_sizes if i == l else f.ranks(i + 1)[0::2] + f.ranks(i + 1)[1::2]
        assert np.array_equal(h.sizes(i), sz), i
        comp = gp > 0
        e = lv[i]
        assert e["kappa1"] == gn.max() and e["kappa2"] == gp.max()
        assert e["d_max"] == sz.max() and e["compressed"] == comp.sum()
        cr = r[comp].sum() / sz[comp].sum() if comp.any() else 0.0
        assert abs(e["compression_ratio"] - cr) <= 1e-12 and 0.0 <= cr <= 1.0
        assert abs(e["rank_avg"] - (r[comp].mean() if comp.any() else 0.0)) <= 1e-9
        k1_all, k2_all = max(k1_all, gn.max()), max(k2_all, gp.max())
        d[i] = sz.max()
    assert st["kappa1"] == k1_all and st["kappa2"] == k2_all
    ah = max((d[i] / d[l]) ** (1.0 / (l - i)) for i in range(1, l))
    assert abs(st["alpha_hat"] - ah) <= 1e-12 * ah
    h.close()
