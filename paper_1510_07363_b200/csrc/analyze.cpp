// lorasp_analyze: host-side symbolic phase.
//
//  * nested partitionings by recursive coordinate bisection (P:l.214-216;
//    reading Z17 in DESIGN.md),
//  * quotient (adjacency) graphs of A at every level (P:l.73-76, l.247-249),
//    distance-1/2 sets (Def. distance, P:l.506-512),
//  * a distance-2 colouring per level (the order within a level is free,
//    P:l.843): lattice rule (sum_a (a+1) g_a) mod (2d+1), validated, greedy
//    fallback (readings Z1/Z2),
//  * a symbolic replay of Alg. 1 (P:l.265-289) in that order: partners of
//    each super-node (well-separated neighbours, P:l.322), the five edge rules
//    of Compress (P:l.383-389), the fill of the fused s/b elimination
//    (P:l.101-106, P:l.396-399), every block ("slot") that ever exists, and a
//    check of the sparsity theorem (P:l.515-521) and of wave disjointness.
//
// Nothing here touches the device.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <unordered_map>

#include "internal.h"
#include "lorasp.h"

namespace lorasp {
namespace {

struct Graph {
  std::vector<std::vector<int>> n1, n2;  // sorted
  int dist(int a, int b) const {
    if (a == b) return 0;
    if (std::binary_search(n1[a].begin(), n1[a].end(), b)) return 1;
    if (std::binary_search(n2[a].begin(), n2[a].end(), b)) return 2;
    return 3;
  }
};

void make_n2(Graph &g) {
  const int K = (int)g.n1.size();
  g.n2.assign(K, {});
  std::vector<int> mark(K, -1);
  for (int c = 0; c < K; ++c) {
    mark[c] = c;
    for (int q : g.n1[c]) mark[q] = c;
    std::vector<int> two;
    for (int q : g.n1[c])
      for (int w : g.n1[q])
        if (mark[w] != c) {
          mark[w] = c;
          two.push_back(w);
        }
    std::sort(two.begin(), two.end());
    g.n2[c] = std::move(two);
  }
}

inline uint64_t key(int u, int v) {
  if (u > v) std::swap(u, v);
  return ((uint64_t)(uint32_t)u << 32) | (uint32_t)v;
}
inline uint64_t dkey(int u, int v) {  // ordered pair u -> v
  return ((uint64_t)(uint32_t)u << 32) | (uint32_t)v;
}

void sorted_insert(std::vector<int> &v, int x) {
  auto it = std::lower_bound(v.begin(), v.end(), x);
  if (it == v.end() || *it != x) v.insert(it, x);
}
void sorted_erase(std::vector<int> &v, int x) {
  auto it = std::lower_bound(v.begin(), v.end(), x);
  if (it != v.end() && *it == x) v.erase(it);
}

}  // namespace

int build_plan(Plan &pl, int64_t n, const int64_t *row_ptr, const int64_t *col_idx, int dim,
               const double *coords, int leaf_size, int depth, double eps, unsigned flags,
               std::string &err) {
  const bool algebraic = (flags & LORASP_ALGEBRAIC) != 0;
  if (algebraic) dim = 1;   // coordinates unused; one pseudo-axis for the colouring
  if (n <= 0 || !row_ptr || !col_idx || (!coords && !algebraic) || dim < 1 || dim > 3 || eps < 0 || eps > 1) {
    err = "analyze: bad argument";
    return -1;
  }
  if (depth <= 0) {
    if (leaf_size <= 0) {
      err = "analyze: need depth > 0 or leaf_size > 0";
      return -1;
    }
    depth = std::max(1, (int)std::lround(std::log2((double)n / leaf_size)));
  }
  if (depth > 24 || ((int64_t)1 << depth) > n) {
    err = "analyze: depth too large for n";
    return -1;
  }
  pl.n = n;
  pl.dim = dim;
  pl.depth = depth;
  pl.eps = eps;
  pl.flags = flags;
  pl.nnz = row_ptr[n];
  pl.row_ptr.assign(row_ptr, row_ptr + n + 1);
  pl.col_idx.assign(col_idx, col_idx + pl.nnz);
  if (row_ptr[0] != 0) {
    err = "analyze: row_ptr[0] != 0";
    return -2;
  }
  for (int64_t i = 0; i < n; ++i) {
    if (row_ptr[i + 1] < row_ptr[i]) {
      err = "analyze: row_ptr not monotone";
      return -2;
    }
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      int64_t j = col_idx[k];
      if (j < 0 || j >= n || (k > row_ptr[i] && col_idx[k - 1] >= j)) {
        err = "analyze: column indices out of range or unsorted";
        return -2;
      }
      // structural symmetry: (j, i) must be present
      if (!std::binary_search(col_idx + row_ptr[j], col_idx + row_ptr[j + 1], i)) {
        err = "analyze: pattern is not structurally symmetric";
        return -2;
      }
    }
  }

  // ---- nested partitionings by coordinate bisection -----------------------
  std::vector<std::vector<int>> cur(1);
  cur[0].resize(n);
  std::iota(cur[0].begin(), cur[0].end(), 0);
  std::vector<std::vector<int>> axis(depth);
  // algebraic partitioning (reading F4): breadth-first level
  // structure of the cluster's induced subgraph from a pseudo-peripheral vertex
  std::vector<int> owner(algebraic ? n : 0, -1), lev(algebraic ? n : 0, -1);
  auto bfs = [&](int src, int cl, std::vector<int> &touched) {
    touched.clear();
    lev[src] = 0;
    touched.push_back(src);
    for (size_t h = 0; h < touched.size(); ++h) {
      const int v = touched[h];
      for (int64_t q = row_ptr[v]; q < row_ptr[v + 1]; ++q) {
        const int j = (int)col_idx[q];
        if (j != v && owner[j] == cl && lev[j] < 0) {
          lev[j] = lev[v] + 1;
          touched.push_back(j);
        }
      }
    }
  };
  for (int k = 0; k < depth; ++k) {
    std::vector<std::vector<int>> nxt(2 * cur.size());
    axis[k].assign(cur.size(), 0);
    if (algebraic)
      for (size_t c = 0; c < cur.size(); ++c)
        for (int v : cur[c]) owner[v] = (int)c;
    for (size_t c = 0; c < cur.size(); ++c) {
      std::vector<int> &mem = cur[c];
      if (mem.empty()) continue;
      if (algebraic) {
        std::vector<int> touched;
        bfs(mem[0], (int)c, touched);   // mem is ascending: mem[0] is the smallest member
        int far = 0, p = touched[0];
        for (int v : touched) far = std::max(far, lev[v]);
        p = n;
        for (int v : touched)
          if (lev[v] == far) p = std::min(p, v);
        for (int v : touched) lev[v] = -1;
        bfs(p, (int)c, touched);
        const int INF = 1 << 30;
        std::vector<std::pair<int, int>> key(mem.size());
        for (size_t t = 0; t < mem.size(); ++t) key[t] = {lev[mem[t]] < 0 ? INF : lev[mem[t]], mem[t]};
        for (int v : touched) lev[v] = -1;
        std::sort(key.begin(), key.end());
        const size_t h = mem.size() / 2;
        std::vector<int> lo, hi;
        for (size_t t = 0; t < key.size(); ++t) (t < h ? lo : hi).push_back(key[t].second);
        std::sort(lo.begin(), lo.end());
        std::sort(hi.begin(), hi.end());
        nxt[2 * c] = std::move(lo);
        nxt[2 * c + 1] = std::move(hi);
        continue;
      }
      double ext[3], mx = 0;
      for (int a = 0; a < dim; ++a) {
        double lo = coords[(int64_t)mem[0] * dim + a], hi = lo;
        for (int q : mem) {
          double x = coords[(int64_t)q * dim + a];
          lo = std::min(lo, x);
          hi = std::max(hi, x);
        }
        ext[a] = hi - lo;
        mx = std::max(mx, ext[a]);
      }
      int a = 0;
      for (int t = 0; t < dim; ++t)
        if (ext[t] >= mx * (1.0 - 1e-9)) {  // ties within 1e-9 -> lowest axis
          a = t;
          break;
        }
      axis[k][c] = a;
      size_t h = mem.size() / 2;
      std::vector<int> tmp = mem;
      auto cmp = [&](int p, int q) {
        double xp = coords[(int64_t)p * dim + a], xq = coords[(int64_t)q * dim + a];
        return xp < xq || (xp == xq && p < q);
      };
      std::nth_element(tmp.begin(), tmp.begin() + h, tmp.end(), cmp);
      std::vector<int> lo(tmp.begin(), tmp.begin() + h), hi(tmp.begin() + h, tmp.end());
      std::sort(lo.begin(), lo.end());
      std::sort(hi.begin(), hi.end());
      nxt[2 * c] = std::move(lo);
      nxt[2 * c + 1] = std::move(hi);
    }
    cur.swap(nxt);
  }
  const int L = depth;
  const int nleaf = 1 << L;
  const bool sym = (flags & LORASP_SPD) != 0;
  pl.leaf_members = cur;
  pl.leaf_of.assign(n, 0);
  pl.leaf_pos.assign(n, 0);
  pl.leaf_size.assign(nleaf, 0);
  for (int c = 0; c < nleaf; ++c) {
    pl.leaf_size[c] = (int)cur[c].size();
    for (size_t t = 0; t < cur[c].size(); ++t) {
      pl.leaf_of[cur[c][t]] = c;
      pl.leaf_pos[cur[c][t]] = (int)t;
    }
  }

  // ---- quotient graphs G_k, k = 0..L ----------------------------------------
  std::vector<Graph> G(L + 1);
  {
    std::vector<std::vector<int>> adj(nleaf);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
        int a = pl.leaf_of[i], b = pl.leaf_of[col_idx[k]];
        if (a != b) adj[a].push_back(b);
      }
    for (auto &v : adj) {
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
    }
    G[L].n1 = std::move(adj);
    for (int k = L - 1; k >= 0; --k) {
      std::vector<std::vector<int>> up(1 << k);
      for (int a = 0; a < (1 << (k + 1)); ++a)
        for (int b : G[k + 1].n1[a])
          if ((a >> 1) != (b >> 1)) up[a >> 1].push_back(b >> 1);
      for (auto &v : up) {
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
      }
      G[k].n1 = std::move(up);
    }
    for (int k = 0; k <= L; ++k) make_n2(G[k]);
  }

  // ---- per level: colouring, order, symbolic replay --------------------------
  pl.lev.assign(L + 1, SymLevel());
  std::vector<char> prev_p_exists;
  std::vector<SymSlot> prev_slots;
  std::vector<int> prev_pos;  // not needed across levels
  int total_waves = 0;
  for (int i = L; i >= 1; --i) {
    SymLevel &lv = pl.lev[i];
    const int K = 1 << (i - 1);
    const int k = i - 1;  // super-nodes are the clusters of P_{i-1}
    const Graph &g = G[k];
    lv.i = i;
    lv.K = K;
    // colouring (lattice rule, validated; greedy fallback)
    lv.colour.assign(K, 0);
    for (int c = 0; c < K; ++c) {
      int gi[3] = {0, 0, 0};
      for (int t = 0; t < k; ++t) {
        int anc = c >> (k - t), bit = (c >> (k - 1 - t)) & 1;
        int a = axis[t][anc];
        gi[a] = 2 * gi[a] + bit;
      }
      int s = 0;
      for (int a = 0; a < dim; ++a) s += (a + 1) * gi[a];
      lv.colour[c] = s % (2 * dim + 1);
    }
    bool ok = true;
    for (int c = 0; c < K && ok; ++c) {
      for (int q : g.n1[c]) ok = ok && lv.colour[q] != lv.colour[c];
      for (int q : g.n2[c]) ok = ok && lv.colour[q] != lv.colour[c];
    }
    lv.lattice = ok;
    if (!ok) {
      for (int c = 0; c < K; ++c) {
        std::vector<int> used;
        for (int q : g.n1[c])
          if (q < c) used.push_back(lv.colour[q]);
        for (int q : g.n2[c])
          if (q < c) used.push_back(lv.colour[q]);
        int x = 0;
        while (std::find(used.begin(), used.end(), x) != used.end()) ++x;
        lv.colour[c] = x;
      }
    }
    lv.order.resize(K);
    std::iota(lv.order.begin(), lv.order.end(), 0);
    const bool natural = (flags & LORASP_ORDER_NATURAL) != 0;
    if (!natural)
      std::stable_sort(lv.order.begin(), lv.order.end(),
                       [&](int a, int b) { return lv.colour[a] < lv.colour[b]; });
    lv.wave_begin.clear();
    for (int t = 0; t < K; ++t)
      if (natural || t == 0 || lv.colour[lv.order[t]] != lv.colour[lv.order[t - 1]])
        lv.wave_begin.push_back(t);
    lv.wave_begin.push_back(K);
    total_waves += (int)lv.wave_begin.size() - 1;
    std::vector<int> pos(K);
    for (int t = 0; t < K; ++t) pos[lv.order[t]] = t;

    // symbolic state
    std::vector<std::vector<int>> adj(2 * K);
    std::unordered_map<uint64_t, int> slot_of;
    auto row_node = [&](int u, int v) {
      if (u == v) return u;
      bool su = u < K, sv = v < K;
      if (su && sv) return pos[u] < pos[v] ? u : v;
      if (su) return u;
      if (sv) return v;
      return std::min(u, v);
    };
    // SPD: slot of the unordered pair {u, v}; LU: slot of Mat(u -> v) (rows v)
    auto get_slot = [&](int u, int v) {
      const uint64_t kk = sym ? key(u, v) : dkey(u, v);
      auto it = slot_of.find(kk);
      if (it != slot_of.end()) return it->second;
      int id = (int)lv.slots.size();
      if (sym) {
        int r = row_node(u, v);
        lv.slots.push_back({r, r == u ? v : u});
      } else {
        lv.slots.push_back({v, u});
      }
      slot_of.emplace(kk, id);
      return id;
    };
    auto cl = [&](int u) { return u < K ? u : u - K; };
    auto add_edge = [&](int u, int v) {
      if (u == v) return;
      sorted_insert(adj[u], v);
      sorted_insert(adj[v], u);
      int d = g.dist(cl(u), cl(v));
      pl.max_edge_distance = std::max(pl.max_edge_distance, d);
    };
    auto del_edge = [&](int u, int v) {
      sorted_erase(adj[u], v);
      sorted_erase(adj[v], u);
    };

    // MergeRedNodes: initial super-node graph
    std::vector<char> s_exists(K, 0);
    if (i == L) {
      for (int c = 0; c < K; ++c)
        s_exists[c] = (pl.leaf_size[2 * c] + pl.leaf_size[2 * c + 1]) > 0;
      for (int c = 0; c < K; ++c) {
        if (!s_exists[c]) continue;
        get_slot(c, c);
        for (int q : g.n1[c])
          if (s_exists[q]) {
            get_slot(c, q);
            if (!sym) get_slot(q, c);
            add_edge(c, q);
          }
      }
    } else {
      const int Kp = 2 * K;  // previous level's cluster count
      for (int c = 0; c < K; ++c) s_exists[c] = prev_p_exists[2 * c] || prev_p_exists[2 * c + 1];
      for (int c = 0; c < K; ++c)
        if (s_exists[c]) get_slot(c, c);
      for (size_t sid = 0; sid < prev_slots.size(); ++sid) {
        const SymSlot &ps = prev_slots[sid];
        if (ps.row < Kp || ps.col < Kp) continue;  // only P-P slots survive
        int xr = ps.row - Kp, xc = ps.col - Kp;
        int a = xr >> 1, b = xc >> 1;
        if (!sym) {   // Mat(P_xc -> P_xr) lands in Mat(S_b -> S_a) (rows S_a)
          int dst = get_slot(b, a);
          if (a != b) add_edge(a, b);
          lv.merge.push_back({dst, (int)sid, xr & 1, xc & 1, xr, xc, false});
          continue;
        }
        int dst = get_slot(a, b);
        if (a != b) add_edge(a, b);
        if (a == b) {
          lv.merge.push_back({dst, (int)sid, xr & 1, xc & 1, xr, xc, false});
          if (xr != xc) lv.merge.push_back({dst, (int)sid, xc & 1, xr & 1, xc, xr, true});
        } else if (lv.slots[dst].row == a) {
          lv.merge.push_back({dst, (int)sid, xr & 1, xc & 1, xr, xc, false});
        } else {
          lv.merge.push_back({dst, (int)sid, xc & 1, xr & 1, xc, xr, true});
        }
      }
    }

    // replay Alg. 1 at level i in processing order
    lv.node.assign(K, SymNode());
    lv.p_exists.assign(K, 0);
    std::vector<char> elim(K, 0);
    for (size_t w = 0; w + 1 < lv.wave_begin.size(); ++w) {
      for (int t = lv.wave_begin[w]; t < lv.wave_begin[w + 1]; ++t) {
        const int c = lv.order[t];
        SymNode &nd = lv.node[c];
        nd.wave = (int)w;
        if (!s_exists[c]) {
          elim[c] = 1;
          continue;
        }
        nd.exists = true;
        const int s = c;
        nd.self_slot = get_slot(s, s);
        // Compress: partners = uneliminated neighbours at distance >= 2 (P:l.322)
        for (int u : adj[s]) {
          if (u < K && elim[u]) continue;
          if (g.dist(c, cl(u)) >= 2) nd.partners.push_back(u);
        }
        if (!nd.partners.empty()) {
          nd.aux = true;
          lv.p_exists[c] = 1;
          const int P = K + c;
          for (int u : nd.partners) {
            if (sym) {
              nd.pslot_src.push_back(get_slot(s, u));
              nd.pslot_dst.push_back(get_slot(P, u));
            } else {
              nd.pslot_src.push_back(get_slot(u, s));    // Mat(p -> s) = B_k^T
              nd.pslot_src2.push_back(get_slot(s, u));   // Mat(s -> p) = A_k
              nd.pslot_dst.push_back(get_slot(P, u));    // Mat(P -> p) = R_k
              nd.pslot_dst2.push_back(get_slot(u, P));   // Mat(p -> P) = Q_k^T
            }
            del_edge(s, u);                 // rule 1
            add_edge(P, u);                 // rules 2/3
          }
        }
        // Eliminate s then b: fill among T = N1(s) + [P(b)]
        for (int u : adj[s]) {
          if (u < K && elim[u]) continue;
          nd.n1.push_back(u);
          if (sym) {
            nd.n1_slot.push_back(get_slot(s, u));
          } else {
            nd.n1_slot.push_back(get_slot(u, s));    // Mat(n -> s): coupling C
            nd.n1_slot2.push_back(get_slot(s, u));   // Mat(s -> n): coupling R
          }
        }
        std::vector<int> T = nd.n1;
        if (nd.aux) T.push_back(K + c);
        if (sym) {
          for (size_t a = 0; a < T.size(); ++a)
            for (size_t b = 0; b <= a; ++b) {
              nd.tslot.push_back(get_slot(T[a], T[b]));
              add_edge(T[a], T[b]);
            }
        } else {
          for (size_t a = 0; a < T.size(); ++a)
            for (size_t b = 0; b < T.size(); ++b) {
              nd.tslot.push_back(get_slot(T[b], T[a]));   // Mat(T_b -> T_a)
              add_edge(T[a], T[b]);
            }
        }
        for (int u : std::vector<int>(adj[s])) del_edge(s, u);  // s eliminated
        elim[c] = 1;
      }
      // wave disjointness: no slot touched by two nodes of the wave
      std::unordered_map<int, int> owner;
      for (int t = lv.wave_begin[w]; t < lv.wave_begin[w + 1]; ++t) {
        const int c = lv.order[t];
        const SymNode &nd = lv.node[c];
        if (!nd.exists) continue;
        auto touch = [&](int sl) {
          auto it = owner.find(sl);
          if (it != owner.end() && it->second != c) return false;
          owner[sl] = c;
          return true;
        };
        bool good = touch(nd.self_slot);
        for (int sl : nd.n1_slot) good = good && touch(sl);
        for (int sl : nd.pslot_src) good = good && touch(sl);
        for (int sl : nd.pslot_dst) good = good && touch(sl);
        for (int sl : nd.pslot_src2) good = good && touch(sl);
        for (int sl : nd.pslot_dst2) good = good && touch(sl);
        for (int sl : nd.n1_slot2) good = good && touch(sl);
        for (int sl : nd.tslot) good = good && touch(sl);
        if (!good) {
          err = "analyze: colour wave is not conflict-free at level " + std::to_string(i);
          return -2;
        }
      }
    }
    prev_p_exists = lv.p_exists;
    prev_slots = lv.slots;
  }
  pl.total_waves = total_waves;
  if (pl.max_edge_distance > 2) {
    err = "analyze: sparsity theorem violated (edge at distance > 2)";
    return -2;
  }

  // ---- leaf scatter map --------------------------------------------------------
  {
    const SymLevel &lv = pl.lev[L];
    std::unordered_map<uint64_t, int> slot_of;
    for (size_t sid = 0; sid < lv.slots.size(); ++sid)
      slot_of.emplace(sym ? key(lv.slots[sid].row, lv.slots[sid].col) : dkey(lv.slots[sid].col, lv.slots[sid].row),
                      (int)sid);
    pl.nnz_slot.assign(pl.nnz, -1);
    pl.nnz_r.assign(pl.nnz, 0);
    pl.nnz_c.assign(pl.nnz, 0);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
        int64_t j = col_idx[k];
        int v = pl.leaf_of[i], u = pl.leaf_of[j];  // Mat(u -> v) = A_{v,u}
        int sv = v >> 1, su = u >> 1;
        int ri = ((v & 1) ? pl.leaf_size[v - 1] : 0) + pl.leaf_pos[i];
        int ci = ((u & 1) ? pl.leaf_size[u - 1] : 0) + pl.leaf_pos[j];
        auto it = slot_of.find(sym ? key(sv, su) : dkey(su, sv));
        if (it == slot_of.end()) {
          err = "analyze: internal error (leaf slot missing)";
          return -2;
        }
        const SymSlot &sl = lv.slots[it->second];
        if (!sym || sv == su || sl.row == sv) {
          pl.nnz_slot[k] = it->second;
          pl.nnz_r[k] = ri;
          pl.nnz_c[k] = ci;
        }
        // else: the mirror entry (j, i) fills this element (symmetric store)
      }
  }
  return 0;
}

}  // namespace lorasp
