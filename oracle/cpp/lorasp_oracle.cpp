// ORACLE for the LoRaSp level sweep (arxiv 1510.07363) -- TEST INFRASTRUCTURE ONLY.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load this library (through oracle/cpp_oracle.py).  The
// product path (liblorasp, paper_1510_07363_b200/) never links or calls it.
// It shares no code, header, table or helper with paper_1510_07363_b200/csrc/:
// it is plain C++17 over std::vector, with NO BLAS / LAPACK, written from the
// paper (PAPER.md, cited "P:l.N") and the readings Z1-Z27 / F1-F4 listed in
// DESIGN.md §3.  Dense kernels are textbook loops:
//   * Householder QR and one-sided (Hestenes) Jacobi SVD        (Eq. lra, P:l.333-355)
//   * column-pivoted Householder QR (Businger-Golub) for RRQR   (f1, P:l.840, reading F1)
//   * partial-pivot LU solves of the pivot blocks               (Eq. elimination, P:l.101-106, Z11)
//   * matrix products as triple loops
//
// Algorithm, in the paper's order:
//   Def. nested partitionings (P:l.214-216) by recursive coordinate bisection (Z17)
//   or breadth-first level structures (F4); quotient graphs (P:l.247-249);
//   distances (P:l.506-512); Alg. 1 (P:l.265-289): MergeRedNodes (P:l.295-313),
//   Compress (P:l.319-394, five edge rules P:l.383-389, Eq. rhszero), Eliminate
//   (P:l.101-106, P:l.396-399); truncation Eq. cutOff1 (P:l.580-584) or the
//   Frobenius rule Eq. curOff6 (P:l.756-761, reading F2); Alg. 2-4 (P:l.407-500);
//   PCG / right-preconditioned GMRES(restart) (P:l.651-669, Z21) and the
//   paper's preconditioned residual Eq. GMRES_residual (P:l.665-669).
//
// Order within a level (Z1/Z2): colour-major order of a validated distance-2
// lattice colouring (greedy fallback), ascending cluster index within a colour;
// "natural" = the paper's literal ascending order.
//
// Parallelism (OpenMP) is across the super-nodes of one colour wave only, and
// only after an explicit check that the wave's nodes read and write pairwise
// disjoint blocks (check_wave_disjoint): under that check the result is, bit for
// bit, the sequential Alg. 1 in the same order, for any thread count (tested).
//
// The C API at the bottom is what oracle/cpp_oracle.py loads.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace orc {

// ---------------------------------------------------------------------------
// Node keys.  ('s', i, c) super-node s_c^[i] (cluster c of P_{i-1});
// ('b', i, c) black node b_c^[i]; ('r', k, c) red node of cluster c of P_k.
// P(b_c^[i]) = ('r', i-1, c) (Def. hierarchical tree, P:l.224-227).
// Integer order of the key = (kind rank s < b < r, level, cluster), the sort
// order used for partner and neighbour lists.
// ---------------------------------------------------------------------------
typedef uint64_t Key;
enum { KS = 0, KB = 1, KR = 2 };
static inline Key mk(int kind, int lev, int64_t c) {
  return ((Key)kind << 60) | ((Key)lev << 44) | (Key)c;
}
static inline int kind_of(Key k) { return (int)(k >> 60); }
static inline int lev_of(Key k) { return (int)((k >> 44) & 0xFFFF); }
static inline int64_t cl_of(Key k) { return (int64_t)(k & ((Key(1) << 44) - 1)); }

struct PairHash {
  size_t operator()(const std::pair<Key, Key> &p) const {
    return (size_t)(p.first * 0x9E3779B97F4A7C15ull ^ (p.second + 0x632BE59BD9B4E019ull + (p.first << 6)));
  }
};

// dense column-major block: rows = |v|, cols = |u| for Mat(e_{u->v}) (P:l.75, l.81)
struct Blk {
  int rows = 0, cols = 0;
  std::vector<double> a;
  Blk() {}
  Blk(int r, int c) : rows(r), cols(c), a((size_t)r * c, 0.0) {}
  double &at(int i, int j) { return a[(size_t)j * rows + i]; }
  double at(int i, int j) const { return a[(size_t)j * rows + i]; }
};

struct Err : std::runtime_error {
  int code;
  Err(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};
enum { E_ARG = -1, E_SINGULAR = -3, E_NOCONV = -4, E_STATE = -8, E_WAVE = -9 };

// ---------------------------------------------------------------------------
// Dense kernels (textbook loops, no BLAS)
// ---------------------------------------------------------------------------
// C (m x n) -= A (m x k) * B (k x n), all column-major with leading dims = rows
static void gemm_sub(int m, int n, int k, const double *A, const double *B, double *C) {
  for (int j = 0; j < n; ++j)
    for (int l = 0; l < k; ++l) {
      const double b = B[(size_t)j * k + l];
      if (b == 0.0) continue;
      const double *a = A + (size_t)l * m;
      double *c = C + (size_t)j * m;
      for (int i = 0; i < m; ++i) c[i] -= a[i] * b;
    }
}
// C (m x n) = A (m x k) * B (k x n)
static void gemm_set(int m, int n, int k, const double *A, const double *B, double *C) {
  std::fill(C, C + (size_t)m * n, 0.0);
  for (int j = 0; j < n; ++j)
    for (int l = 0; l < k; ++l) {
      const double b = B[(size_t)j * k + l];
      if (b == 0.0) continue;
      const double *a = A + (size_t)l * m;
      double *c = C + (size_t)j * m;
      for (int i = 0; i < m; ++i) c[i] += a[i] * b;
    }
}

// Partial-pivot LU (Doolittle, row interchanges): P A = L U stored in place.
struct LU {
  int n = 0;
  std::vector<double> a;   // column-major n x n, L (unit, below) and U
  std::vector<int> piv;    // row swapped with row k at step k
};
// reading Z11: singular if min |u_kk| < 1e-13 max |A_ij|
static void lu_factor(const Blk &A, LU &f) {
  const int n = A.rows;
  f.n = n;
  f.a = A.a;
  f.piv.assign(n, 0);
  double amax = 0.0;
  for (double v : A.a) amax = std::max(amax, std::fabs(v));
  double umin = INFINITY;
  double *a = f.a.data();
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = std::fabs(a[(size_t)k * n + k]);
    for (int i = k + 1; i < n; ++i)
      if (std::fabs(a[(size_t)k * n + i]) > best) {
        best = std::fabs(a[(size_t)k * n + i]);
        p = i;
      }
    f.piv[k] = p;
    if (p != k)
      for (int j = 0; j < n; ++j) std::swap(a[(size_t)j * n + k], a[(size_t)j * n + p]);
    const double ukk = a[(size_t)k * n + k];
    umin = std::min(umin, std::fabs(ukk));
    if (ukk == 0.0) continue;
    for (int i = k + 1; i < n; ++i) a[(size_t)k * n + i] /= ukk;
    for (int j = k + 1; j < n; ++j) {
      const double ukj = a[(size_t)j * n + k];
      if (ukj == 0.0) continue;
      for (int i = k + 1; i < n; ++i) a[(size_t)j * n + i] -= a[(size_t)k * n + i] * ukj;
    }
  }
  if (n > 0 && !(umin >= 1e-13 * std::max(amax, 1e-300))) throw Err(E_SINGULAR, "singular pivot");
}
// X (n x nrhs) <- A^{-1} X
static void lu_solve(const LU &f, double *X, int nrhs) {
  const int n = f.n;
  const double *a = f.a.data();
  for (int c = 0; c < nrhs; ++c) {
    double *x = X + (size_t)c * n;
    for (int k = 0; k < n; ++k)
      if (f.piv[k] != k) std::swap(x[k], x[f.piv[k]]);
    for (int k = 0; k < n; ++k) {   // L y = P x (unit lower)
      const double v = x[k];
      if (v == 0.0) continue;
      for (int i = k + 1; i < n; ++i) x[i] -= a[(size_t)k * n + i] * v;
    }
    for (int k = n - 1; k >= 0; --k) {   // U x = y
      x[k] /= a[(size_t)k * n + k];
      const double v = x[k];
      if (v == 0.0) continue;
      for (int i = 0; i < k; ++i) x[i] -= a[(size_t)k * n + i] * v;
    }
  }
}

// Householder reflector of x (len n): H x = beta e1, H = I - tau v v^T, v[0] = 1.
static void householder(double *x, int n, double &tau, double &beta) {
  double s = 0.0;
  for (int i = 1; i < n; ++i) s += x[i] * x[i];
  const double alpha = x[0];
  if (s == 0.0) {
    tau = 0.0;
    beta = alpha;
    return;
  }
  const double nrm = std::sqrt(alpha * alpha + s);
  beta = alpha <= 0.0 ? nrm : -nrm;
  const double v0 = alpha - beta;
  for (int i = 1; i < n; ++i) x[i] /= v0;
  tau = (beta - alpha) / beta;
  x[0] = 1.0;
}
// apply H = I - tau v v^T (v = x[k..R), v[0]=1 stored in column k of W) to columns j0..m-1
static void apply_householder(double *W, int R, int k, double tau, int j0, int m) {
  if (tau == 0.0) return;
  const double *v = W + (size_t)k * R + k;
  for (int j = j0; j < m; ++j) {
    double *w = W + (size_t)j * R + k;
    double d = 0.0;
    for (int i = 0; i < R - k; ++i) d += v[i] * w[i];
    d *= tau;
    for (int i = 0; i < R - k; ++i) w[i] -= d * v[i];
  }
}

// Right singular values / vectors of M (R x m, column-major): sigma descending
// (m values; the last m - min(R, m) are zero), V (m x m) orthogonal.
// Step 1 (only when R > m): Householder QR, M = Q T; T (m x m upper triangular)
// has the same singular values and right singular vectors as M.
// Step 2: one-sided Jacobi (Hestenes) on the columns of U (T, or M itself):
// rotate pairs (p, q) until every pair is orthogonal to |u_p.u_q| <= tol
// sqrt(|u_p|^2 |u_q|^2), tol = rows * DBL_EPSILON; then sigma_k = |u_k|, V = the
// accumulated rotations.  60 sweeps without convergence is an error (S:l.268).
static void svd_right(const double *M, int R, int m, std::vector<double> &sigma, std::vector<double> &V) {
  int rows;
  std::vector<double> U;
  if (R > m) {
    std::vector<double> W(M, M + (size_t)R * m);
    for (int k = 0; k < m; ++k) {
      double tau, beta;
      householder(W.data() + (size_t)k * R + k, R - k, tau, beta);
      apply_householder(W.data(), R, k, tau, k + 1, m);
      W[(size_t)k * R + k] = beta;
    }
    rows = m;
    U.assign((size_t)m * m, 0.0);
    for (int j = 0; j < m; ++j)
      for (int i = 0; i <= j; ++i) U[(size_t)j * m + i] = W[(size_t)j * R + i];
  } else {
    rows = R;
    U.assign(M, M + (size_t)R * m);
  }
  V.assign((size_t)m * m, 0.0);
  for (int j = 0; j < m; ++j) V[(size_t)j * m + j] = 1.0;
  const double tol = std::max(rows, 1) * DBL_EPSILON;
  // a column of norm <= tol ||M||_F is numerically zero: its rotations are skipped
  // (rank-deficient and wide stacks would otherwise rotate rounding noise forever;
  // the sigma it stands for is below every threshold eps sigma_0 used here)
  double fro2 = 0.0;
  for (double v : U) fro2 += v * v;
  const double negl = tol * tol * fro2;
  int sweep = 0;
  for (; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < m - 1; ++p)
      for (int q = p + 1; q < m; ++q) {
        double *up = U.data() + (size_t)p * rows, *uq = U.data() + (size_t)q * rows;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = 0; i < rows; ++i) {
          al += up[i] * up[i];
          be += uq[i] * uq[i];
          ga += up[i] * uq[i];
        }
        if (ga == 0.0 || std::fabs(ga) <= tol * std::sqrt(al * be) || std::min(al, be) <= negl) continue;
        rotated = true;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (int i = 0; i < rows; ++i) {
          const double a = up[i], b = uq[i];
          up[i] = c * a - s * b;
          uq[i] = s * a + c * b;
        }
        double *vp = V.data() + (size_t)p * m, *vq = V.data() + (size_t)q * m;
        for (int i = 0; i < m; ++i) {
          const double a = vp[i], b = vq[i];
          vp[i] = c * a - s * b;
          vq[i] = s * a + c * b;
        }
      }
    if (!rotated) break;
  }
  if (sweep == 60) throw Err(E_NOCONV, "one-sided Jacobi did not converge in 60 sweeps");
  std::vector<double> nrm(m);
  for (int j = 0; j < m; ++j) {
    double s = 0.0;
    for (int i = 0; i < rows; ++i) s += U[(size_t)j * rows + i] * U[(size_t)j * rows + i];
    nrm[j] = std::sqrt(s);
  }
  std::vector<int> idx(m);
  for (int j = 0; j < m; ++j) idx[j] = j;
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return nrm[a] > nrm[b]; });
  sigma.assign(m, 0.0);
  std::vector<double> Vs((size_t)m * m);
  for (int j = 0; j < m; ++j) {
    sigma[j] = nrm[idx[j]];
    const double *src = V.data() + (size_t)idx[j] * m;
    // sign: largest-magnitude entry positive (comparable dumps; V is basis-free, Z8)
    int im = 0;
    for (int i = 1; i < m; ++i)
      if (std::fabs(src[i]) > std::fabs(src[im])) im = i;
    const double sg = src[im] < 0.0 ? -1.0 : 1.0;
    for (int i = 0; i < m; ++i) Vs[(size_t)j * m + i] = sg * src[i];
  }
  V.swap(Vs);
}

// Column-pivoted Householder QR (Businger-Golub) of M (R x m): at step k the
// remaining column of largest norm over rows k..R-1 (ties -> smaller index) is
// swapped to position k.  Returns d_k = |R_kk| (k < min(R, m)) and the
// permutation, and leaves R (upper trapezoid) in W.
static void qr_colpiv(std::vector<double> &W, int R, int m, std::vector<double> &d, std::vector<int> &perm) {
  const int kmax = std::min(R, m);
  perm.resize(m);
  for (int j = 0; j < m; ++j) perm[j] = j;
  d.assign(kmax, 0.0);
  for (int k = 0; k < kmax; ++k) {
    int jb = k;
    double best = -1.0;
    for (int j = k; j < m; ++j) {
      double s = 0.0;
      const double *w = W.data() + (size_t)j * R;
      for (int i = k; i < R; ++i) s += w[i] * w[i];
      if (s > best) {
        best = s;
        jb = j;
      }
    }
    if (jb != k) {
      for (int i = 0; i < R; ++i) std::swap(W[(size_t)k * R + i], W[(size_t)jb * R + i]);
      std::swap(perm[k], perm[jb]);
    }
    double tau, beta;
    householder(W.data() + (size_t)k * R + k, R - k, tau, beta);
    apply_householder(W.data(), R, k, tau, k + 1, m);
    W[(size_t)k * R + k] = beta;
    for (int i = k + 1; i < R; ++i) W[(size_t)k * R + i] = 0.0;
    d[k] = std::fabs(beta);
  }
}
// Orthonormal basis (m x r) of the column span of X (m x r, full column rank):
// Householder QR, Q formed explicitly by applying the reflectors to I[:, :r].
static std::vector<double> orth_basis(const std::vector<double> &X, int m, int r) {
  std::vector<double> W = X;
  std::vector<double> taus(r);
  for (int k = 0; k < r; ++k) {
    double tau, beta;
    householder(W.data() + (size_t)k * m + k, m - k, tau, beta);
    apply_householder(W.data(), m, k, tau, k + 1, r);
    taus[k] = tau;
  }
  std::vector<double> Q((size_t)m * r, 0.0);
  for (int j = 0; j < r; ++j) Q[(size_t)j * m + j] = 1.0;
  for (int k = r - 1; k >= 0; --k) {   // Q = H_0 ... H_{r-1} I
    const double *v = W.data() + (size_t)k * m + k;
    for (int j = 0; j < r; ++j) {
      double *q = Q.data() + (size_t)j * m + k;
      double dd = 0.0;
      for (int i = 0; i < m - k; ++i) dd += (i == 0 ? 1.0 : v[i]) * q[i];
      dd *= taus[k];
      for (int i = 0; i < m - k; ++i) q[i] -= dd * (i == 0 ? 1.0 : v[i]);
    }
  }
  return Q;
}

// ---------------------------------------------------------------------------
// Nested partitionings (P:l.214-216)
// ---------------------------------------------------------------------------
struct Tree {
  int depth = 0;
  std::vector<std::vector<std::vector<int64_t>>> clusters;   // [k][c] ascending members
  std::vector<std::vector<int>> axis;                        // [k][c] split axis (k < depth)
  std::vector<int64_t> leaf_of;
};

// Recursive coordinate bisection (reading Z17): axis of largest extent (extents
// within a relative 1e-9 of the largest tie -> lowest axis), members sorted by
// (coordinate, index), the low half floor(|C|/2) is child 2c.
static Tree bisection_tree(int64_t n, int dim, const double *xy, int depth) {
  Tree t;
  t.depth = depth;
  t.clusters.resize(depth + 1);
  t.axis.resize(depth);
  t.clusters[0].resize(1);
  for (int64_t q = 0; q < n; ++q) t.clusters[0][0].push_back(q);
  for (int k = 0; k < depth; ++k) {
    const int64_t ncl = (int64_t)1 << k;
    t.axis[k].assign(ncl, 0);
    t.clusters[k + 1].resize(2 * ncl);
    for (int64_t c = 0; c < ncl; ++c) {
      const std::vector<int64_t> &mem = t.clusters[k][c];
      if (mem.empty()) continue;
      std::vector<double> lo(dim, INFINITY), hi(dim, -INFINITY);
      for (int64_t q : mem)
        for (int a = 0; a < dim; ++a) {
          lo[a] = std::min(lo[a], xy[q * dim + a]);
          hi[a] = std::max(hi[a], xy[q * dim + a]);
        }
      double emax = -INFINITY;
      for (int a = 0; a < dim; ++a) emax = std::max(emax, hi[a] - lo[a]);
      int ax = 0;
      for (int a = 0; a < dim; ++a)
        if (hi[a] - lo[a] >= emax * (1.0 - 1e-9)) {
          ax = a;
          break;
        }
      t.axis[k][c] = ax;
      std::vector<int64_t> srt = mem;
      std::sort(srt.begin(), srt.end(), [&](int64_t p, int64_t q) {
        const double xp = xy[p * dim + ax], xq = xy[q * dim + ax];
        return xp < xq || (xp == xq && p < q);
      });
      const size_t h = mem.size() / 2;
      std::vector<int64_t> a(srt.begin(), srt.begin() + h), b(srt.begin() + h, srt.end());
      std::sort(a.begin(), a.end());
      std::sort(b.begin(), b.end());
      t.clusters[k + 1][2 * c] = std::move(a);
      t.clusters[k + 1][2 * c + 1] = std::move(b);
    }
  }
  t.leaf_of.assign(n, 0);
  for (size_t c = 0; c < t.clusters[depth].size(); ++c)
    for (int64_t q : t.clusters[depth][c]) t.leaf_of[q] = (int64_t)c;
  return t;
}

// Algebraic bisection (reading F4): breadth-first level structure of the
// cluster's induced subgraph from a pseudo-peripheral vertex (BFS from the
// smallest member; then from the smallest vertex of the last level), members
// ordered by (level, index), unreachable members last; first floor(|C|/2) -> 2c.
static Tree bisection_tree_algebraic(int64_t n, const int64_t *rp, const int64_t *ci, int depth) {
  Tree t;
  t.depth = depth;
  t.clusters.resize(depth + 1);
  t.axis.resize(depth);
  t.clusters[0].resize(1);
  for (int64_t q = 0; q < n; ++q) t.clusters[0][0].push_back(q);
  std::vector<int64_t> inset(n, -1), lev(n, -1);
  const int64_t INF = (int64_t)1 << 60;
  auto bfs = [&](int64_t src, int64_t tag) {   // levels within the cluster tagged `tag`
    std::vector<int64_t> touched{src}, frontier{src};
    lev[src] = 0;
    while (!frontier.empty()) {
      std::vector<int64_t> nxt;
      for (int64_t v : frontier)
        for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {
          const int64_t j = ci[e];
          if (j != v && inset[j] == tag && lev[j] < 0) {
            lev[j] = lev[v] + 1;
            nxt.push_back(j);
            touched.push_back(j);
          }
        }
      frontier.swap(nxt);
    }
    return touched;
  };
  int64_t tag = 0;
  for (int k = 0; k < depth; ++k) {
    const int64_t ncl = (int64_t)1 << k;
    t.axis[k].assign(ncl, 0);
    t.clusters[k + 1].resize(2 * ncl);
    for (int64_t c = 0; c < ncl; ++c) {
      const std::vector<int64_t> &mem = t.clusters[k][c];
      if (mem.empty()) continue;
      ++tag;
      for (int64_t v : mem) inset[v] = tag;
      std::vector<int64_t> t1 = bfs(mem[0], tag);
      int64_t far = 0;
      for (int64_t v : t1) far = std::max(far, lev[v]);
      int64_t p = INF;
      for (int64_t v : t1)
        if (lev[v] == far) p = std::min(p, v);
      for (int64_t v : t1) lev[v] = -1;
      std::vector<int64_t> t2 = bfs(p, tag);
      std::vector<std::pair<int64_t, int64_t>> keyed;
      keyed.reserve(mem.size());
      for (int64_t v : mem) keyed.push_back({lev[v] < 0 ? INF : lev[v], v});
      for (int64_t v : t2) lev[v] = -1;
      std::sort(keyed.begin(), keyed.end());
      const size_t h = mem.size() / 2;
      std::vector<int64_t> a, b;
      for (size_t q = 0; q < keyed.size(); ++q) (q < h ? a : b).push_back(keyed[q].second);
      std::sort(a.begin(), a.end());
      std::sort(b.begin(), b.end());
      t.clusters[k + 1][2 * c] = std::move(a);
      t.clusters[k + 1][2 * c + 1] = std::move(b);
    }
  }
  t.leaf_of.assign(n, 0);
  for (size_t c = 0; c < t.clusters[depth].size(); ++c)
    for (int64_t q : t.clusters[depth][c]) t.leaf_of[q] = (int64_t)c;
  return t;
}

// ---------------------------------------------------------------------------
// Quotient graphs (P:l.247-249, symmetrised, Z9) and distance sets (P:l.506-512)
// ---------------------------------------------------------------------------
struct Level {
  std::vector<std::vector<int64_t>> N1, N2;   // sorted
  bool near1(int64_t a, int64_t b) const { return std::binary_search(N1[a].begin(), N1[a].end(), b); }
  bool near2(int64_t a, int64_t b) const { return std::binary_search(N2[a].begin(), N2[a].end(), b); }
};
static Level make_level(int64_t n, const int64_t *rp, const int64_t *ci, const std::vector<int64_t> &leaf_of,
                        int shift, int64_t ncl) {
  Level L;
  L.N1.assign(ncl, {});
  for (int64_t i = 0; i < n; ++i) {
    const int64_t a = leaf_of[i] >> shift;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      const int64_t b = leaf_of[ci[e]] >> shift;
      if (a != b) {
        L.N1[a].push_back(b);
        L.N1[b].push_back(a);
      }
    }
  }
  for (auto &v : L.N1) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
  L.N2.assign(ncl, {});
  for (int64_t c = 0; c < ncl; ++c) {
    std::vector<int64_t> two;
    for (int64_t q : L.N1[c])
      for (int64_t w : L.N1[q])
        if (w != c && !L.near1(c, w)) two.push_back(w);
    std::sort(two.begin(), two.end());
    two.erase(std::unique(two.begin(), two.end()), two.end());
    L.N2[c] = std::move(two);
  }
  return L;
}

// Distance-2 colouring (reading Z2): lattice rule colour = (sum_a (a+1) g_a) mod
// (2 dim + 1), g_a = the cluster's index along axis a read off its bisection
// path; accepted only if no two clusters within distance 2 share a colour, else
// greedy (ascending index, smallest colour unused by lower-indexed clusters
// within distance 2).
static std::vector<int> colour_level(const Tree &t, int k, int dim, const Level &L) {
  const int64_t ncl = (int64_t)1 << k;
  std::vector<int> col(ncl);
  for (int64_t c = 0; c < ncl; ++c) {
    std::vector<int64_t> g(dim, 0);
    for (int s = 0; s < k; ++s) {
      const int64_t anc = c >> (k - s), bit = (c >> (k - 1 - s)) & 1;
      const int a = t.axis[s][anc];
      g[a] = 2 * g[a] + bit;
    }
    int64_t sum = 0;
    for (int a = 0; a < dim; ++a) sum += (a + 1) * g[a];
    col[c] = (int)(sum % (2 * dim + 1));
  }
  bool ok = true;
  for (int64_t c = 0; c < ncl && ok; ++c) {
    for (int64_t q : L.N1[c]) ok = ok && col[q] != col[c];
    for (int64_t q : L.N2[c]) ok = ok && col[q] != col[c];
  }
  if (ok) return col;
  std::fill(col.begin(), col.end(), -1);
  for (int64_t c = 0; c < ncl; ++c) {
    std::set<int> used;
    for (int64_t q : L.N1[c])
      if (q < c) used.insert(col[q]);
    for (int64_t q : L.N2[c])
      if (q < c) used.insert(col[q]);
    int x = 0;
    while (used.count(x)) ++x;
    col[c] = x;
  }
  return col;
}

// ---------------------------------------------------------------------------
// The H-tree state and Alg. 1
// ---------------------------------------------------------------------------
enum { F_NATURAL = 1, F_SYMSTACK = 2, F_RRQR = 4, F_ALGEBRAIC = 8, F_TRACE = 16, F_FROBENIUS = 32 };

struct CompressOut {   // results of one Compress, computed before the edits
  std::vector<Key> partners;
  std::vector<double> sigma;   // min(R, m) values (RRQR: |R_kk|)
  int r = 0;
  std::vector<double> V;       // m x r
  std::vector<Blk> Rk, Qk;     // per partner: A_k V (|p| x r), B_k V (|p| x r)
};
struct ElimPlan {   // symbolic elimination of one node
  Key p = 0;
  bool active = false;   // size > 0
  std::vector<Key> ins, outs;
};

struct Factorizer {
  int64_t n = 0;
  int l = 0, dim = 1, flags = 0, nthreads = 1;
  double eps = 0.0;
  Tree tree;
  std::vector<Level> lev;   // quotient graph of P_k, k = 0..l
  std::unordered_map<Key, int> size;
  std::unordered_map<std::pair<Key, Key>, std::unique_ptr<Blk>, PairHash> M;   // (u, v): Mat(e_{u->v})
  std::unordered_map<Key, std::set<Key>> out, inn;
  std::unordered_set<Key> eliminated;
  std::unordered_map<Key, int64_t> order;
  int64_t counter = 0;
  std::unordered_map<Key, LU> pivots;
  std::map<std::pair<int, int64_t>, int> rank;
  std::map<std::pair<int, int64_t>, std::vector<double>> sigma;
  std::map<std::pair<int, int64_t>, int> npartners, nn1;
  std::vector<std::vector<int64_t>> level_order;     // [i]
  std::vector<std::vector<int>> level_wave;          // [i] wave id of each position
  std::vector<std::vector<char>> wave_solve_par;     // [i][wave] solve may run the wave in parallel
  std::vector<std::string> trace;
  int max_edge_distance = 0;
  int64_t waves_parallel = 0, waves_total = 0;

  int sz(Key u) const {
    auto it = size.find(u);
    return it == size.end() ? 0 : it->second;
  }
  std::pair<int, int64_t> cluster_level(Key u) const {   // (level of P, cluster)
    return kind_of(u) == KR ? std::make_pair(lev_of(u), cl_of(u)) : std::make_pair(lev_of(u) - 1, cl_of(u));
  }
  int distance(Key u, Key v) const {   // Def. distance (P:l.506-508)
    auto a = cluster_level(u), b = cluster_level(v);
    const int k = std::min(a.first, b.first);
    const int64_t cu = a.second >> (a.first - k), cv = b.second >> (b.first - k);
    if (cu == cv) return 0;
    if (lev[k].near1(cu, cv)) return 1;
    if (lev[k].near2(cu, cv)) return 2;
    return 3;
  }
  Blk *get(Key u, Key v) const {
    auto it = M.find({u, v});
    return it == M.end() ? nullptr : it->second.get();
  }
  Blk *set(Key u, Key v, Blk &&b) {
    auto &slot = M[{u, v}];
    slot.reset(new Blk(std::move(b)));
    out[u].insert(v);
    inn[v].insert(u);
    if (u != v) max_edge_distance = std::max(max_edge_distance, distance(u, v));
    return slot.get();
  }
  void del(Key u, Key v) {
    M.erase({u, v});
    auto io = out.find(u);
    if (io != out.end()) io->second.erase(v);
    auto ii = inn.find(v);
    if (ii != inn.end()) ii->second.erase(u);
  }
  Blk *get_or_zero(Key u, Key v) {
    Blk *b = get(u, v);
    return b ? b : set(u, v, Blk(sz(v), sz(u)));
  }
  std::vector<Key> nb_sorted(Key s) const {   // (out[s] | inn[s]) - {s}, sorted
    std::set<Key> nb;
    auto io = out.find(s);
    if (io != out.end()) nb.insert(io->second.begin(), io->second.end());
    auto ii = inn.find(s);
    if (ii != inn.end()) nb.insert(ii->second.begin(), ii->second.end());
    nb.erase(s);
    return std::vector<Key>(nb.begin(), nb.end());
  }
  std::string name(Key u) const {
    const char k = "sbr"[kind_of(u)];
    return std::string(1, k) + " " + std::to_string(lev_of(u)) + " " + std::to_string(cl_of(u));
  }

  // -- Initialize(l)  (P:l.291-293): Mat(e_{u->v}) = A_{v,u} ------------------
  void init_leaves(const int64_t *rp, const int64_t *ci, const double *va) {
    std::vector<int64_t> pos(n);
    for (size_t c = 0; c < tree.clusters[l].size(); ++c) {
      size[mk(KR, l, c)] = (int)tree.clusters[l][c].size();
      for (size_t t = 0; t < tree.clusters[l][c].size(); ++t) pos[tree.clusters[l][c][t]] = (int64_t)t;
    }
    for (int64_t i = 0; i < n; ++i)
      for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
        const int64_t j = ci[e];
        Blk *b = get_or_zero(mk(KR, l, tree.leaf_of[j]), mk(KR, l, tree.leaf_of[i]));
        b->at((int)pos[i], (int)pos[j]) += va[e];
      }
  }

  // -- MergeRedNodes  (P:l.295-313, Eq. merge) --------------------------------
  void merge(int i) {
    const int64_t nsup = (int64_t)1 << (i - 1);
    for (int64_t c = 0; c < nsup; ++c) size[mk(KS, i, c)] = sz(mk(KR, i, 2 * c)) + sz(mk(KR, i, 2 * c + 1));
    for (int64_t rc = 0; rc < 2 * nsup; ++rc) {
      const Key u = mk(KR, i, rc);
      auto io = out.find(u);
      if (io == out.end()) continue;
      std::vector<Key> tgts(io->second.begin(), io->second.end());
      for (Key v : tgts) {
        if (kind_of(v) != KR || lev_of(v) != i) continue;
        std::unique_ptr<Blk> blk = std::move(M[{u, v}]);
        del(u, v);
        const Key su = mk(KS, i, cl_of(u) / 2), sv = mk(KS, i, cl_of(v) / 2);
        // Mat(s_j -> s_j') = [[r0->r0', r1->r0'], [r0->r1', r1->r1']]
        const int ro = (cl_of(v) % 2 == 0) ? 0 : sz(mk(KR, i, cl_of(v) - 1));
        const int co = (cl_of(u) % 2 == 0) ? 0 : sz(mk(KR, i, cl_of(u) - 1));
        Blk *t = get_or_zero(su, sv);
        for (int jj = 0; jj < blk->cols; ++jj)
          for (int ii = 0; ii < blk->rows; ++ii) t->at(ro + ii, co + jj) += blk->at(ii, jj);
      }
    }
    if (flags & F_TRACE) trace.push_back("merge " + std::to_string(i));
  }

  // -- Compress numerics (P:l.319-358): reads the store only ------------------
  void compress_compute(int i, int64_t c, CompressOut &co) const {
    const Key s = mk(KS, i, c);
    const int m = sz(s);
    for (Key u : nb_sorted(s))
      if (!eliminated.count(u) && sz(u) > 0 && distance(s, u) >= 2) co.partners.push_back(u);
    co.r = 0;
    if (m == 0 || co.partners.empty()) return;
    // Eq. lra: stack A_k = Mat(s->p_k) (|p_k| x m) and B_k with B_k^T = Mat(p_k->s)
    const bool sym = flags & F_SYMSTACK;
    int R = 0;
    for (Key p : co.partners) R += sz(p);
    const int Rtot = sym ? R : 2 * R;
    std::vector<double> S((size_t)Rtot * m, 0.0);
    int off = 0;
    for (Key p : co.partners) {
      const int mp = sz(p);
      if (const Blk *A = get(s, p))
        for (int j = 0; j < m; ++j)
          for (int t = 0; t < mp; ++t) S[(size_t)j * Rtot + off + t] = A->at(t, j);
      off += mp;
    }
    if (!sym)
      for (Key p : co.partners) {
        const int mp = sz(p);
        if (const Blk *B = get(p, s))   // B (m x mp) = Mat(p->s); stack B^T
          for (int j = 0; j < m; ++j)
            for (int t = 0; t < mp; ++t) S[(size_t)j * Rtot + off + t] = B->at(j, t);
        off += mp;
      }
    std::vector<double> Vfull;
    if (flags & F_RRQR) {
      // f1 (reading F1): |R_kk| >= eps |R_00| prefix; V = orthonormal basis of the
      // rows of R[:r, :] P^T
      std::vector<double> W = S, d;
      std::vector<int> perm;
      qr_colpiv(W, Rtot, m, d, perm);
      co.sigma.assign(m, 0.0);
      for (size_t k = 0; k < d.size(); ++k) co.sigma[k] = d[k];
      int r;
      if (d.empty() || d[0] == 0.0) r = 0;                       // Z4
      else if (eps == 0.0) r = m;                                // Z3
      else {
        r = (int)d.size();
        for (size_t k = 0; k < d.size(); ++k)
          if (d[k] < eps * d[0]) {
            r = (int)k;
            break;
          }
      }
      co.r = r;
      if (r == 0) return;
      if (r > (int)d.size()) {   // eps = 0 with fewer rows than columns
        co.V.assign((size_t)m * r, 0.0);
        for (int j = 0; j < r; ++j) co.V[(size_t)j * m + j] = 1.0;
      } else {
        std::vector<double> X((size_t)m * r, 0.0);   // X[perm[j], t] = R[t, j]
        for (int j = 0; j < m; ++j)
          for (int t = 0; t < r && t <= j; ++t) X[(size_t)t * m + perm[j]] = W[(size_t)j * Rtot + t];
        co.V = orth_basis(X, m, r);
      }
    } else {
      std::vector<double> sg;
      svd_right(S.data(), Rtot, m, sg, Vfull);
      co.sigma.assign(sg.begin(), sg.begin() + std::min(Rtot, m));
      const double s0 = sg.empty() ? 0.0 : sg[0];
      int r = 0;
      if (s0 == 0.0) r = 0;                                      // Z4
      else if (eps == 0.0) r = m;                                // Z3: nothing truncated
      else if (flags & F_FROBENIUS) r = frobenius_rank(sg);
      else
        for (int k = 0; k < m; ++k) r += sg[k] >= eps * s0;     // Eq. cutOff1, ties kept (Z5)
      co.r = r;
      co.V.assign(Vfull.begin(), Vfull.begin() + (size_t)m * r);
    }
    // Eqs. anterpol / interpol: R_k = A_k V, Q_k = B_k V
    const int r = co.r;
    for (Key p : co.partners) {
      const int mp = sz(p);
      Blk Rk(mp, r), Qk(mp, r);
      if (const Blk *A = get(s, p)) gemm_set(mp, r, m, A->a.data(), co.V.data(), Rk.a.data());
      if (const Blk *B = get(p, s)) {   // B_k = Mat(p->s)^T (mp x m)
        std::vector<double> Bt((size_t)mp * m);
        for (int j = 0; j < m; ++j)
          for (int t = 0; t < mp; ++t) Bt[(size_t)j * mp + t] = B->at(j, t);
        gemm_set(mp, r, m, Bt.data(), co.V.data(), Qk.a.data());
      }
      co.Rk.push_back(std::move(Rk));
      co.Qk.push_back(std::move(Qk));
    }
  }
  // F2, Eq. curOff6 (P:l.756-761): r = the smallest k with
  //   ||B - U_k S_k V_k^T||_F = sqrt(sum_{t >= k} sigma_t^2) < eps ||all levels below||_F,
  // reading F2: ||all levels below||_F^2 = frob_D2 = sum over the levels j >= i
  // processed so far (this one included) of the squared Frobenius norms of every
  // super-node block Mat(u -> v) present right after MergeRedNodes of level j.
  // The SPD-path stack [A] carries half the energy of [A; B] (sigma^2 doubles).
  int frobenius_rank(const std::vector<double> &sg) const {
    const double budget = eps * eps * frob_D2;
    const double w = (flags & F_SYMSTACK) ? 2.0 : 1.0;
    int r = (int)sg.size();
    double tail = 0.0;
    while (r > 0 && tail + w * sg[r - 1] * sg[r - 1] < budget) {
      tail += w * sg[r - 1] * sg[r - 1];
      --r;
    }
    return r;
  }
  double frob_D2 = 0.0;
  std::map<int, double> frob_level;   // D^2 in force while level i is processed

  // -- Compress edits: edge rules (P:l.383-389) --------------------------------
  void compress_apply(int i, int64_t c, CompressOut &co) {
    const Key s = mk(KS, i, c), b = mk(KB, i, c), P = mk(KR, i - 1, c);
    const int m = sz(s);
    rank[{i, c}] = co.r;
    sigma[{i, c}] = co.sigma;
    npartners[{i, c}] = (int)co.partners.size();
    if (m == 0 || co.partners.empty()) {
      size[b] = size[P] = 0;
      return;
    }
    if (flags & F_TRACE) {
      std::string t = "compress " + name(s) + " :";
      for (size_t k = 0; k < co.partners.size(); ++k) t += " " + name(co.partners[k]);
      trace.push_back(t);
    }
    for (Key p : co.partners) {   // rule 1: remove s -> p_k, p_k -> s
      del(s, p);
      del(p, s);
    }
    const int r = co.r;
    size[b] = size[P] = r;
    if (r == 0) return;
    for (size_t k = 0; k < co.partners.size(); ++k) {
      const Key p = co.partners[k];
      set(P, p, std::move(co.Rk[k]));                 // rule 2: P(b) -> p_k with R_k
      const Blk &Q = co.Qk[k];                        // rule 3: p_k -> P(b) with Q_k^T
      Blk Qt(r, Q.rows);
      for (int j = 0; j < Q.rows; ++j)
        for (int t = 0; t < r; ++t) Qt.at(t, j) = Q.at(j, t);
      set(p, P, std::move(Qt));
    }
    Blk Vt(r, m), Vb(m, r);                           // rule 4: s -> b (V^T), b -> s (V)
    for (int j = 0; j < r; ++j)
      for (int t = 0; t < m; ++t) {
        Vt.at(j, t) = co.V[(size_t)j * m + t];
        Vb.at(t, j) = co.V[(size_t)j * m + t];
      }
    set(s, b, std::move(Vt));
    set(b, s, std::move(Vb));
    Blk I1(r, r), I2(r, r);                           // rule 5: b <-> P(b) with -I_r
    for (int t = 0; t < r; ++t) I1.at(t, t) = I2.at(t, t) = -1.0;
    set(b, P, std::move(I1));
    set(P, b, std::move(I2));
    // RHS(b) = RHS(P(b)) = 0 (Eq. rhszero) -- applied in the solve
  }

  // -- Eliminate (P:l.101-106, l.396-399): symbolic part -----------------------
  ElimPlan elim_symbolic(Key p) {
    ElimPlan e;
    e.p = p;
    if (sz(p) > 0) {
      if (!get(p, p)) throw Err(E_SINGULAR, "node " + name(p) + " has no pivot block");
      e.active = true;
      for (Key k : inn[p])
        if (k != p && !eliminated.count(k)) e.ins.push_back(k);
      for (Key j : out[p])
        if (j != p && !eliminated.count(j)) e.outs.push_back(j);
      for (Key k : e.ins)
        for (Key j : e.outs) get_or_zero(k, j);
    }
    eliminated.insert(p);
    order[p] = counter++;
    if ((flags & F_TRACE) && e.active) trace.push_back("eliminate " + name(p));
    return e;
  }
  // numeric part: Mat(k->j) -= Mat(p->j) Mat(p->p)^{-1} Mat(k->p)
  void elim_numeric(const ElimPlan &e, LU &lu) const {
    if (!e.active) return;
    const Blk *piv = get(e.p, e.p);
    lu_factor(*piv, lu);
    const int m = piv->rows;
    for (Key k : e.ins) {
      const Blk *Mkp = get(k, e.p);
      Blk X = *Mkp;   // m x |k|
      lu_solve(lu, X.a.data(), X.cols);
      for (Key j : e.outs) {
        const Blk *Mpj = get(e.p, j);   // |j| x m
        Blk *T = get(k, j);             // |j| x |k|
        gemm_sub(T->rows, T->cols, m, Mpj->a.data(), X.a.data(), T->a.data());
      }
    }
  }

  // Blocks a node's compress + elimination reads and writes: the wave may run in
  // parallel only if no node writes a block another node reads or writes, and no
  // node's adjacency changes under another (then any schedule = the sequential one).
  struct Footprint {
    std::vector<std::pair<Key, Key>> rd, wr;
  };
  Footprint footprint(int i, int64_t c, const CompressOut &co, const ElimPlan &es, const ElimPlan &eb) const {
    Footprint f;
    const Key s = mk(KS, i, c), b = mk(KB, i, c), P = mk(KR, i - 1, c);
    for (Key p : co.partners) {
      f.rd.push_back({s, p});
      f.rd.push_back({p, s});
      f.wr.push_back({s, p});
      f.wr.push_back({p, s});
      f.wr.push_back({P, p});
      f.wr.push_back({p, P});
    }
    f.wr.push_back({s, b});
    f.wr.push_back({b, s});
    f.wr.push_back({b, P});
    f.wr.push_back({P, b});
    for (const ElimPlan *e : {&es, &eb}) {
      if (!e->active) continue;
      f.rd.push_back({e->p, e->p});
      for (Key k : e->ins) f.rd.push_back({k, e->p});
      for (Key j : e->outs) f.rd.push_back({e->p, j});
      for (Key k : e->ins)
        for (Key j : e->outs) f.wr.push_back({k, j});
    }
    return f;
  }
  bool wave_disjoint(const std::vector<Footprint> &fp, const std::vector<Key> &sup) const {
    std::unordered_map<std::pair<Key, Key>, int, PairHash> writer;
    std::unordered_map<Key, int> touched;   // nodes whose adjacency a node edits
    for (size_t a = 0; a < fp.size(); ++a)
      for (auto &w : fp[a].wr) {
        auto it = writer.find(w);
        if (it != writer.end() && it->second != (int)a) return false;
        writer[w] = (int)a;
        for (Key x : {w.first, w.second}) {
          auto t = touched.find(x);
          if (t == touched.end()) touched[x] = (int)a;
          else if (t->second != (int)a) touched[x] = -1;   // shared partner: edits on distinct blocks
        }
      }
    for (size_t a = 0; a < fp.size(); ++a) {
      for (auto &r : fp[a].rd) {
        auto it = writer.find(r);
        if (it != writer.end() && it->second != (int)a) return false;
      }
      // another node must not edit s's adjacency (its partner list was read first)
      auto t = touched.find(sup[a]);
      if (t != touched.end() && t->second != (int)a) return false;
    }
    return true;
  }

  // -- Alg. 1 (P:l.265-289) ----------------------------------------------------
  void run() {
    level_order.assign(l + 1, {});
    level_wave.assign(l + 1, {});
    wave_solve_par.assign(l + 1, {});
    for (int i = l; i >= 1; --i) {
      merge(i);
      if (flags & F_FROBENIUS)   // reading F2: this level's super-node blocks join the denominator
        for (auto &kv : M)
          if (kind_of(kv.first.first) == KS && lev_of(kv.first.first) == i && kind_of(kv.first.second) == KS &&
              lev_of(kv.first.second) == i)
            for (double v : kv.second->a) frob_D2 += v * v;
      frob_level[i] = frob_D2;
      const int k = i - 1;
      const int64_t ncl = (int64_t)1 << k;
      std::vector<int64_t> seq(ncl);
      for (int64_t c = 0; c < ncl; ++c) seq[c] = c;
      std::vector<int> col(ncl, 0);
      if (flags & F_NATURAL) {
        for (int64_t c = 0; c < ncl; ++c) col[c] = (int)c;   // one node per wave
      } else {
        col = colour_level(tree, k, dim, lev[k]);
        std::stable_sort(seq.begin(), seq.end(), [&](int64_t a, int64_t b) { return col[a] < col[b]; });
      }
      level_order[i] = seq;
      level_wave[i].assign(ncl, 0);
      size_t w0 = 0;
      int wid = 0;
      while (w0 < seq.size()) {
        size_t w1 = w0 + 1;
        while (w1 < seq.size() && col[seq[w1]] == col[seq[w0]]) ++w1;
        for (size_t t = w0; t < w1; ++t) level_wave[i][t] = wid;
        wave_solve_par[i].push_back(run_wave(i, std::vector<int64_t>(seq.begin() + w0, seq.begin() + w1)));
        ++wid;
        w0 = w1;
      }
    }
  }

  // one colour wave: (1) compress numerics of every node (read-only), (2) in
  // order: edits, N1, symbolic elimination of s then b, (3) numeric elimination.
  // A wave whose footprints are not disjoint runs node by node (sequential).
  char run_wave(int i, const std::vector<int64_t> &wave) {
    const size_t W = wave.size();
    ++waves_total;
    std::vector<CompressOut> co(W);
    std::vector<ElimPlan> es(W), eb(W);
    std::vector<Footprint> fp(W);
    std::vector<LU> lus(W), lub(W);
    if (W > 1 && nthreads > 1) {
      // (1) parallel compress numerics on a copy-free read-only store
      std::vector<std::string> errs(W);
      std::vector<int> codes(W, 0);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
      for (long t = 0; t < (long)W; ++t) {
        try {
          compress_compute(i, wave[t], co[t]);
        } catch (const Err &e) {
          codes[t] = e.code;
          errs[t] = e.what();
        }
      }
      for (size_t t = 0; t < W; ++t)
        if (codes[t]) throw Err(codes[t], errs[t]);
      // (2) structural edits in order; then the footprints are checked: an
      // overlap is an error (distance-2 colouring makes them disjoint, SURVEY
      // 8.0; the sequential 1-thread run has no such check and is the fallback)
      for (size_t t = 0; t < W; ++t) {
        compress_apply(i, wave[t], co[t]);
        nn1[{i, wave[t]}] = (int)nb_now(mk(KS, i, wave[t])).size();
        es[t] = elim_symbolic(mk(KS, i, wave[t]));
        eb[t] = elim_symbolic(mk(KB, i, wave[t]));
        fp[t] = footprint(i, wave[t], co[t], es[t], eb[t]);
      }
      std::vector<Key> sup(W);
      for (size_t t = 0; t < W; ++t) sup[t] = mk(KS, i, wave[t]);
      if (!wave_disjoint(fp, sup)) throw Err(E_WAVE, "wave footprints overlap at level " + std::to_string(i));
      ++waves_parallel;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
      for (long t = 0; t < (long)W; ++t) {
        try {
          elim_numeric(es[t], lus[t]);
          elim_numeric(eb[t], lub[t]);
        } catch (const Err &e) {
          codes[t] = e.code;
          errs[t] = e.what() + std::string(" at ") + name(es[t].p);
        }
      }
      for (size_t t = 0; t < W; ++t)
        if (codes[t]) throw Err(codes[t], errs[t]);
    } else {
      for (size_t t = 0; t < W; ++t) {
        compress_compute(i, wave[t], co[t]);
        compress_apply(i, wave[t], co[t]);
        nn1[{i, wave[t]}] = (int)nb_now(mk(KS, i, wave[t])).size();
        es[t] = elim_symbolic(mk(KS, i, wave[t]));
        try {
          elim_numeric(es[t], lus[t]);
        } catch (const Err &e) {
          throw Err(e.code, std::string(e.what()) + " at " + name(es[t].p));
        }
        eb[t] = elim_symbolic(mk(KB, i, wave[t]));
        try {
          elim_numeric(eb[t], lub[t]);
        } catch (const Err &e) {
          throw Err(e.code, std::string(e.what()) + " at " + name(eb[t].p));
        }
        fp[t] = footprint(i, wave[t], co[t], es[t], eb[t]);
      }
    }
    for (size_t t = 0; t < W; ++t) {
      if (es[t].active) pivots[es[t].p] = std::move(lus[t]);
      if (eb[t].active) pivots[eb[t].p] = std::move(lub[t]);
    }
    // the solve may run this wave's nodes in parallel iff their forward targets
    // (out-neighbours eliminated later, reds) are pairwise disjoint
    std::unordered_map<Key, size_t> tgt;
    for (size_t t = 0; t < W; ++t)
      for (const ElimPlan *e : {&es[t], &eb[t]}) {
        for (Key q : e->outs) {
          auto it = tgt.find(q);
          if (it != tgt.end() && it->second != t) return 0;
          tgt[q] = t;
        }
      }
    return 1;
  }
  std::vector<Key> nb_now(Key s) const {
    std::vector<Key> r;
    for (Key u : nb_sorted(s))
      if (!eliminated.count(u)) r.push_back(u);
    return r;
  }

  // ---------------------------------------------------------------------------
  // Alg. 2-4 (P:l.401-500): x ~= A^{-1} b
  // ---------------------------------------------------------------------------
  double ord(Key q) const {   // reds are eliminated as part of the next level's super-node
    if (kind_of(q) == KR) return INFINITY;
    auto it = order.find(q);
    return it == order.end() ? INFINITY : (double)it->second;
  }
  void solve(const double *b, double *x, int nth) const {
    std::unordered_map<Key, std::vector<double>> rhs, var;
    for (size_t c = 0; c < tree.clusters[l].size(); ++c) {   // SetRHS: leaves get b
      std::vector<double> v;
      for (int64_t q : tree.clusters[l][c]) v.push_back(b[q]);
      rhs[mk(KR, l, c)] = std::move(v);
    }
    // every node that can appear gets its (zero) RHS first (Eq. rhszero), so the
    // parallel waves below never insert into the maps
    for (auto &kv : size)
      if (!rhs.count(kv.first)) rhs[kv.first].assign(kv.second, 0.0);
    for (auto &kv : size) var[kv.first];
    auto solve_l = [&](Key p) {   // Alg. 3
      if (sz(p) == 0) return;
      std::vector<double> f = rhs.at(p);
      lu_solve(pivots.at(p), f.data(), 1);
      const double op = ord(p);
      for (Key q : out.at(p))
        if (q != p && ord(q) > op) {
          const Blk *B = get(p, q);   // |q| x |p|
          std::vector<double> &rq = rhs.at(q);
          gemm_sub(B->rows, 1, B->cols, B->a.data(), f.data(), rq.data());
        }
    };
    auto solve_u = [&](Key p) {   // Alg. 4
      if (sz(p) == 0) {
        var.at(p).clear();
        return;
      }
      std::vector<double> v = rhs.at(p);
      const double op = ord(p);
      auto ii = inn.find(p);
      if (ii != inn.end())
        for (Key q : ii->second)
          if (q != p && ord(q) > op) {
            const Blk *B = get(q, p);   // |p| x |q|
            gemm_sub(B->rows, 1, B->cols, B->a.data(), var.at(q).data(), v.data());
          }
      lu_solve(pivots.at(p), v.data(), 1);
      var.at(p) = std::move(v);
    };
    for (int i = l; i >= 1; --i) {   // forward substitution
      for (int64_t c = 0; c < ((int64_t)1 << (i - 1)); ++c) {   // Eq. concatRHS
        std::vector<double> v = rhs.at(mk(KR, i, 2 * c));
        const std::vector<double> &w = rhs.at(mk(KR, i, 2 * c + 1));
        v.insert(v.end(), w.begin(), w.end());
        rhs[mk(KS, i, c)] = std::move(v);
      }
      const auto &seq = level_order[i];
      size_t w0 = 0;
      while (w0 < seq.size()) {
        size_t w1 = w0 + 1;
        while (w1 < seq.size() && level_wave[i][w1] == level_wave[i][w0]) ++w1;
        const bool par = nth > 1 && wave_solve_par[i][level_wave[i][w0]];
#pragma omp parallel for schedule(dynamic, 1) num_threads(nth) if (par)
        for (long t = (long)w0; t < (long)w1; ++t) {
          solve_l(mk(KS, i, seq[t]));
          solve_l(mk(KB, i, seq[t]));
        }
        w0 = w1;
      }
    }
    for (int i = 1; i <= l; ++i) {   // backward substitution, reverse order
      const auto &seq = level_order[i];
      size_t w1 = seq.size();
      while (w1 > 0) {
        size_t w0 = w1 - 1;
        while (w0 > 0 && level_wave[i][w0 - 1] == level_wave[i][w1 - 1]) --w0;
        const bool par = nth > 1 && wave_solve_par[i][level_wave[i][w0]];
#pragma omp parallel for schedule(dynamic, 1) num_threads(nth) if (par)
        for (long t = (long)w1 - 1; t >= (long)w0; --t) {
          solve_u(mk(KB, i, seq[t]));
          solve_u(mk(KS, i, seq[t]));
        }
        w1 = w0;
      }
      for (int64_t c = 0; c < ((int64_t)1 << (i - 1)); ++c) {   // SplitVar (Eq. concatX)
        const std::vector<double> &s = var.at(mk(KS, i, c));
        const int n0 = sz(mk(KR, i, 2 * c));
        var[mk(KR, i, 2 * c)] = std::vector<double>(s.begin(), s.begin() + std::min<size_t>(n0, s.size()));
        var[mk(KR, i, 2 * c + 1)] = std::vector<double>(s.begin() + std::min<size_t>(n0, s.size()), s.end());
      }
    }
    for (size_t c = 0; c < tree.clusters[l].size(); ++c) {
      const std::vector<double> &v = var.at(mk(KR, l, c));
      for (size_t t = 0; t < tree.clusters[l][c].size(); ++t) x[tree.clusters[l][c][t]] = v[t];
    }
  }
};

// ---------------------------------------------------------------------------
// Krylov consumers (P:l.651-669)
// ---------------------------------------------------------------------------
struct Csr {
  int64_t n;
  const int64_t *rp, *ci;
  const double *va;
};
static void spmv(const Csr &A, const double *x, double *y) {   // y = A x, row by row
  for (int64_t i = 0; i < A.n; ++i) {
    double s = 0.0;
    for (int64_t e = A.rp[i]; e < A.rp[i + 1]; ++e) s += A.va[e] * x[A.ci[e]];
    y[i] = s;
  }
}
static double dot(const std::vector<double> &a, const std::vector<double> &b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
static double nrm2(const std::vector<double> &a) { return std::sqrt(dot(a, a)); }
static double true_relres(const Csr &A, const double *b, const std::vector<double> &x, double nb) {
  std::vector<double> r(A.n);
  spmv(A, x.data(), r.data());
  for (int64_t i = 0; i < A.n; ++i) r[i] = b[i] - r[i];
  return nrm2(r) / nb;
}

struct KrylovOut {
  int iters = 0, converged = 0, breakdown = 0;
  double relres = 0.0;
};
// PCG (readings Z21/Z24/Z27): x0 = 0; stop when ||r_k|| / ||b|| <= tol; iters =
// number of A-products; breakdown when p^T A p <= 0 or r^T z <= 0.
static KrylovOut pcg(const Csr &A, const Factorizer &F, int nth, const double *b, double *xo, double tol, int maxit) {
  const int64_t n = A.n;
  std::vector<double> bb(b, b + n), x(n, 0.0), r = bb, z(n), p, q(n);
  KrylovOut o;
  const double nb = nrm2(bb);
  if (nb == 0.0) {
    std::copy(x.begin(), x.end(), xo);
    o.converged = 1;
    return o;
  }
  F.solve(r.data(), z.data(), nth);
  p = z;
  double rz = dot(r, z);
  int it = 1;
  for (; it <= maxit; ++it) {
    spmv(A, p.data(), q.data());
    const double pq = dot(p, q);
    if (pq <= 0.0 || rz <= 0.0) {
      o.iters = it - 1;
      o.breakdown = 1;
      o.relres = true_relres(A, b, x, nb);
      std::copy(x.begin(), x.end(), xo);
      return o;
    }
    const double alpha = rz / pq;
    for (int64_t i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * q[i];
    }
    if (nrm2(r) / nb <= tol) {
      o.iters = it;
      o.converged = 1;
      o.relres = true_relres(A, b, x, nb);
      std::copy(x.begin(), x.end(), xo);
      return o;
    }
    F.solve(r.data(), z.data(), nth);
    const double rz2 = dot(r, z);
    const double beta = rz2 / rz;
    for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    rz = rz2;
  }
  o.iters = maxit;
  o.relres = true_relres(A, b, x, nb);
  std::copy(x.begin(), x.end(), xo);
  return o;
}
// Right-preconditioned GMRES(restart) (reading Z21): A M y = b, x = M y, MGS
// Arnoldi, Givens rotations, stop on the recurrence estimate |g_{k+1}| / ||b||
// <= tol; iters = number of Arnoldi steps; true residual checked at exit.
static KrylovOut gmres(const Csr &A, const Factorizer &F, int nth, const double *b, double *xo, double tol,
                       int restart, int maxit) {
  const int64_t n = A.n;
  std::vector<double> x(n, 0.0);
  KrylovOut o;
  std::vector<double> bb(b, b + n);
  const double nb = nrm2(bb);
  if (nb == 0.0) {
    std::copy(x.begin(), x.end(), xo);
    o.converged = 1;
    return o;
  }
  int it = 0;
  std::vector<double> w(n), Ax(n);
  while (it < maxit) {
    spmv(A, x.data(), Ax.data());
    std::vector<double> r(n);
    for (int64_t i = 0; i < n; ++i) r[i] = b[i] - Ax[i];
    const double beta = nrm2(r);
    if (beta / nb <= tol) {
      o.iters = it;
      o.converged = 1;
      o.relres = beta / nb;
      std::copy(x.begin(), x.end(), xo);
      return o;
    }
    std::vector<std::vector<double>> Vb{r}, Z;
    for (auto &v : Vb[0]) v /= beta;
    std::vector<double> H((size_t)(restart + 1) * restart, 0.0), cs(restart), sn(restart), g(restart + 1, 0.0);
    auto h = [&](int i, int j) -> double & { return H[(size_t)j * (restart + 1) + i]; };
    g[0] = beta;
    int k_used = 0;
    bool done = false;
    for (int k = 0; k < restart; ++k) {
      std::vector<double> z(n);
      F.solve(Vb[k].data(), z.data(), nth);
      spmv(A, z.data(), w.data());
      Z.push_back(std::move(z));
      for (int j = 0; j <= k; ++j) {   // modified Gram-Schmidt
        h(j, k) = dot(w, Vb[j]);
        for (int64_t i = 0; i < n; ++i) w[i] -= h(j, k) * Vb[j][i];
      }
      const double hn = nrm2(w);
      h(k + 1, k) = hn;
      for (int j = 0; j < k; ++j) {   // previous Givens rotations
        const double t = cs[j] * h(j, k) + sn[j] * h(j + 1, k);
        h(j + 1, k) = -sn[j] * h(j, k) + cs[j] * h(j + 1, k);
        h(j, k) = t;
      }
      const double den = std::hypot(h(k, k), h(k + 1, k));
      if (den == 0.0) {
        cs[k] = 1.0;
        sn[k] = 0.0;
      } else {
        cs[k] = h(k, k) / den;
        sn[k] = h(k + 1, k) / den;
      }
      h(k, k) = cs[k] * h(k, k) + sn[k] * h(k + 1, k);
      h(k + 1, k) = 0.0;
      g[k + 1] = -sn[k] * g[k];
      g[k] = cs[k] * g[k];
      ++it;
      k_used = k + 1;
      if (std::fabs(g[k + 1]) / nb <= tol || it >= maxit) {
        done = true;
        break;
      }
      if (hn == 0.0 && den == 0.0) {
        done = true;
        break;
      }
      std::vector<double> v = w;
      const double d = hn > 0.0 ? hn : 1.0;
      for (auto &e : v) e /= d;
      Vb.push_back(std::move(v));
    }
    std::vector<double> y(k_used);   // back substitution H y = g
    for (int i = k_used - 1; i >= 0; --i) {
      double s = g[i];
      for (int j = i + 1; j < k_used; ++j) s -= h(i, j) * y[j];
      y[i] = s / h(i, i);
    }
    for (int j = 0; j < k_used; ++j)
      for (int64_t i = 0; i < n; ++i) x[i] += y[j] * Z[j][i];
    if (done) {
      const double rel = true_relres(A, b, x, nb);
      o.iters = it;
      o.relres = rel;
      o.converged = (rel <= tol * 10 || std::fabs(g[k_used]) / nb <= tol) ? 1 : 0;
      std::copy(x.begin(), x.end(), xo);
      return o;
    }
  }
  o.iters = it;
  o.relres = true_relres(A, b, x, nb);
  o.converged = o.relres <= tol;
  std::copy(x.begin(), x.end(), xo);
  return o;
}

}  // namespace orc

// ---------------------------------------------------------------------------
// C API (loaded by oracle/cpp_oracle.py)
// ---------------------------------------------------------------------------
using namespace orc;
static thread_local std::string g_err;

extern "C" {
typedef struct OrcHandle {
  Factorizer F;
} OrcHandle;

const char *orc_last_error() { return g_err.c_str(); }

int orc_factorize(int64_t n, const int64_t *rp, const int64_t *ci, const double *va, int dim, const double *xy,
                  int depth, double eps, int flags, int nthreads, OrcHandle **out) {
  try {
    if (n <= 0 || depth < 1 || depth > 30 || eps < 0.0 || !out) throw Err(E_ARG, "bad argument");
    std::unique_ptr<OrcHandle> h(new OrcHandle);
    Factorizer &F = h->F;
    F.n = n;
    F.l = depth;
    F.eps = eps;
    F.flags = flags;
    F.nthreads = std::max(1, nthreads);
    if (flags & F_ALGEBRAIC) {
      F.dim = 1;
      F.tree = bisection_tree_algebraic(n, rp, ci, depth);
    } else {
      F.dim = dim;
      F.tree = bisection_tree(n, dim, xy, depth);
    }
    F.lev.resize(depth + 1);
    for (int k = 0; k <= depth; ++k) F.lev[k] = make_level(n, rp, ci, F.tree.leaf_of, depth - k, (int64_t)1 << k);
    F.init_leaves(rp, ci, va);
    F.run();
    *out = h.release();
    return 0;
  } catch (const Err &e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception &e) {
    g_err = e.what();
    return -100;
  }
}

void orc_free(OrcHandle *h) { delete h; }

int orc_solve(OrcHandle *h, const double *b, double *x, int nthreads) {
  try {
    h->F.solve(b, x, std::max(1, nthreads));
    return 0;
  } catch (const std::exception &e) {
    g_err = e.what();
    return -100;
  }
}

int orc_ranks(OrcHandle *h, int level, int *ranks) {   // 2^(level-1) entries
  const int64_t nc = (int64_t)1 << (level - 1);
  for (int64_t c = 0; c < nc; ++c) {
    auto it = h->F.rank.find({level, c});
    ranks[c] = it == h->F.rank.end() ? 0 : it->second;
  }
  return 0;
}
// number of stored singular values of node (level, c); copies up to cap
int orc_sigma(OrcHandle *h, int level, int64_t c, double *buf, int cap) {
  auto it = h->F.sigma.find({level, c});
  if (it == h->F.sigma.end()) return 0;
  const int k = (int)it->second.size();
  for (int t = 0; t < std::min(k, cap); ++t) buf[t] = it->second[t];
  return k;
}
int orc_level_order(OrcHandle *h, int level, int64_t *seq, int *wave) {
  const auto &s = h->F.level_order[level];
  for (size_t t = 0; t < s.size(); ++t) {
    seq[t] = s[t];
    wave[t] = h->F.level_wave[level][t];
  }
  return (int)s.size();
}
int orc_node_counts(OrcHandle *h, int level, int *npart, int *nn1) {
  const int64_t nc = (int64_t)1 << (level - 1);
  for (int64_t c = 0; c < nc; ++c) {
    auto a = h->F.npartners.find({level, c});
    auto b = h->F.nn1.find({level, c});
    npart[c] = a == h->F.npartners.end() ? 0 : a->second;
    nn1[c] = b == h->F.nn1.end() ? 0 : b->second;
  }
  return 0;
}
// trace lines joined by '\n'; returns the full length
int64_t orc_trace(OrcHandle *h, char *buf, int64_t cap) {
  std::string s;
  for (auto &t : h->F.trace) s += t + "\n";
  if (buf && cap > 0) {
    const int64_t k = std::min<int64_t>(cap - 1, (int64_t)s.size());
    std::memcpy(buf, s.data(), k);
    buf[k] = 0;
  }
  return (int64_t)s.size();
}
// info[0] max edge distance, [1] waves run in parallel, [2] waves total,
// [3] stored blocks, [4] stored doubles (blocks + pivots)
int orc_info(OrcHandle *h, int64_t *info) {
  info[0] = h->F.max_edge_distance;
  info[1] = h->F.waves_parallel;
  info[2] = h->F.waves_total;
  info[3] = (int64_t)h->F.M.size();
  int64_t d = 0;
  for (auto &kv : h->F.M) d += (int64_t)kv.second->a.size();
  for (auto &kv : h->F.pivots) d += (int64_t)kv.second.a.size();
  info[4] = d;
  return 0;
}

// Frobenius rule (F2): ||all levels below||_F^2 in force at level i (0 if unused)
double orc_frob_d2(OrcHandle *h, int level) {
  auto it = h->F.frob_level.find(level);
  return it == h->F.frob_level.end() ? 0.0 : it->second;
}

// size of node (kind 0 = s, 1 = b, 2 = r; level; cluster)
int orc_size(OrcHandle *h, int kind, int level, int64_t c) { return h->F.sz(mk(kind, level, c)); }

int orc_spmv(int64_t n, const int64_t *rp, const int64_t *ci, const double *va, const double *x, double *y) {
  spmv(Csr{n, rp, ci, va}, x, y);
  return 0;
}

// method 0 = PCG, 1 = GMRES(restart).  out: iters, converged, breakdown; relres
int orc_krylov(OrcHandle *h, int64_t n, const int64_t *rp, const int64_t *ci, const double *va, const double *b,
               double *x, double tol, int method, int restart, int maxit, int nthreads, int *iters, int *converged,
               int *breakdown, double *relres) {
  try {
    Csr A{n, rp, ci, va};
    KrylovOut o = method == 0 ? pcg(A, h->F, std::max(1, nthreads), b, x, tol, maxit)
                              : gmres(A, h->F, std::max(1, nthreads), b, x, tol, restart, maxit);
    *iters = o.iters;
    *converged = o.converged;
    *breakdown = o.breakdown;
    *relres = o.relres;
    return 0;
  } catch (const std::exception &e) {
    g_err = e.what();
    return -100;
  }
}

// Eq. GMRES_residual (P:l.665-669): ||Ã b - Ã A x|| / ||Ã b||
double orc_paper_residual(OrcHandle *h, int64_t n, const int64_t *rp, const int64_t *ci, const double *va,
                          const double *b, const double *x, int nthreads) {
  std::vector<double> ab(n), ax(n), aax(n);
  h->F.solve(b, ab.data(), std::max(1, nthreads));
  spmv(Csr{n, rp, ci, va}, x, ax.data());
  h->F.solve(ax.data(), aax.data(), std::max(1, nthreads));
  double num = 0.0, den = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    num += (ab[i] - aax[i]) * (ab[i] - aax[i]);
    den += ab[i] * ab[i];
  }
  return std::sqrt(num) / std::sqrt(den);
}

// kernel-level pins: right singular values of M (R x m column-major)
int orc_test_svd(const double *Mm, int R, int m, double *sigma, double *V) {
  try {
    std::vector<double> s, v;
    svd_right(Mm, R, m, s, v);
    std::copy(s.begin(), s.end(), sigma);
    std::copy(v.begin(), v.end(), V);
    return 0;
  } catch (const Err &e) {
    g_err = e.what();
    return e.code;
  }
}
// x = A^{-1} b with the oracle's partial-pivot LU (n x n column-major)
int orc_test_lu_solve(const double *A, int n, double *b, int nrhs) {
  try {
    Blk B(n, n);
    std::copy(A, A + (size_t)n * n, B.a.begin());
    LU f;
    lu_factor(B, f);
    lu_solve(f, b, nrhs);
    return 0;
  } catch (const Err &e) {
    g_err = e.what();
    return e.code;
  }
}
// column-pivoted QR: |R_kk| (min(R,m)) and the permutation
int orc_test_qrcp(const double *Mm, int R, int m, double *d, int *perm) {
  std::vector<double> W(Mm, Mm + (size_t)R * m), dd;
  std::vector<int> p;
  qr_colpiv(W, R, m, dd, p);
  std::copy(dd.begin(), dd.end(), d);
  std::copy(p.begin(), p.end(), perm);
  return 0;
}
}
