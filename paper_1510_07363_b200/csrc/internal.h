// Internal structures of liblorasp (not part of the C ABI).
//
// Node ids inside a level i (clusters c = 0..K-1 of P_{i-1}, K = 2^(i-1)):
//   S_c  = c       super-node s_c^[i]            (P:l.224-226)
//   P_c  = K + c   its red parent P(b_c^[i])     (P:l.227)
// The black node b_c^[i] never owns a stored block: its couplings (V, -I and
// the fill of s's elimination) live inside the node's fused pivot record F.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace lorasp {

// A stored block ("slot") holds Mat(col -> row), i.e. rows = equations of the
// row node, cols = variables of the col node (P:l.75, P:l.81).  On the SPD
// path each unordered pair is stored once; the row node is the one
// eliminated first (P nodes count as after every S node of the level; two P
// nodes: the smaller cluster).
struct SymSlot {
  int row, col;
};

// Merge source: level-(i+1) P-P slot copied into a level-i S-S slot
// (MergeRedNodes, P:l.298-304).
struct MergeSrc {
  int dst_slot;      // level-i slot {S_a, S_b}, rows = S_a
  int src_slot;      // level-(i+1) slot
  int dst_qr, dst_qc;  // which child red (0/1) of S_a (rows) / S_b (cols) the source lands in
  int src_cluster_r;   // cluster (of P_i) whose vars index the destination rows
  int src_cluster_c;   // cluster (of P_i) whose vars index the destination cols
  bool trans;          // source stored with rows = src_cluster_c
};

// Slots on the SPD path are unordered pairs (one orientation stored); on the
// general (LU) path every ordered pair u -> v has its own slot Mat(u -> v)
// (rows v, cols u).
struct SymNode {
  bool exists = false;  // structural size > 0
  bool aux = false;     // has well-separated partners -> Compress, b and P(b) exist
  int wave = -1;
  std::vector<int> partners;    // level node ids, sorted (S by cluster, then P)
  std::vector<int> pslot_src;   // SPD: {S_c, p_k} (rows S_c = A_k^T); LU: Mat(p_k -> S_c) (rows S_c = B_k^T)
  std::vector<int> pslot_src2;  // LU: Mat(S_c -> p_k) (rows p_k = A_k)
  std::vector<int> pslot_dst;   // SPD: {P_c, p_k};  LU: Mat(P_c -> p_k) (rows p_k = R_k)
  std::vector<int> pslot_dst2;  // LU: Mat(p_k -> P_c) (rows P_c = Q_k^T)
  std::vector<int> n1;          // uneliminated neighbours at elimination (S/P ids), sorted
  std::vector<int> n1_slot;     // SPD: {S_c, n};  LU: Mat(n -> S_c) (rows S_c: coupling C)
  std::vector<int> n1_slot2;    // LU: Mat(S_c -> n) (rows n: coupling R)
  int self_slot = -1;           // slot {S_c, S_c}
  // T = n1 + [P_c if aux]
  // SPD: tslot[a*(a+1)/2 + b] = slot {T_a, T_b}, b <= a
  // LU:  tslot[a*|T| + b]     = Mat(T_b -> T_a)
  std::vector<int> tslot;
};

struct SymLevel {
  int i = 0, K = 0;
  std::vector<int> order;       // clusters in processing order
  std::vector<int> colour;      // colour of each cluster
  std::vector<int> wave_begin;  // wave w = order[wave_begin[w] .. wave_begin[w+1])
  std::vector<SymNode> node;    // by cluster
  std::vector<SymSlot> slots;
  std::vector<MergeSrc> merge;  // i < depth
  std::vector<char> p_exists;   // P_c has edges (== node[c].aux)
  bool lattice = true;          // lattice colouring accepted (else greedy)
};

struct Plan {
  int64_t n = 0;
  int dim = 0, depth = 0;
  double eps = 0;
  unsigned flags = 0;
  int64_t nnz = 0;
  std::vector<int64_t> row_ptr, col_idx;
  std::vector<int> leaf_of;         // leaf cluster of each dof
  std::vector<int> leaf_pos;        // position inside its leaf cluster
  std::vector<int> leaf_size;       // |C| of each leaf cluster
  std::vector<std::vector<int>> leaf_members;  // ascending
  std::vector<SymLevel> lev;        // lev[i], i = 1..depth
  // leaf scatter: nnz k -> slot of the leaf level, row, col inside it (or slot -1)
  std::vector<int> nnz_slot, nnz_r, nnz_c;
  int max_edge_distance = 0;        // Theorem P:l.515-521 check (must be <= 2)
  int total_waves = 0;
};

// analyze.cpp
int build_plan(Plan &pl, int64_t n, const int64_t *row_ptr, const int64_t *col_idx, int dim,
               const double *coords, int leaf_size, int depth, double eps, unsigned flags,
               std::string &err);

}  // namespace lorasp
