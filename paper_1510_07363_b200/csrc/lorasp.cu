// liblorasp: host orchestration of the level sweep + the C ABI (include/lorasp.h).
//
// factor(): for each level i = l..1 (Alg. 1, P:l.265-289)
//   level start : exact super-node sizes m_c (from the ranks of level i+1),
//                 bound-allocated block slots in a per-level arena, zeroed;
//                 MergeRedNodes (P:l.295-313) = leaf scatter (i = l) or copies
//                 of the level-(i+1) red-red blocks;
//   per colour wave (distance-2 colouring => all nodes of a wave touch
//   disjoint blocks, so the wave is one batch):
//     Compress (P:l.319-394): Gram of the stacked well-separated blocks
//       (k_gemm2) -> symmetric eigen-solver + rank (k_tridiag_reg / k_tridiag_cl
//       + k_eig_t ..., or k_rrqr with LORASP_RRQR) -> ranks (read by the host
//       in the first sweep; predicted and verified afterwards, recorded graph)
//       -> R_k = A_k V written to the new P(b) <-> p_k blocks (k_gemm2);
//     Eliminate s then b (P:l.101-106, l.396-399), fused: gather the pivot
//       K = [[S, V], [V^T, 0]] and coupling C into the node's record F
//       (k_copy), K = L D L^T and L^{-1} (k_pivot_blk / LU: k_pivot_lu_blk),
//       Z = L^{-1} C (k_gemm2), Schur update T_ab -= Z_a^T D Z_b into the target
//       blocks (k_gemm2).
//   The frozen records F = [L^{-1} | Z] are the factor used by apply().
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <dlfcn.h>
#include <nccl.h>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "internal.h"
#include "kernels.cuh"
#include "pivot_warp.cuh"
#include "lorasp.h"

namespace lorasp {

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      throw Err(LORASP_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));      \
    }                                                                                  \
  } while (0)

struct Err {
  int code;
  std::string msg;
  Err(int c, std::string m) : code(c), msg(std::move(m)) {}
};

// Sweep kernels go out with programmatic dependent launch: the next kernel's
// CTAs are scheduled while the current one drains and block in pdl_enter()
// until its memory is visible (hides the ~launch gap between the ~400
// dependent launches of a factorization).  LORASP_NO_PDL: plain launches.
static const bool g_pdl = getenv("LORASP_NO_PDL") == nullptr;
template <typename... KArgs, typename... Args>
static void launch_k(void (*kern)(KArgs...), dim3 grid, unsigned block, size_t smem, cudaStream_t st,
                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

static const int SMEM_LIMIT = 226 * 1024;  // dynamic; leaves room for static smem
static const int EIG_REG_MIN = 3;
static const size_t EIG_REG_SMEM = 200 * 1024;
// generic eigen path: shared memory for d/e/tau/..., A when it fits, and an
// inverse-iteration batch of 16 vectors (5 m doubles + m bytes each)
static int eig_generic_cap(int m) {
  const int64_t mp = (m + 8) & ~7;
  const int64_t base = 6 * mp + std::max(m, 512);
  const int64_t per = 5 * (int64_t)m + (m + 7) / 8;
  const int64_t withA = base + (int64_t)m * m + 16 * per;
  const int64_t lim = SMEM_LIMIT / 8;
  if (withA <= lim) return (int)withA;
  return (int)lim;   // A in global scratch; the rest of the 226 KB serves the batches
}

// growable device buffer; growth synchronises the stream first (no in-flight use)
// bumped by every device (re)allocation: a recorded factorization graph holds
// raw pointers and is only replayed while this is unchanged
static std::atomic<long long> g_alloc_gen{0};   // handles may allocate from several threads
struct CaptureAbort {};

struct DevBuf {
  void *p = nullptr;
  size_t cap = 0;
  const char *tag = "";   // debug name (LORASP_POISON=<tag>|all NaN-fills new allocations)
  void ensure(size_t bytes, cudaStream_t st) {
    if (bytes <= cap) return;
    {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      if (st && cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
        throw CaptureAbort{};   // growth inside a graph capture: record later
    }
    ++g_alloc_gen;
    if (p) {
      // side streams (split pivots, eigen classes) may read any workspace: growth
      // is rare, so wait for the whole device rather than only `st`
      CK(cudaDeviceSynchronize());
      CK(cudaFree(p));
      p = nullptr;
      cap = 0;
    }
    size_t nb = std::max<size_t>(bytes + bytes / 4, 1 << 20);
    if (cudaMalloc(&p, nb) != cudaSuccess) {
      cudaGetLastError();
      throw Err(LORASP_E_OOM, "device allocation of " + std::to_string(nb) + " bytes failed");
    }
    static const char *poison = getenv("LORASP_POISON");   // debug: NaN-fill new buffers
    if (poison && (!strcmp(poison, "all") || (tag[0] && strstr(poison, tag)))) {
      cudaMemset(p, 0xFF, nb);   // legacy stream: completes before any later work on the library's streams
      cudaDeviceSynchronize();
    }
    cap = nb;
  }
  template <class T>
  T *as() const { return reinterpret_cast<T *>(p); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Host -> device upload of a pageable host buffer, ordered on `st` and complete on
// return.  A plain cudaMemcpy from pageable memory goes on the legacy stream and may
// return before its DMA lands; kernels on the library's non-blocking streams are not
// ordered after it (a fresh handle could then read recycled memory).
static void h2d_sync(void *dst, const void *src, size_t bytes, cudaStream_t st) {
  if (!bytes) return;
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));
}

// bump pool of device chunks for the frozen factor records
struct Pool {
  struct Chunk {
    double *p;
    size_t cap;
  };
  std::vector<Chunk> chunks;
  size_t ci = 0, used = 0, total_used = 0;
  double *alloc(size_t nd) {
    nd = (nd + 31) & ~size_t(31);
    while (ci < chunks.size() && used + nd > chunks[ci].cap) {
      ++ci;
      used = 0;
    }
    if (ci == chunks.size()) {
      ++g_alloc_gen;
      size_t cap = std::max<size_t>(nd, size_t(32) << 20);  // >= 256 MB
      double *p = nullptr;
      if (cudaMalloc(&p, cap * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        throw Err(LORASP_E_OOM, "factor pool allocation failed");
      }
      if (getenv("LORASP_POISON") && (!strcmp(getenv("LORASP_POISON"), "all") || strstr(getenv("LORASP_POISON"), "pool")))
      {
        cudaMemset(p, 0xFF, cap * sizeof(double));   // debug: NaN-fill
        cudaDeviceSynchronize();
      }
      chunks.push_back({p, cap});
      used = 0;
    }
    double *r = chunks[ci].p + used;
    used += nd;
    total_used += nd;
    return r;
  }
  void reset() { ci = 0; used = 0; total_used = 0; }
  void release() {
    for (auto &c : chunks) cudaFree(c.p);
    chunks.clear();
    reset();
  }
};

// host-side pinned staging + device mirror for task descriptors
struct Staging {
  char *h = nullptr;
  DevBuf d;
  size_t cap = 0, used = 0;
  void init(size_t bytes, cudaStream_t st) {
    if (h) cudaFreeHost(h);
    CK(cudaMallocHost(&h, bytes));
    cap = bytes;
    d.ensure(bytes, st);
    used = 0;
  }
  // make room for a group of pushes that one launch consumes together
  void reserve(size_t bytes, cudaStream_t st) {
    if (cap_mode) return;
    size_t need = bytes + 4096;
    if (used + need <= cap) return;
    flush(st);
    CK(cudaStreamSynchronize(st));
    sync_side();
    used = 0;
    pend = 0;
    if (need > cap) init(std::max(need, cap * 2), st);
  }
  // Kernels on the side streams (split pivots on stream2, eigen-solver classes)
  // read descriptors from the device ring too: a wrap or reset must wait for
  // them as well as for `st`, else the next H2D copy on `st` overwrites
  // descriptors a pending side-stream kernel has yet to read.
  std::vector<cudaStream_t> side;
  void sync_side() {
    for (cudaStream_t s : side)
      if (s) CK(cudaStreamSynchronize(s));
  }
  // copy `bytes` of src into staging; the H2D copy of everything pushed since
  // the last flush() is one cudaMemcpyAsync (descriptors of a whole wave travel
  // together).  Returns the device pointer.
  size_t pend = 0;   // start of the not-yet-copied range
  // graph capture: descriptors go to `blob` (host) at their final offsets in the
  // persistent device buffer `gd`, copied once after the capture
  bool cap_mode = false, cap_overflow = false;
  std::vector<char> blob;
  char *gd = nullptr;
  size_t gd_cap = 0, total = 0;   // total: bytes pushed by the current factorization
  void *push_deferred(const void *src, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return cap_mode ? (void *)gd : d.p;
    size_t need = (bytes + 255) & ~size_t(255);
    if (cap_mode) {
      const size_t off = blob.size();
      blob.resize(off + need);
      std::memcpy(blob.data() + off, src, bytes);
      if (off + need > gd_cap) {
        cap_overflow = true;
        return gd;
      }
      return gd + off;
    }
    total += need;
    if (used + need > cap) {
      flush(st);
      CK(cudaStreamSynchronize(st));
      sync_side();
      used = 0;
      pend = 0;
      if (need > cap) init(std::max(need, cap * 2), st);
    }
    std::memcpy(h + used, src, bytes);
    void *dp = d.as<char>() + used;
    used += need;
    return dp;
  }
  void flush(cudaStream_t st) {
    if (cap_mode) return;
    if (used > pend) CK(cudaMemcpyAsync(d.as<char>() + pend, h + pend, used - pend, cudaMemcpyHostToDevice, st));
    pend = used;
  }
  void *push(const void *src, size_t bytes, cudaStream_t st) {
    void *dp = push_deferred(src, bytes, st);
    flush(st);
    return dp;
  }
  // Only after a sync of `st`.  Side-stream readers of the ring (eigen classes,
  // split-pivot part 2) are joined into `st` by events before that sync; wraps
  // inside a wave (push_deferred / reserve) still wait for the side streams.
  void reset() {
    if (cap_mode) return;
    used = 0;
    pend = 0;
  }
  void release() {
    if (h) cudaFreeHost(h);
    h = nullptr;
    d.release();
  }
};

// per-kernel-class CUDA-event timing (enabled with lorasp_set_timing)
enum KClass {
  K_SCATTER, K_MERGE, K_GRAM, K_JACOBI, K_PROJECT, K_ASSEMBLE, K_PIVOT, K_ZGEMM, K_SCHUR,
  K_APPLY_FWD, K_APPLY_BWD, K_SPMV, K_DOT, K_VEC, K_NCLASS
};
static const char *KNAME[K_NCLASS] = {"leaf_scatter", "merge_copy", "gram_gemm", "eig_tridiag",
                                      "project_gemm", "assemble_copy", "pivot_chol_inv", "trsm_gemm",
                                      "schur_gemm", "apply_fwd", "apply_bwd", "spmv", "dot", "vec"};
static const char *KKERNEL[K_NCLASS] = {"k_leaf_scatter", "k_copy", "k_gemm2_dmma", "k_eig_warp | k_tridiag_* + k_eig_t", "k_gemm2_dmma", "k_copy",
                                        "k_pivot", "k_gemm2_dmma", "k_gemm2_dmma", "k_apply_fwd_df + k_apply_bwd_df | k_apply_fwd", "k_apply_bwd",
                                        "k_spmv", "k_dot_partial+k_dot_final", "k_axpby/k_sub/k_set_rhs/k_get_x"};
struct KStat {
  double ms = 0, flops = 0, bytes = 0;
  int64_t launches = 0;
};
struct TimedEv {
  int cls;
  cudaEvent_t a, b;
  double flops, bytes;
  int nl;   // kernel launches the event pair brackets
};

struct NodeRec {  // one eliminated (s, b) pair, for apply + stats
  int level, c, m, r, W, ld;
  int64_t zf_off = 0, zb_off = 0, lb_off = 0;
  double *F;
  std::vector<int> T;  // level node ids (S: c', P: K + c')
  std::vector<int> w;  // widths
};

}  // namespace lorasp

using namespace lorasp;

// ranks a rank-predicted sweep logged (device -> pinned host, stream order)
struct RankLog {
  int level;
  size_t pos;
  std::vector<int> comp;
};

struct lorasp_ctx {
  Plan plan;
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string last_error;
  bool factored = false;
  bool mem_ready = false;
  // numeric state
  std::vector<std::vector<int>> msz, rnk;  // [level][cluster]
  std::vector<std::vector<double>> sigma0; // unused placeholder for stats
  DevBuf d_values, d_rowptr, d_colidx, d_dest, arena[2], ws_G, ws_V, ws_sig, ws_X, ws_ctr, ws_piv, d_ranks,
      d_status, d_vec, d_y, d_perm, d_b, d_x, d_kry, d_apnodes, d_apsegs, d_dotpart;
  int *h_ranks = nullptr;
  int *h_status = nullptr;
  double *h_dot = nullptr;
  Pool fpool;
  Staging stg;
  std::vector<NodeRec> recs;
  // apply plan
  std::vector<int> ap_wave_begin;  // in recs order (factor order), per wave
  std::vector<int> ap_part_begin;  // split apply: Z parts of wave w in [ap_part_begin[w], ap_ypart_begin[w])
  std::vector<int> ap_ypart_begin, ap_lpart_begin, ap_part_end;   // then y row slabs, then L column slabs
  std::vector<char> ap_wave_split; // wave uses the split kernels
  // per-wave shared-memory footprint of the fused kernels (waves of small
  // records run many more CTAs per SM than the global worst case allows)
  std::vector<int> ap_wave_ch;
  std::vector<size_t> ap_wave_fsm, ap_wave_bsm;
  DevBuf d_apparts, d_upart;
  bool no_split_apply = getenv("LORASP_NO_SPLIT_APPLY") != nullptr;
  // dataflow apply (single GPU): one persistent launch per direction with
  // per-node dependency counters (k_apply_fwd_df / k_apply_bwd_df); bitwise the
  // wave launches' result (LORASP_NO_DF selects the wave launches, for the tests)
  bool no_df = getenv("LORASP_NO_DF") != nullptr;
  bool ap_df_ok = false;
  DevBuf d_apdf, d_apcontr, d_apdfl, d_zob, d_dfcnt;
  int ap_df_n = 0, ap_df_nt = 0, ap_df_wave = 0, ap_df_ch = 0, ap_df_gf = 0, ap_df_gb = 0;
  size_t ap_df_fsm = 0, ap_df_bsm = 0;
  std::vector<double> ap_wave_flops, ap_wave_bytes;  // per wave, one pass (fwd or bwd)
  size_t ap_fwd_smem = 0, ap_bwd_smem = 0, ap_y_smem = 0;
  int ap_chunk = 0;
  // the forward + backward wave launches of one apply, captured once per
  // factorization (static after it) and replayed as one graph launch
  cudaGraphExec_t ap_graph = nullptr;
  // split pivot (SPD): chol(S) + L11^{-1} of the wave's super-nodes on a second
  // stream, overlapped with the compress (whose rank sync follows)
  cudaStream_t stream2 = nullptr;     // least priority: fills SMs the sweep leaves idle
  cudaStream_t stream_hi = nullptr;   // greatest priority: the factorization itself
  cudaEvent_t ev_s0 = nullptr, ev_s1 = nullptr, ev_u = nullptr;
  cudaStream_t stream_eig = nullptr;   // register-tile eigen path beside the cluster / generic one
  cudaEvent_t ev_ef = nullptr, ev_ej = nullptr;
  cudaStream_t stream_cl[3] = {nullptr, nullptr, nullptr};   // tridiagonalisation classes 2, 3, 4
  cudaEvent_t ev_cf = nullptr, ev_cj[3] = {nullptr, nullptr, nullptr};
  bool s1_pending = false;
  DevBuf ws_S, ws_Y, ws_T1, d_sp, ws_piv2;   // ws_piv2: blocked split-pivot part 1 (stream2)
  DevBuf d_frob, d_frobpart;   // f2: ||all levels below||_F^2 (device scalar) and per-slot partial sums
  void *h_sp = nullptr;     // pinned upload of the part-1 copy + pivot task lists
  size_t h_sp_cap = 0;
  bool no_split = getenv("LORASP_NO_SPLIT") != nullptr;
  // rank-predicted schedule: after a factorization, its ranks predict the
  // next one's (same pattern); the host then builds and enqueues every wave
  // without the per-wave rank synchronisation, the device ranks are logged
  // and verified at the end, and a mismatch re-runs the synchronised sweep
  std::vector<std::vector<int>> rank_cache;
  bool cache_valid = false, replay_used = false;
  int replay_hits = 0, replay_misses = 0;
  int64_t split_nodes = 0;   // fused pivots factored by the split path (last factorization)
  bool no_replay = getenv("LORASP_NO_REPLAY") != nullptr;
  int *h_ranklog = nullptr;
  size_t ranklog_cap = 0;
  std::vector<int64_t> ap_graph_sig;   // launch parameters the graph was captured with
  bool no_graph = getenv("LORASP_NO_GRAPH") != nullptr;
  int64_t vec_len = 0;
  bool dest_ready = false;
  std::vector<int64_t> leaf_soff;  // leaf-level slot offsets used for d_dest
  // stats
  double flops_model = 0, t_factor_ms = 0, t_host_ms = 0, t_sync_ms = 0;
  int64_t launches_factor = 0, launches_apply = 0, launches_krylov = 0;
  int64_t f_doubles = 0;
  bool debug = getenv("LORASP_DEBUG") != nullptr;
  // LU path: partial pivoting inside the fused pivots (k_pivot_lu, pivot = 1),
  // switched on (for the rest of the handle's life) when the no-pivot kernels
  // report LORASP_NEED_PIVOT; SPD path: a failed signed Cholesky re-plans the
  // handle on the general LU path (reading Z12)
  bool lu_pivot = false;
  int lu_pivot_switches = 0, spd_fallbacks = 0;
  std::string spd_fallback_node;
  std::vector<double> an_coords;   // analyze inputs kept for a re-plan
  int an_dim = 0, an_leaf = 0;
  // kernel timing
  bool timing = false;
  unsigned timing_mask = 0;
  std::vector<cudaEvent_t> evpool;
  std::vector<TimedEv> pend;
  KStat kst[K_NCLASS];
  // distributed factorization (lorasp_set_dist): subtree owner-computes with
  // per-wave exchanges through the caller's collective callback
  int dist_rank = 0, dist_world = 1, dist_l0 = 0;
  lorasp_coll_fn dist_fn = nullptr;
  void *dist_user = nullptr;
  void *dist_send = nullptr, *dist_recv = nullptr;
  int64_t dist_send_cap = 0, dist_recv_cap = 0;
  int64_t dist_bytes = 0, dist_calls = 0;
  int64_t dist_apply_bytes = 0, dist_apply_calls = 0;   // vector exchanges of the distributed apply
  // distributed apply (records stay on their owner): per wave, the number of
  // owned nodes (ordered first in the wave's ApNode range) and, per rank, the
  // vector segments its nodes write: forward = the target RHS segments,
  // backward = the nodes' own Var segments (offsets into d_vec, lengths)
  std::vector<int> ap_wave_nown;
  std::vector<std::vector<std::vector<std::pair<int64_t, int64_t>>>> ap_dirty_f, ap_dirty_b;
  // library-owned NCCL communicator (lorasp_set_dist_nccl): the transport of the
  // per-wave collectives instead of the caller's callback
  ncclComm_t nccl = nullptr;
  DevBuf nccl_send, nccl_recv;
  // neighbour push: per level, per slot, the ranks that read or update it later
  // (owners of the nodes whose plan references it, and -- through MergeRedNodes --
  // every reader of the next level's slot it lands in); bytes moved per (src, dst)
  // pair of the current all-to-all-v exchange
  std::vector<std::vector<uint32_t>> slot_readers;
  std::vector<int64_t> a2a_counts;   // world x world, bytes, [src * world + dst]
  int piv_maxn_hint = 0;   // batch-independent pivot path choice (max n of the whole wave)
  int piv_cnt_hint = 0;    // ... and its node count (distributed: every rank's nodes)
  // recorded factorization: a verified rank-predicted sweep captured once as a
  // CUDA graph (descriptors resident in fg_desc) and replayed while the ranks,
  // the allocations and the timing mask stay the same
  cudaGraphExec_t fgraph = nullptr;
  DevBuf fg_desc;
  long long fg_gen = -1;
  unsigned fg_timing = 0;
  std::vector<TimedEv> fg_pend;
  std::vector<RankLog> fg_rlog;
  int64_t fg_fdoubles = 0;
  bool no_fgraph = getenv("LORASP_NO_FGRAPH") != nullptr;
  bool fgraph_used = false;
  int fg_captures = 0, fg_failures = 0;
  int64_t fg_launches = 0;
  int eig_clmax_hint = 0, eig_bigmax_hint = 0, eig_regmax_hint = 0;   // the same for the eigen-solver classes
  int eig_reg_wave_n = 0;   // distributed: register-tile eigen tasks of the whole wave
  int eig_all_wave_n = 0;   // distributed: eigen tasks of the whole wave
  int eig_cl_wave_n[5] = {0, 0, 0, 0, 0};   // distributed: cluster-class eigen tasks of the whole wave
};

namespace {

inline dim3 grid1(int64_t n, int bs = 256) {
  int64_t g = (n + bs - 1) / bs;
  return dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16)));
}

int tbeg_force(lorasp_ctx *h, int cls);
int tbeg(lorasp_ctx *h, int cls) {
  if (!h->timing || !((h->timing_mask >> cls) & 1u)) return -1;
  return tbeg_force(h, cls);
}
int tbeg_force(lorasp_ctx *h, int cls) {
  size_t need = 2 * (h->pend.size() + 1);
  while (h->evpool.size() < need) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    h->evpool.push_back(e);
  }
  TimedEv t{cls, h->evpool[need - 2], h->evpool[need - 1], 0, 0, 1};
  if (h->stg.cap_mode) CK(cudaEventRecordWithFlags(t.a, h->stream, cudaEventRecordExternal));
  else CK(cudaEventRecord(t.a, h->stream));
  h->pend.push_back(t);
  return (int)h->pend.size() - 1;
}
void tend(lorasp_ctx *h, int idx, double flops, double bytes) {
  if (idx < 0) return;
  if (h->stg.cap_mode) CK(cudaEventRecordWithFlags(h->pend[idx].b, h->stream, cudaEventRecordExternal));
  else CK(cudaEventRecord(h->pend[idx].b, h->stream));
  h->pend[idx].flops = flops;
  h->pend[idx].bytes = bytes;
}
// after a stream sync: fold the recorded launches into the per-class totals
void tflush(lorasp_ctx *h) {
  for (const TimedEv &t : h->pend) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, t.a, t.b));
    KStat &k = h->kst[t.cls];
    k.ms += ms;
    k.flops += t.flops;
    k.bytes += t.bytes;
    k.launches += t.nl;
  }
  h->pend.clear();
}

bool is_device_ptr(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Cluster eigen path (128 < m <= 512): k_tridiag_cl over a CTA cluster, then
// k_eig_t<false, true> (eigenvalues, inverse iteration, back-transformation).
static int eig_cl_class(int m) {
  if (m > EIG_REG_M && m <= 160) return 4;   // one CTA: k_tridiag_reg<5, 16, 10> (5 x 10 tile per thread)
  if (m > EIG_REG_M && m <= 256) return 1;
  if (m > 256 && m <= 384) return 2;
  if (m > 384 && m <= 512) return 3;
  return 0;
}

// clusters of this shape that can be co-resident on the device (GPC-limited:
// at most one 16-CTA cluster per GPC), queried once per shape
template <int QR, int UC, int CL>
static int tridiag_cl_fit() {
  static int fit = -1;
  if (fit < 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = (size_t)21 * 32 * QR * 8;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, k_tridiag_cl<QR, UC, CL>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      nc = 0;
    }
    fit = nc;
    if (getenv("LORASP_DEBUG")) fprintf(stderr, "[lorasp] k_tridiag_cl<%d, %d, %d>: %d co-resident clusters\n", QR, UC, CL, nc);
  }
  return fit;
}

template <int QR, int UC, int CL>
static void launch_tridiag_cl_t(cudaStream_t st, const EigTask *dt, int n, double eps, long long *prof) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n * CL));
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = (size_t)21 * 32 * QR * 8;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k_tridiag_cl<QR, UC, CL>, dt, eps, prof));
}

// Cluster width per wave: the per-step latency falls with fewer columns per
// warp (UC), so a wave whose nodes all fit on the device at once takes the
// widest cluster that still fits (16 / 8 / 4 CTAs); wider waves keep the
// narrower cluster (or, m <= 160, the one-CTA register-tile kernel).  wave_n:
// the class's nodes in the whole wave, so that distributed ranks pick the
// single-GPU shape.
static void launch_tridiag_cl(cudaStream_t st, const EigTask *dt, int n, int cls, double eps,
                              long long *prof = nullptr, int wave_n = 0) {
  if (wave_n <= 0) wave_n = n;
  if (cls == 4) {   // 128 < m <= 160
    if (wave_n <= tridiag_cl_fit<5, 2, 8>()) launch_tridiag_cl_t<5, 2, 8>(st, dt, n, eps, prof);
    else   // the register-tile tridiagonalisation in one CTA (the record format is shared)
      launch_k(k_tridiag_reg<false, 5, 16, 10>, (unsigned)n, 512, 0, st, dt, eps, (long long *)nullptr);
    return;
  }
  if (cls == 1) {
    if (wave_n <= tridiag_cl_fit<8, 2, 8>()) launch_tridiag_cl_t<8, 2, 8>(st, dt, n, eps, prof);
    else launch_tridiag_cl_t<8, 4, 4>(st, dt, n, eps, prof);
  } else if (cls == 2) {
    if (wave_n <= tridiag_cl_fit<12, 2, 16>()) launch_tridiag_cl_t<12, 2, 16>(st, dt, n, eps, prof);
    else launch_tridiag_cl_t<12, 3, 8>(st, dt, n, eps, prof);
  } else {
    launch_tridiag_cl_t<16, 2, 16>(st, dt, n, eps, prof);
  }
}

// Register-tile eigen path for m <= 128: tridiagonalisation (tile class c:
// 32 / 64 / 128 rows) then k_eig_t<true>.
// wave_n: register-tile tasks in the whole wave (all ranks), which decides the
// launch shape so that a distributed sweep runs the single-GPU kernels
static int launch_eig_reg(cudaStream_t st, EigTask *ds, int n, int c, double eps, int *dstatus, int wave_n) {
  if (c == 0) launch_k(k_tridiag_reg<false, 1, 4, 8>, (unsigned)n, 128, 0, st, ds, eps, (long long *)nullptr);
  else if (c == 1) launch_k(k_tridiag_reg<false, 2, 8, 8>, (unsigned)n, 256, 0, st, ds, eps, (long long *)nullptr);
  else launch_k(k_tridiag_reg<false>, (unsigned)n, EIG_REG_THREADS, 0, st, ds, eps, (long long *)nullptr);
  CK(cudaGetLastError());
  // waves of many nodes (several per SM) with m in (64, 128]: the one-CTA
  // k_eig_t keeps a whole SM for one node through phases that use a fraction of
  // it (lambda_0 in one warp, one thread per inverse-iteration vector); the
  // throughput pipeline runs many nodes per SM instead: eigenvalues (128
  // threads, 2 lanes per eigenvalue), rank + inverse iteration (one warp per 8
  // vectors), MGS + back-transformation (256 threads per node)
  if (c == 2 && wave_n > 148 && eps > 0.0) {
    const int mp = (128 + 8) & ~7;
    launch_k(k_eigvals_cl, (unsigned)n, 128, (size_t)3 * mp * 8, st, (const EigTask *)ds, eps, 1, 2);
    const int64_t per = 5 * (int64_t)128 + (128 + 7) / 8;
    const int cap = (int)(2 * mp + 8 * per);
    launch_k(k_invit_multi, (unsigned)(n * 16), 32, (size_t)cap * 8, st, (const EigTask *)ds, 16, cap, eps);
    launch_k(k_orthbt, (unsigned)n, 256, ORTHBT_SMEM, st, (const EigTask *)ds);
    CK(cudaGetLastError());
    return 4;
  }
  // waves wider than the GPU are throughput bound: for m <= 64 half the shared
  // memory (still room for ~30 inverse-iteration vectors per batch) lets two
  // CTAs share an SM
  // (m <= 128 keeps 16 warps: r may exceed 64 = 8 vectors per warp x 8 warps;
  // the 8-warp form would need the rank before the launch, which only the
  // rank-predicted sweep has, and the two schedules must agree bit for bit)
  const bool narrow = wave_n > 148 && c <= 1;
  const size_t esm = narrow ? (c <= 1 ? EIG_REG_SMEM / 2 : (size_t)110 * 1024) : EIG_REG_SMEM;
  const int eth = (c == 2 && !narrow) ? EIG_REG_THREADS : 256;
  launch_k(k_eig_t<true>, (unsigned)n, eth, esm, st, ds, eps, (int)(esm / 8), dstatus);
  CK(cudaGetLastError());
  return 2;
}

// After k_tridiag_cl: eigenvalues + rank (k_eig_t<false, true>), chunked
// inverse iteration, MGS, chunked back-transformation.  Returns the launches.
static int launch_pre_post(cudaStream_t st, EigTask *dp, int n, int mmax, double eps, int *dstatus,
                           cudaEvent_t *pev = nullptr) {
  if (eps == 0.0) {   // V = I, r = m (reading Z3)
    launch_k(k_eig_t<false, true>, (unsigned)n, EIG_REG_THREADS, SMEM_LIMIT, st, dp, eps, SMEM_LIMIT / 8, dstatus);
    CK(cudaGetLastError());
    return 1;
  }
  // eigenvalues over several CTAs per node (about 40 candidates each)
  const int nev = std::max(1, std::min(16, (mmax + 39) / 40));
  launch_k(k_eigvals_cl, (unsigned)(n * nev), 512, (size_t)3 * ((mmax + 8) & ~7) * 8, st, (const EigTask *)dp, eps,
           nev, 32);
  CK(cudaGetLastError());
  const int cap = SMEM_LIMIT / 8;
  const int64_t per = 5 * (int64_t)mmax + (mmax + 7) / 8;
  const int mp = (mmax + 8) & ~7;
  const int nb = (int)std::min<int64_t>(256, (cap - 2 * mp) / per);
  const int nch = (mmax + nb - 1) / nb;
  if (pev) cudaEventRecord(pev[0], st);
  launch_k(k_invit_multi, (unsigned)(n * nch), 256, SMEM_LIMIT, st, dp, nch, cap, eps);
  CK(cudaGetLastError());
  if (pev) cudaEventRecord(pev[1], st);
  {
    // block Gram-Schmidt over a cluster: CTA c owns <= 32 vectors (two per warp)
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(512);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (mmax <= 256) {
      cfg.gridDim = dim3((unsigned)(n * 8));
      at[0].val.clusterDim.x = 8;
      cfg.dynamicSmemBytes = (size_t)orth_bgs_smem_doubles<8>() * 8;
      CK(cudaLaunchKernelEx(&cfg, k_orth_bgs<8, 8>, (const EigTask *)dp));
    } else if (mmax <= 384) {
      cfg.gridDim = dim3((unsigned)(n * 16));
      at[0].val.clusterDim.x = 16;
      cfg.dynamicSmemBytes = (size_t)orth_bgs_smem_doubles<12>() * 8;
      CK(cudaLaunchKernelEx(&cfg, k_orth_bgs<12, 16>, (const EigTask *)dp));
    } else {
      cfg.gridDim = dim3((unsigned)(n * 16));
      at[0].val.clusterDim.x = 16;
      cfg.dynamicSmemBytes = (size_t)orth_bgs_smem_doubles<16>() * 8;
      CK(cudaLaunchKernelEx(&cfg, k_orth_bgs<16, 16>, (const EigTask *)dp));
    }
  }
  CK(cudaGetLastError());
  if (pev) cudaEventRecord(pev[2], st);
  // few nodes (the upper levels): 16 vectors per CTA, the reflector chain is
  // latency-bound and the SMs are idle; many nodes: more vectors per CTA
  if (n * ((mmax + 15) / 16) <= 2 * 148) {
    const int nc = (mmax + 15) / 16;
    if (mmax <= 256) launch_k(k_backtr_multi<8, 1>, (unsigned)(n * nc), 512, SMEM_LIMIT, st, dp, nc, cap);
    else if (mmax <= 384) launch_k(k_backtr_multi<12, 1>, (unsigned)(n * nc), 512, SMEM_LIMIT, st, dp, nc, cap);
    else launch_k(k_backtr_multi<16, 1>, (unsigned)(n * nc), 512, SMEM_LIMIT, st, dp, nc, cap);
  } else if (mmax <= 256) {
    const int nc = (mmax + 63) / 64;
    launch_k(k_backtr_multi<8, 4>, (unsigned)(n * nc), 512, SMEM_LIMIT, st, dp, nc, cap);
  } else if (mmax <= 384) {
    const int nc = (mmax + 47) / 48;
    launch_k(k_backtr_multi<12, 3>, (unsigned)(n * nc), 512, SMEM_LIMIT, st, dp, nc, cap);
  } else {
    const int nc = (mmax + 31) / 32;
    launch_k(k_backtr_multi<16, 2>, (unsigned)(n * nc), 512, SMEM_LIMIT, st, dp, nc, cap);
  }
  CK(cudaGetLastError());
  return 4;
}

static void set_eig_attrs() {
  CK(cudaFuncSetAttribute(k_invit_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
  CK(cudaFuncSetAttribute(k_orth_bgs<8, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, orth_bgs_smem_doubles<8>() * 8));
  CK(cudaFuncSetAttribute(k_orth_bgs<12, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, orth_bgs_smem_doubles<12>() * 8));
  CK(cudaFuncSetAttribute(k_orth_bgs<16, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, orth_bgs_smem_doubles<16>() * 8));
  CK(cudaFuncSetAttribute(k_orth_bgs<12, 16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(k_orth_bgs<16, 16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(k_backtr_multi<8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
  CK(cudaFuncSetAttribute(k_backtr_multi<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
  CK(cudaFuncSetAttribute(k_backtr_multi<12, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
  CK(cudaFuncSetAttribute(k_backtr_multi<16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
  CK(cudaFuncSetAttribute(k_backtr_multi<12, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
  CK(cudaFuncSetAttribute(k_backtr_multi<16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
  CK(cudaFuncSetAttribute(k_eig_t<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)EIG_REG_SMEM));
  CK(cudaFuncSetAttribute(k_eig_warp<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)(EIGW_SMEM_DOUBLES * sizeof(double))));
  CK(cudaFuncSetAttribute(k_eig_warp<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)(EIGW_SMEM_DOUBLES * sizeof(double))));
  CK(cudaFuncSetAttribute(k_eig_warp<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)(EIGW_SMEM_DOUBLES * sizeof(double))));
  CK(cudaFuncSetAttribute(k_eig_t<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
  CK(cudaFuncSetAttribute(k_eig_t<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
  CK(cudaFuncSetAttribute(k_tridiag_cl<8, 4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 21 * 32 * 8 * 8));
  CK(cudaFuncSetAttribute(k_tridiag_cl<12, 3, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 21 * 32 * 12 * 8));
  CK(cudaFuncSetAttribute(k_tridiag_cl<16, 2, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 21 * 32 * 16 * 8));
  CK(cudaFuncSetAttribute(k_tridiag_cl<16, 2, 16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(k_tridiag_cl<8, 2, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 21 * 32 * 8 * 8));
  CK(cudaFuncSetAttribute(k_tridiag_cl<12, 2, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 21 * 32 * 12 * 8));
  CK(cudaFuncSetAttribute(k_tridiag_cl<12, 2, 16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(k_tridiag_cl<5, 2, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 21 * 32 * 5 * 8));

}

void ensure_mem(lorasp_ctx *h) {
  {
    struct {
      DevBuf *b;
      const char *t;
    } tg[] = {{&h->arena[0], "arena"}, {&h->arena[1], "arena"}, {&h->ws_G, "ws_G"}, {&h->ws_V, "ws_V"},
              {&h->ws_sig, "ws_sig"}, {&h->ws_X, "ws_X"}, {&h->ws_ctr, "ws_ctr"}, {&h->ws_piv, "ws_piv"},
              {&h->ws_S, "ws_S"}, {&h->ws_Y, "ws_Y"}, {&h->ws_T1, "ws_T1"}, {&h->ws_piv2, "ws_piv2"}, {&h->d_ranks, "d_ranks"},
              {&h->d_vec, "d_vec"}, {&h->d_y, "d_y"}, {&h->d_kry, "d_kry"}, {&h->fg_desc, "fg_desc"}};
    for (auto &x : tg) x.b->tag = x.t;
  }
  if (h->mem_ready) return;
  CK(cudaSetDevice(h->device));
  const Plan &pl = h->plan;
  h->d_rowptr.ensure((pl.n + 1) * sizeof(int64_t), h->stream);
  h->d_colidx.ensure(std::max<int64_t>(1, pl.nnz) * sizeof(int64_t), h->stream);
  h2d_sync(h->d_rowptr.p, pl.row_ptr.data(), (pl.n + 1) * sizeof(int64_t), h->stream);
  h2d_sync(h->d_colidx.p, pl.col_idx.data(), pl.nnz * sizeof(int64_t), h->stream);
  h->d_values.ensure(std::max<int64_t>(1, pl.nnz) * sizeof(double), h->stream);
  h->d_status.ensure(64, h->stream);
  CK(cudaMallocHost(&h->h_ranks, sizeof(int) * (1 << 20)));
  CK(cudaMallocHost(&h->h_status, 64));
  CK(cudaMallocHost(&h->h_dot, 1024 * sizeof(double)));   // GMRES Hessenberg column (restart <= 1000)
  h->d_dotpart.ensure((DOT_BLOCKS + 1024) * sizeof(double), h->stream);
  h->stg.init(size_t(64) << 20, h->stream);
  set_eig_attrs();
  {
    int least = 0, greatest = 0;
    CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    CK(cudaStreamCreateWithPriority(&h->stream2, cudaStreamNonBlocking, least));
    CK(cudaStreamCreateWithPriority(&h->stream_hi, cudaStreamNonBlocking, greatest));
    CK(cudaStreamCreateWithPriority(&h->stream_eig, cudaStreamNonBlocking, greatest));
    for (auto &cs : h->stream_cl) CK(cudaStreamCreateWithPriority(&cs, cudaStreamNonBlocking, greatest));
    h->stg.side = {h->stream2, h->stream_hi, h->stream_eig, h->stream_cl[0], h->stream_cl[1], h->stream_cl[2]};
  }
  CK(cudaEventCreateWithFlags(&h->ev_cf, cudaEventDisableTiming));
  for (auto &e : h->ev_cj) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&h->ev_ef, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&h->ev_ej, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&h->ev_u, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&h->ev_s0, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&h->ev_s1, cudaEventDisableTiming));
  CK(cudaFuncSetAttribute(k_pivot, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
  CK(cudaFuncSetAttribute(k_pivot_lu, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
  CK(cudaFuncSetAttribute(k_pivot_blk, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
  CK(cudaFuncSetAttribute(k_pivot_lu_blk, cudaFuncAttributeMaxDynamicSharedMemorySize, 216 * 1024));
  CK(cudaFuncSetAttribute(k_apply_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
  CK(cudaFuncSetAttribute(k_apply_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
  CK(cudaFuncSetAttribute(k_apply_fwd_y, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
  CK(cudaFuncSetAttribute(k_apply_fwd_df, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
  CK(cudaFuncSetAttribute(k_orthbt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ORTHBT_SMEM));
  CK(cudaFuncSetAttribute(k_apply_bwd_df, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
  CK(cudaFuncSetAttribute(k_apply_fwd_z, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
  CK(cudaFuncSetAttribute(k_apply_bwd_z, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
  CK(cudaFuncSetAttribute(k_apply_bwd_l, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
  h->mem_ready = true;
}

template <class T>
T *push(lorasp_ctx *h, const std::vector<T> &v) {
  return reinterpret_cast<T *>(h->stg.push(v.data(), v.size() * sizeof(T), h->stream));
}
template <class T>
T *pushd(lorasp_ctx *h, const std::vector<T> &v) {   // deferred: copied at the next flush
  return reinterpret_cast<T *>(h->stg.push_deferred(v.data(), v.size() * sizeof(T), h->stream));
}
template <class T>
size_t vbytes(const std::vector<T> &v) {
  return ((v.size() * sizeof(T) + 255) & ~size_t(255)) + 256;
}

// launch on descriptors already staged (pushd + flush)
void launch_gemm_dev(lorasp_ctx *h, const GemmTask *dt, const GemmSeg *ds, size_t ntasks, int cls, double flops,
                     double bytes) {
  if (ntasks == 0) return;
  int ev = cls >= 0 ? tbeg(h, cls) : -1;
  launch_k(k_gemm2_dmma, (unsigned)ntasks, 128, 0, h->stream, dt, ds);   // DMMA beats DFMA on every shape
  tend(h, ev, flops, bytes);
  ++h->launches_factor;
  CK(cudaGetLastError());
}
void launch_copy_dev(lorasp_ctx *h, const CopyTask *dt, const std::vector<CopyTask> &tasks, int cls) {
  if (tasks.empty()) return;
  double bytes = 0;
  for (const CopyTask &t : tasks) bytes += (t.mode == 0 ? 16.0 : 8.0) * t.rows * t.cols;
  int ev = cls >= 0 ? tbeg(h, cls) : -1;
  launch_k(k_copy, (unsigned)tasks.size(), 256, 0, h->stream, dt);
  tend(h, ev, 0, bytes);
  ++h->launches_factor;
  CK(cudaGetLastError());
}

void launch_gemm(lorasp_ctx *h, const std::vector<GemmTask> &tasks, const std::vector<GemmSeg> &segs,
                 int cls, double flops, double bytes) {
  if (tasks.empty()) return;
  h->stg.reserve(segs.size() * sizeof(GemmSeg) + tasks.size() * sizeof(GemmTask), h->stream);
  GemmSeg *ds = push(h, segs);
  GemmTask *dt = push(h, tasks);
  int ev = cls >= 0 ? tbeg(h, cls) : -1;
  launch_k(k_gemm2_dmma, (unsigned)tasks.size(), 128, 0, h->stream, dt, ds);
  tend(h, ev, flops, bytes);
  ++h->launches_factor;
  CK(cudaGetLastError());
}

// eigen tasks: m <= 128 -> register-tile kernel (512 threads), else the generic one
// eigen tasks: 64 < m <= 128 -> register-tile kernel (512 threads); otherwise
// the generic shared/global-memory kernel (faster for small m, measured with
// tools/eig_cmp.py)


void launch_eig(lorasp_ctx *h, const std::vector<EigTask> &et, EigTask *de, int max_m, int cap) {
  if (h->plan.flags & LORASP_RRQR) {   // f1: pivoted QR compressor, one launch for the wave
    if (et.empty()) return;
    for (const EigTask &e : et)
      if (e.m > RRQR_MAXM) throw Err(LORASP_E_ARG, "LORASP_RRQR: node of size " + std::to_string(e.m) + " > 512");
    // one launch for the wave (classes would run back to back): 128 threads
    // when every node has m <= 64 (cheaper barriers), else 512 (16 warps share
    // the Gram-Schmidt coefficients of larger ranks)
    int mm = 0;
    for (const EigTask &e : et) mm = std::max(mm, e.m);
    if (mm <= 64)
      launch_k(k_rrqr<128>, (unsigned)et.size(), 128, 0, h->stream, (const EigTask *)de, h->plan.eps,
               h->d_status.as<int>());
    else
      launch_k(k_rrqr<512>, (unsigned)et.size(), 512, 0, h->stream, (const EigTask *)de, h->plan.eps,
               h->d_status.as<int>());
    ++h->launches_factor;
    CK(cudaGetLastError());
    return;
  }
  {   // every stack of the wave has m <= 32: one warp per node (k_eig_warp)
    int mm = 0;
    for (const EigTask &e : et) mm = std::max(mm, e.m);
    if (h->eig_regmax_hint > 0) mm = std::max(mm, h->eig_regmax_hint);
    if (!et.empty() && mm <= EIGW_M) {
      // waves of up to 4 nodes per SM: 4 warps per node share the eigenvalue
      // phase (measured: 4 lanes per eigenvalue beat 8 at m = 24 / 32); wider
      // waves: one warp per node (throughput).  The whole wave decides
      // (distributed).
      const int nwave = h->eig_all_wave_n > 0 ? h->eig_all_wave_n : (int)et.size();
      const size_t smem = EIGW_SMEM_DOUBLES * sizeof(double);
      if (nwave <= 4 * 148)
        launch_k(k_eig_warp<4>, (unsigned)et.size(), 128, smem, h->stream, (const EigTask *)de, h->plan.eps,
                 h->d_status.as<int>());
      else
        launch_k(k_eig_warp<1>, (unsigned)et.size(), 32, smem, h->stream, (const EigTask *)de, h->plan.eps,
                 h->d_status.as<int>());
      ++h->launches_factor;
      CK(cudaGetLastError());
      return;
    }
  }
  std::vector<EigTask> small, big, clt[5];
  bool reg_fork = false;
  for (const EigTask &e : et) {
    const int cls = eig_cl_class(e.m);
    if (e.m >= EIG_REG_MIN && e.m <= EIG_REG_M) small.push_back(e);
    else if (cls) clt[cls].push_back(e);
    else big.push_back(e);
  }
  const bool single = (small.size() == et.size()) || (big.size() == et.size());
  if (!small.empty()) {
    // register-tile path, by tile class (32 / 64 / 128 rows); the whole 200 KB
    // of shared memory serves A + the inverse-iteration batches
    // one launch pair at the largest tile class of the wave: the classes would
    // otherwise run one after the other, each a full chain of latency-bound steps
    std::vector<EigTask> rc[3];
    int cmax = 0;
    for (auto &e : small) cmax = std::max(cmax, e.m <= 32 ? 0 : (e.m <= 64 ? 1 : 2));
    if (h->eig_regmax_hint > 0) cmax = std::max(cmax, h->eig_regmax_hint <= 32 ? 0 : (h->eig_regmax_hint <= 64 ? 1 : 2));
    rc[cmax] = small;
    EigTask *ds[3] = {nullptr, nullptr, nullptr};
    for (int c = 0; c < 3; ++c)
      if (!rc[c].empty()) ds[c] = (single && rc[c].size() == et.size()) ? de : push(h, rc[c]);
    // with cluster / generic tasks in the same wave the register-tile pair runs
    // on its own stream beside them (few nodes per class: the SMs are idle)
    reg_fork = !single;
    cudaStream_t rs = h->stream;
    if (reg_fork) {
      CK(cudaEventRecord(h->ev_ef, h->stream));
      CK(cudaStreamWaitEvent(h->stream_eig, h->ev_ef, 0));
      rs = h->stream_eig;
    }
    for (int c = 0; c < 3; ++c)
      if (ds[c])
        h->launches_factor += launch_eig_reg(rs, ds[c], (int)rc[c].size(), c, h->plan.eps, h->d_status.as<int>(),
                                             h->eig_reg_wave_n > 0 ? h->eig_reg_wave_n : (int)small.size());
    if (reg_fork) CK(cudaEventRecord(h->ev_ej, h->stream_eig));
  }
  std::vector<EigTask> post;
  {
    // the tridiagonalisation classes side by side (classes 2, 3, 4 on their own streams)
    EigTask *dc[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    int ncls = 0;
    for (int c = 1; c <= 4; ++c)
      if (!clt[c].empty()) {
        dc[c] = push(h, clt[c]);
        ++ncls;
      }
    const bool fork = ncls > 1;
    if (fork) CK(cudaEventRecord(h->ev_cf, h->stream));
    for (int c = 1; c <= 4; ++c) {
      if (!dc[c]) continue;
      cudaStream_t cs = h->stream;
      if (fork && c > 1) {
        cs = h->stream_cl[c - 2];
        CK(cudaStreamWaitEvent(cs, h->ev_cf, 0));
      }
      launch_tridiag_cl(cs, dc[c], (int)clt[c].size(), c, h->plan.eps, nullptr,
                        h->eig_cl_wave_n[c] > 0 ? h->eig_cl_wave_n[c] : (int)clt[c].size());
      ++h->launches_factor;
      if (cs != h->stream) {
        CK(cudaEventRecord(h->ev_cj[c - 2], cs));
        CK(cudaStreamWaitEvent(h->stream, h->ev_cj[c - 2], 0));
      }
      post.insert(post.end(), clt[c].begin(), clt[c].end());
    }
  }
  if (!post.empty()) {
    EigTask *dp = push(h, post);
    int mmax = h->eig_clmax_hint;
    for (auto &e : post) mmax = std::max(mmax, e.m);
    h->launches_factor += launch_pre_post(h->stream, dp, (int)post.size(), mmax, h->plan.eps, h->d_status.as<int>());
  }
  if (!big.empty()) {
    EigTask *db = single ? de : push(h, big);
    int mb = h->eig_bigmax_hint;
    for (auto &e : big) mb = std::max(mb, e.m);
    launch_k(k_eig_t<false>, (unsigned)big.size(), EIG_THREADS, (size_t)eig_generic_cap(mb) * 8, h->stream, 
        db, h->plan.eps, eig_generic_cap(mb), h->d_status.as<int>());
    ++h->launches_factor;
    CK(cudaGetLastError());
  }
  if (reg_fork) CK(cudaStreamWaitEvent(h->stream, h->ev_ej, 0));
  (void)max_m;
  (void)cap;
}

// One k_copy CTA moves one task; a large block (a whole n x n pivot inverse,
// a big super-node block) as one task ran on a single SM at a few GB/s.  Tasks
// above COPY_CTA_ELEMS elements are cut into rectangles of at most that many
// (whole-column runs; rows split only for very tall columns).  Tasks never
// overlap in their writes, so the pieces may run in any order.  The diagonal
// fill (mode 2) is cut into column runs with their own diagonal rows.
static const int64_t COPY_CTA_ELEMS = 16384;
void split_copies(std::vector<CopyTask> &tasks) {
  bool any = false;
  for (const CopyTask &t : tasks)
    if ((int64_t)t.rows * t.cols > COPY_CTA_ELEMS) any = true;
  if (!any) return;
  std::vector<CopyTask> out;
  out.reserve(tasks.size() * 2);
  for (const CopyTask &t : tasks) {
    if ((int64_t)t.rows * t.cols <= COPY_CTA_ELEMS || t.rows <= 0 || t.cols <= 0 || t.mode == 2) {
      out.push_back(t);
      continue;
    }
    const int rb = (int)std::min<int64_t>(t.rows, 4096);
    const int cb = (int)std::max<int64_t>(1, COPY_CTA_ELEMS / rb);
    for (int c0 = 0; c0 < t.cols; c0 += cb)
      for (int r0 = 0; r0 < t.rows; r0 += rb) {
        CopyTask p = t;
        p.rows = std::min(rb, t.rows - r0);
        p.cols = std::min(cb, t.cols - c0);
        p.dst = t.dst + r0 + (int64_t)c0 * t.ldd;
        if (t.mode == 0)   // trans: dst(i, j) = src(j, i)
          p.src = t.trans ? t.src + c0 + (int64_t)r0 * t.lds : t.src + r0 + (int64_t)c0 * t.lds;
        out.push_back(p);
      }
  }
  tasks.swap(out);
}

void launch_copy(lorasp_ctx *h, std::vector<CopyTask> tasks, int cls) {
  if (tasks.empty()) return;
  split_copies(tasks);
  CopyTask *dt = push(h, tasks);
  double bytes = 0;
  for (const CopyTask &t : tasks) bytes += (t.mode == 0 ? 16.0 : 8.0) * t.rows * t.cols;
  int ev = cls >= 0 ? tbeg(h, cls) : -1;
  launch_k(k_copy, (unsigned)tasks.size(), 256, 0, h->stream, dt);
  tend(h, ev, 0, bytes);
  ++h->launches_factor;
  CK(cudaGetLastError());
}

// tile a logical M x N product into 64x64 tasks
void add_tiles(std::vector<GemmTask> &tasks, GemmTask base, int kmax_by_row = 0) {
  (void)kmax_by_row;
  if (base.N <= 32) {   // narrow product (e.g. R_k = A_k^T V with r <= 32)
    for (int tm = 0; tm < base.M; tm += GT) {
      GemmTask t = base;
      t.tm = tm;
      t.tn = 0;
      t.tnw = 32;
      tasks.push_back(t);
    }
    return;
  }
  for (int tn = 0; tn < base.N; tn += GT)
    for (int tm = 0; tm < base.M; tm += GT) {
      GemmTask t = base;
      t.tm = tm;
      t.tn = tn;
      tasks.push_back(t);
    }
}

double node_flops(int m, int r, int R, int W, bool sym) {
  // SURVEY §8(d) algorithmic work: compress + fused elimination; R is the stack
  // height (doubled on the LU path by the B_k), the [x2] terms double for LU.
  // Here W already includes the r columns of P(b).
  const double x2 = sym ? 1.0 : 2.0;
  double f = 0;
  if (R > 0) f += (double)R * m * m + 9.0 * m * m * (double)m + 2.0 * R * m * (double)r;
  f += x2 * (((double)m * m * m + (double)r * r * r) / 3.0 + ((double)m * m + (double)r * r) * W +
             (double)(m + r) * W * W);
  return f;
}

// Blocked path for fused SPD pivots with n = m + r > PIV_SMALL_N (right-looking
// signed Cholesky in 64-column panels, then blocked forward substitution for
// L^{-1} in a scratch X, copied back over the pivot).  The whole launch
// sequence is planned on the host first, with every descriptor in one blob, so
// that it can run on the main stream (descriptors through the staging ring) or
// on stream2 beside the compress (split pivot, part 1; its own upload).
// Scratch per node: X (n x n) | S (n x 64) | T (np x 64 x 64) | Wt (64 x 64).
struct BlockedPlan {
  struct Step {
    int kind;            // 0: k_pivot_blk on 64 x 64 diagonal blocks, 1: k_copy, 2: k_gemm2_dmma
    size_t off, n;       // descriptors (PivTask / CopyTask / GemmTask) in the blob
    size_t soff;         // GemmSeg array (kind 2)
  };
  std::vector<char> blob;
  std::vector<Step> steps;
  int64_t ws_doubles = 0;
  template <class T>
  size_t add(const std::vector<T> &v) {
    const size_t off = blob.size();
    blob.resize(off + ((v.size() * sizeof(T) + 255) & ~size_t(255)));
    if (!v.empty()) std::memcpy(blob.data() + off, v.data(), v.size() * sizeof(T));
    return off;
  }
};

static int64_t blocked_ws_doubles_one(int n) {
  return (int64_t)n * n + (int64_t)n * 64 + (int64_t)((n + 63) / 64) * 4096 + 4096;
}
static size_t blocked_ws_bytes(const std::vector<PivTask> &big) {
  int64_t tot = 0;
  for (const PivTask &t : big) tot += blocked_ws_doubles_one(t.m + t.r);
  return (size_t)tot * 8 + 256;
}

void build_blocked_plan(const std::vector<PivTask> &big, double *wb, BlockedPlan &plan) {
  std::vector<int64_t> off(big.size());
  int64_t tot = 0;
  int np_max = 0;
  for (size_t q = 0; q < big.size(); ++q) {
    const int n = big[q].m + big[q].r;
    off[q] = tot;
    tot += blocked_ws_doubles_one(n);
    np_max = std::max(np_max, (n + 63) / 64);
  }
  plan.ws_doubles = tot;
  auto Xp = [&](size_t q) { return wb + off[q]; };
  auto Sp = [&](size_t q) { const int n = big[q].m + big[q].r; return wb + off[q] + (int64_t)n * n; };
  auto Tp = [&](size_t q) { const int n = big[q].m + big[q].r; return wb + off[q] + (int64_t)n * n + (int64_t)n * 64; };
  auto Wp = [&](size_t q) {
    const int n = big[q].m + big[q].r;
    return wb + off[q] + (int64_t)n * n + (int64_t)n * 64 + (int64_t)((n + 63) / 64) * 4096;
  };
  auto step_copy = [&](std::vector<CopyTask> &ct) {
    split_copies(ct);
    if (!ct.empty()) plan.steps.push_back({1, plan.add(ct), ct.size(), 0});
  };
  auto step_gemm = [&](const std::vector<GemmTask> &g, const std::vector<GemmSeg> &sg) {
    if (g.empty()) return;
    const size_t so = plan.add(sg);
    plan.steps.push_back({2, plan.add(g), g.size(), so});
  };
  for (int p = 0; p < np_max; ++p) {
    std::vector<PivTask> dt;
    std::vector<CopyTask> ct;
    std::vector<GemmTask> g1, g2;
    std::vector<GemmSeg> s1, s2;
    for (size_t q = 0; q < big.size(); ++q) {
      const PivTask &t = big[q];
      const int n = t.m + t.r, j0 = 64 * p;
      if (j0 >= n) continue;
      const int b = std::min(64, n - j0), j1 = j0 + b, rest = n - j1;
      {   // diagonal block: k_pivot_blk on the b x b block (local signs: m - j0 plus)
        const int ml = std::max(0, std::min(b, t.m - j0));
        PivTask d{t.F + j0 + (int64_t)j0 * t.ld, t.ld, ml, b - ml, t.node};
        d.Xo = Xp(q) + j0 + (int64_t)j0 * n;
        d.ldxo = n;
        d.Wt = Wp(q);
        dt.push_back(d);
      }
      if (rest == 0) continue;
      CopyTask c{};
      c.src = t.F + j1 + (int64_t)j0 * t.ld;
      c.lds = t.ld;
      c.dst = Sp(q);
      c.ldd = n;
      c.rows = rest;
      c.cols = b;
      c.mode = 0;
      c.alpha = 1.0;
      ct.push_back(c);
      // L21 = S Wt
      GemmTask g{};
      g.C = t.F + j1 + (int64_t)j0 * t.ld;
      g.ldc = t.ld;
      g.M = rest;
      g.N = b;
      g.beta = 0;
      g.seg0 = (int)s1.size();
      g.nseg = 1;
      s1.push_back(GemmSeg{Sp(q), Wp(q), n, 64, b, 1.0});
      add_tiles(g1, g);
      // K22 -= L21 D1 L21^T (lower tiles)
      const int spos = std::max(0, std::min(b, t.m - j0));
      const double *L21 = t.F + j1 + (int64_t)j0 * t.ld;
      GemmTask u{};
      u.C = t.F + j1 + (int64_t)j1 * t.ld;
      u.ldc = t.ld;
      u.M = rest;
      u.N = rest;
      u.tb = 1;
      u.beta = 1;
      u.seg0 = (int)s2.size();
      if (spos > 0) s2.push_back(GemmSeg{L21, L21, t.ld, t.ld, spos, -1.0});
      if (spos < b) s2.push_back(GemmSeg{L21 + (int64_t)spos * t.ld, L21 + (int64_t)spos * t.ld, t.ld, t.ld,
                                         b - spos, 1.0});
      u.nseg = (int)s2.size() - u.seg0;
      for (int tn = 0; tn < rest; tn += GT)
        for (int tm = tn; tm < rest; tm += GT) {
          GemmTask x = u;
          x.tm = tm;
          x.tn = tn;
          g2.push_back(x);
        }
    }
    if (!dt.empty()) plan.steps.push_back({0, plan.add(dt), dt.size(), 0});
    step_copy(ct);
    step_gemm(g1, s1);
    step_gemm(g2, s2);
  }
  // blocked inversion: X_ip = -X_ii * sum_{k=p}^{i-1} L_ik X_kp
  for (int i = 1; i < np_max; ++i) {
    std::vector<GemmTask> g1, g2;
    std::vector<GemmSeg> s1, s2;
    for (size_t q = 0; q < big.size(); ++q) {
      const PivTask &t = big[q];
      const int n = t.m + t.r, i0 = 64 * i;
      if (i0 >= n) continue;
      const int bi = std::min(64, n - i0);
      for (int p = 0; p < i; ++p) {
        const int p0 = 64 * p, bp = 64;
        GemmTask g{};
        g.C = Tp(q) + (int64_t)p * 4096;   // T_ip: bi x 64, ld 64, slot p
        g.ldc = 64;
        g.M = bi;
        g.N = bp;
        g.beta = 0;
        g.seg0 = (int)s1.size();
        g.nseg = 1;
        s1.push_back(GemmSeg{t.F + i0 + (int64_t)p0 * t.ld, Xp(q) + p0 + (int64_t)p0 * n, t.ld, n, i0 - p0, 1.0});
        add_tiles(g1, g);
        GemmTask x{};
        x.C = Xp(q) + i0 + (int64_t)p0 * n;
        x.ldc = n;
        x.M = bi;
        x.N = bp;
        x.beta = 0;
        x.seg0 = (int)s2.size();
        x.nseg = 1;
        s2.push_back(GemmSeg{Xp(q) + i0 + (int64_t)i0 * n, Tp(q) + (int64_t)p * 4096, n, 64, bi, -1.0});
        add_tiles(g2, x);
      }
    }
    step_gemm(g1, s1);
    step_gemm(g2, s2);
  }
  std::vector<CopyTask> ct;
  for (size_t q = 0; q < big.size(); ++q) {
    const PivTask &t = big[q];
    const int n = t.m + t.r;
    CopyTask c{};
    c.src = Xp(q);
    c.lds = n;
    c.dst = t.F;
    c.ldd = t.ld;
    c.rows = n;
    c.cols = n;
    c.mode = 0;
    c.alpha = 1.0;
    ct.push_back(c);
  }
  step_copy(ct);
}

// The plan's scratch is zeroed first (the upper blocks of X stay zero).
void run_blocked_plan(lorasp_ctx *h, const BlockedPlan &plan, const char *dbase, double *ws, cudaStream_t st) {
  CK(cudaMemsetAsync(ws, 0, plan.ws_doubles * 8, st));
  for (const BlockedPlan::Step &s : plan.steps) {
    if (s.kind == 0)
      launch_k(k_pivot_blk, (unsigned)s.n, 512, pivb_smem_bytes(64), st, (const PivTask *)(dbase + s.off),
               h->d_status.as<int>());
    else if (s.kind == 1)
      launch_k(k_copy, (unsigned)s.n, 256, 0, st, (const CopyTask *)(dbase + s.off));
    else
      launch_k(k_gemm2_dmma, (unsigned)s.n, 128, 0, st, (const GemmTask *)(dbase + s.off),
               (const GemmSeg *)(dbase + s.soff));
    ++h->launches_factor;
    CK(cudaGetLastError());
  }
}

// Fused pivots of one wave: nodes whose pivot fits one CTA's shared memory go
// through k_pivot_blk; larger ones through the blocked path (k_pivot_blk on the
// 64 x 64 diagonal blocks + k_gemm2_dmma).
static const int PIV_SMALL_N = 160;

void pivots(lorasp_ctx *h, const std::vector<PivTask> &pv, double f_piv, double b_piv) {
  cudaStream_t st = h->stream;
  std::vector<PivTask> small, big;
  int max_n = 0;
  for (const PivTask &t : pv) {
    const int n = t.m + t.r;
    if (n <= PIV_SMALL_N) {
      small.push_back(t);
      max_n = std::max(max_n, n);
    } else {
      big.push_back(t);
    }
  }
  if (!small.empty() && h->piv_maxn_hint > max_n) max_n = std::min(h->piv_maxn_hint, PIV_SMALL_N);
  int ev = tbeg(h, K_PIVOT);
  if (!small.empty()) {
    PivTask *dp = push(h, small);
    // one warp per node when the wave is wide (throughput: several nodes per SM);
    // a few nodes run faster on the block kernel (measured per node: ~40-55 us for
    // the warp kernel vs ~22 us for k_pivot_blk at n = 32)
    const bool wide = (h->piv_cnt_hint > 0 ? (size_t)h->piv_cnt_hint : small.size()) > 2 * 148;
    if (max_n <= PIVW_MAXN && wide) {
      constexpr int W = PivW<1>::WARPS;
      launch_k(k_pivot_warp<1>, (unsigned)((small.size() + W - 1) / W), 32 * W, PivW<1>::SMEM, st, (const PivTask *)dp,
               (int)small.size(), h->d_status.as<int>());
    } else if (max_n <= PIVB_MAXN) {
      const size_t sm = pivb_smem_bytes(max_n);
      launch_k(k_pivot_blk, (unsigned)small.size(), 512, sm, st, dp, h->d_status.as<int>());
    } else {
      int64_t want = (int64_t)max_n * max_n + max_n;
      int cap = (int)std::min<int64_t>(want, SMEM_LIMIT / 8);
      cap = std::max(cap, max_n);
      launch_k(k_pivot, (unsigned)small.size(), 512, cap * 8, st, dp, cap, h->d_status.as<int>());
    }
    ++h->launches_factor;
    CK(cudaGetLastError());
  }
  if (!big.empty()) {
    h->ws_piv.ensure(blocked_ws_bytes(big), st);
    BlockedPlan plan;
    build_blocked_plan(big, h->ws_piv.as<double>(), plan);
    h->stg.reserve(plan.blob.size() + 256, st);
    const char *dbase = static_cast<const char *>(h->stg.push(plan.blob.data(), plan.blob.size(), st));
    run_blocked_plan(h, plan, dbase, h->ws_piv.as<double>(), st);
  }
  tend(h, ev, f_piv, b_piv);
}

// LU path: fused pivots by no-pivot LU (k_pivot_lu: shared memory when the
// n x n pivot fits, else in place in global memory), L^{-1} and U^{-T} written
// to the first two record regions.
void pivots_lu(lorasp_ctx *h, const std::vector<PivTask> &pv, double f_piv, double b_piv) {
  if (pv.empty()) return;
  int max_n = 0;
  for (const PivTask &t : pv) max_n = std::max(max_n, t.m + t.r);
  max_n = std::max(max_n, h->piv_maxn_hint);
  std::vector<PivTask> pvp;
  if (h->lu_pivot) {   // partial pivoting (k_pivot_lu only)
    pvp = pv;
    for (PivTask &t : pvp) t.pivot = 1;
  }
  PivTask *dp = push(h, h->lu_pivot ? pvp : pv);
  int ev = tbeg(h, K_PIVOT);
  const bool wide = (h->piv_cnt_hint > 0 ? (size_t)h->piv_cnt_hint : pv.size()) > 2 * 148;
  if (max_n <= PIVW_MAXN && !h->lu_pivot && wide) {   // one warp per node (wide waves)
    constexpr int W = PivW<1>::WARPS;
    launch_k(k_pivot_lu_warp<1>, (unsigned)((pv.size() + W - 1) / W), 32 * W, PivW<1>::SMEM, h->stream,
             (const PivTask *)dp, (int)pv.size(), h->d_status.as<int>());
  } else if (max_n <= PIVLU_MAXN && !h->lu_pivot) {
    const size_t sm = pivb_smem_bytes(max_n);
    launch_k(k_pivot_lu_blk, (unsigned)pv.size(), 512, sm, h->stream, dp, h->d_status.as<int>());
  } else {
    int64_t want = (int64_t)max_n * max_n + 2 * max_n;
    int cap = (int)std::min<int64_t>(want, SMEM_LIMIT / 8);
    cap = std::max(cap, 2 * max_n);
    if (h->lu_pivot && want > cap && 18 * (int64_t)max_n > cap)
      throw Err(LORASP_E_ARG, "pivot block of order " + std::to_string(max_n) + " too large for partial pivoting");
    launch_k(k_pivot_lu, (unsigned)pv.size(), 512, cap * 8, h->stream, dp, cap, h->d_status.as<int>());
  }
  tend(h, ev, f_piv, b_piv);
  ++h->launches_factor;
  CK(cudaGetLastError());
}

// ---- distributed factorization (include/lorasp.h) --------------
int dist_owner_of(int level, int c, int l0) {
  const int sh = level - 1 - l0;
  return sh >= 0 ? (c >> sh) : 0;
}

// NCCL entry points, resolved at run time: the libnccl.so.2 already in the
// process (e.g. torch's) when there is one, else the system's.  Link-time
// binding would risk two different libnccl builds in one process.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
};
static const NcclApi *nccl_api() {
  static NcclApi api;
  static bool tried = false;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (tried) return api.CommInitRank ? &api : nullptr;
  tried = true;
  void *lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) return nullptr;
  api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(lib, "ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))dlsym(lib, "ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))dlsym(lib, "ncclCommDestroy");
  api.AllGather = (decltype(api.AllGather))dlsym(lib, "ncclAllGather");
  api.AllReduce = (decltype(api.AllReduce))dlsym(lib, "ncclAllReduce");
  api.GetErrorString = (decltype(api.GetErrorString))dlsym(lib, "ncclGetErrorString");
  api.Send = (decltype(api.Send))dlsym(lib, "ncclSend");
  api.Recv = (decltype(api.Recv))dlsym(lib, "ncclRecv");
  api.GroupStart = (decltype(api.GroupStart))dlsym(lib, "ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))dlsym(lib, "ncclGroupEnd");
  if (!api.GetUniqueId || !api.CommInitRank || !api.CommDestroy || !api.AllGather || !api.AllReduce || !api.Send ||
      !api.Recv || !api.GroupStart || !api.GroupEnd) {
    api.CommInitRank = nullptr;
    return nullptr;
  }
  return &api;
}
#define NCK(x)                                                                                    \
  do {                                                                                            \
    ncclResult_t r_ = (x);                                                                        \
    if (r_ != ncclSuccess)                                                                        \
      throw Err(LORASP_E_NCCL, std::string("NCCL: ") +                                            \
                                   (nccl_api() && nccl_api()->GetErrorString ? nccl_api()->GetErrorString(r_) \
                                                                             : "error"));       \
  } while (0)

void dist_call(lorasp_ctx *h, int kind, int64_t nbytes) {
  ++h->dist_calls;
  if (h->nccl) {   // library-owned communicator, on the library stream
    const NcclApi *api = nccl_api();
    if (kind == LORASP_COLL_RESERVE) {
      h->nccl_send.ensure(nbytes, h->stream);
      h->nccl_recv.ensure(nbytes * h->dist_world, h->stream);
      h->dist_send = h->nccl_send.p;
      h->dist_recv = h->nccl_recv.p;
      h->dist_send_cap = (int64_t)h->nccl_send.cap;
      h->dist_recv_cap = (int64_t)h->nccl_recv.cap;
    } else if (kind == LORASP_COLL_ALLGATHER) {
      NCK(api->AllGather(h->dist_send, h->dist_recv, (size_t)nbytes, ncclUint8, h->nccl, h->stream));
      CK(cudaStreamSynchronize(h->stream));
    } else if (kind == LORASP_COLL_ALLTOALLV) {   // grouped point-to-point: only the neighbours' blocks
      const int G = h->dist_world, me = h->dist_rank;
      const int64_t *cn = h->a2a_counts.data();
      int64_t so = 0, ro = 0;
      NCK(api->GroupStart());
      for (int p = 0; p < G; ++p) {
        if (cn[me * G + p] > 0 && p != me)
          NCK(api->Send(static_cast<char *>(h->dist_send) + so, (size_t)cn[me * G + p], ncclUint8, p, h->nccl,
                        h->stream));
        if (cn[p * G + me] > 0 && p != me)
          NCK(api->Recv(static_cast<char *>(h->dist_recv) + ro, (size_t)cn[p * G + me], ncclUint8, p, h->nccl,
                        h->stream));
        so += cn[me * G + p];
        ro += cn[p * G + me];
      }
      NCK(api->GroupEnd());
      CK(cudaStreamSynchronize(h->stream));
    } else {
      NCK(api->AllReduce(h->dist_send, h->dist_send, (size_t)nbytes / 4, ncclInt32, ncclMax, h->nccl, h->stream));
      CK(cudaStreamSynchronize(h->stream));
    }
    return;
  }
  if (h->dist_fn(h->dist_user, kind, nbytes) != 0)
    throw Err(LORASP_E_CUDA, "distributed exchange callback failed (kind " + std::to_string(kind) + ")");
}

void dist_reserve(lorasp_ctx *h, int64_t nbytes) {
  if (h->dist_send_cap >= nbytes && h->dist_recv_cap >= nbytes * h->dist_world) return;
  dist_call(h, LORASP_COLL_RESERVE, nbytes);
  if (h->dist_send_cap < nbytes || h->dist_recv_cap < nbytes * h->dist_world)
    throw Err(LORASP_E_ARG, "distributed exchange buffers too small after the reserve callback");
}

// max over ranks of n device ints (non-owned entries are 0) and of the status
// pair; results to host_out[0..n) and h->h_status[0..2)
void dist_allmax_ints(lorasp_ctx *h, const int *dev, size_t n, int *host_out) {
  const int64_t nbytes = (int64_t)(n + 2) * sizeof(int);
  dist_reserve(h, nbytes);
  int *sb = static_cast<int *>(h->dist_send);
  if (n) CK(cudaMemcpyAsync(sb, dev, n * sizeof(int), cudaMemcpyDeviceToDevice, h->stream));
  CK(cudaMemcpyAsync(sb + n, h->d_status.p, 2 * sizeof(int), cudaMemcpyDeviceToDevice, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  // status codes are negative: the max over ranks of -code keeps any failure
  {
    int stv[2];
    CK(cudaMemcpy(stv, sb + n, 2 * sizeof(int), cudaMemcpyDeviceToHost));
    stv[0] = -stv[0];
    CK(cudaMemcpy(sb + n, stv, 2 * sizeof(int), cudaMemcpyHostToDevice));
  }
  dist_call(h, LORASP_COLL_MAXINT, nbytes);
  std::vector<int> tmp(n + 2);
  CK(cudaMemcpy(tmp.data(), sb, nbytes, cudaMemcpyDeviceToHost));
  for (size_t q = 0; q < n; ++q) host_out[q] = tmp[q];
  h->h_status[0] = -tmp[n];
  h->h_status[1] = tmp[n + 1];
}

// contiguous n-double copy as k_copy tasks of <= 2048 x 16 doubles
void contig_copies(std::vector<CopyTask> &ct, const double *src, double *dst, int64_t n) {
  while (n > 0) {
    CopyTask t{};
    t.mode = 0;
    t.alpha = 1.0;
    t.src = src;
    t.dst = dst;
    int64_t take;
    if (n >= 2048) {
      t.rows = 2048;
      t.cols = (int)std::min<int64_t>(16, n / 2048);
      take = (int64_t)t.rows * t.cols;
    } else {
      t.rows = (int)n;
      t.cols = 1;
      take = n;
    }
    t.lds = t.ldd = t.rows;
    ct.push_back(t);
    src += take;
    dst += take;
    n -= take;
  }
}

using DirtyList = std::vector<std::pair<double *, int64_t>>;

// end of a colour wave: every rank's written regions (lists in the same order
// on every rank) travel in one all-gather and are copied into the store
void dist_exchange(lorasp_ctx *h, const std::vector<DirtyList> &dirty) {
  const int G = h->dist_world, me = h->dist_rank;
  int64_t mx = 0;
  for (int g = 0; g < G; ++g) {
    int64_t t = 0;
    for (auto &pr : dirty[g]) t += pr.second;
    mx = std::max(mx, t);
  }
  if (mx == 0) return;
  const int64_t nbytes = mx * 8;
  dist_reserve(h, nbytes);
  std::vector<CopyTask> ct;
  double *send = static_cast<double *>(h->dist_send);
  int64_t off = 0;
  for (auto &pr : dirty[me]) {
    contig_copies(ct, pr.first, send + off, pr.second);
    off += pr.second;
  }
  launch_copy(h, ct, -1);
  CK(cudaStreamSynchronize(h->stream));
  dist_call(h, LORASP_COLL_ALLGATHER, nbytes);
  h->dist_bytes += nbytes;
  ct.clear();
  const double *recv = static_cast<const double *>(h->dist_recv);
  for (int g = 0; g < G; ++g) {
    if (g == me) continue;
    off = 0;
    for (auto &pr : dirty[g]) {
      contig_copies(ct, recv + (int64_t)g * mx + off, pr.first, pr.second);
      off += pr.second;
    }
  }
  launch_copy(h, ct, -1);
}



// per level, per slot: bit mask of the ranks that reference the slot later (see
// lorasp_ctx::slot_readers), from the top level down (a slot merged into the
// next level inherits that slot's readers)
void build_slot_readers(lorasp_ctx *h) {
  const Plan &pl = h->plan;
  h->slot_readers.assign(pl.depth + 1, {});
  for (int i = 1; i <= pl.depth; ++i) {
    const SymLevel &lv = pl.lev[i];
    std::vector<uint32_t> &mk = h->slot_readers[i];
    mk.assign(lv.slots.size(), 0u);
    for (int c = 0; c < lv.K; ++c) {
      const SymNode &nd = lv.node[c];
      if (!nd.exists) continue;
      const uint32_t bit = 1u << dist_owner_of(i, c, h->dist_l0);
      auto add = [&](const std::vector<int> &v) {
        for (int sl : v)
          if (sl >= 0) mk[sl] |= bit;
      };
      if (nd.self_slot >= 0) mk[nd.self_slot] |= bit;
      add(nd.n1_slot);
      add(nd.n1_slot2);
      add(nd.pslot_src);
      add(nd.pslot_src2);
      add(nd.pslot_dst);
      add(nd.pslot_dst2);
      add(nd.tslot);
    }
    if (i > 1)   // MergeRedNodes into level i-1 (lev[i-1].merge: sources are level-i slots)
      for (const MergeSrc &ms : pl.lev[i - 1].merge) mk[ms.src_slot] |= h->slot_readers[i - 1][ms.dst_slot];
  }
}

// end of a colour wave (neighbour push): block k written by rank q goes only to
// the ranks in its reader mask; one all-to-all-v (grouped NCCL send / recv)
void dist_push(lorasp_ctx *h, const std::vector<std::vector<std::pair<double *, int64_t>>> &wr,
               const std::vector<uint32_t> &masks, const std::vector<int> &writer) {
  const int G = h->dist_world, me = h->dist_rank;
  // lists[q][p]: blocks q sends to p, in one order every rank derives
  std::vector<std::vector<DirtyList>> lists(G, std::vector<DirtyList>(G));
  for (size_t k = 0; k < wr.size(); ++k) {
    const int q = writer[k];
    for (int p = 0; p < G; ++p)
      if (p != q && ((masks[k] >> p) & 1u))
        for (auto &pr : wr[k]) lists[q][p].push_back(pr);
  }
  h->a2a_counts.assign((size_t)G * G, 0);
  int64_t out = 0, in = 0;
  for (int q = 0; q < G; ++q)
    for (int p = 0; p < G; ++p) {
      int64_t t = 0;
      for (auto &pr : lists[q][p]) t += pr.second;
      h->a2a_counts[(size_t)q * G + p] = 8 * t;
      if (q == me) out += 8 * t;
      if (p == me) in += 8 * t;
    }
  int64_t any = 0;
  for (int64_t c : h->a2a_counts) any += c;
  if (!any) return;
  dist_reserve(h, std::max(out, in));
  std::vector<CopyTask> ct;
  double *send = static_cast<double *>(h->dist_send);
  int64_t off = 0;
  for (int p = 0; p < G; ++p)
    for (auto &pr : lists[me][p]) {
      contig_copies(ct, pr.first, send + off, pr.second);
      off += pr.second;
    }
  launch_copy(h, ct, -1);
  CK(cudaStreamSynchronize(h->stream));
  dist_call(h, LORASP_COLL_ALLTOALLV, std::max(out, in));
  h->dist_bytes += out;
  ct.clear();
  const double *recv = static_cast<const double *>(h->dist_recv);
  off = 0;
  for (int q = 0; q < G; ++q)
    for (auto &pr : lists[q][me]) {
      contig_copies(ct, recv + off, pr.first, pr.second);
      off += pr.second;
    }
  launch_copy(h, ct, -1);
}

void copy_values(lorasp_ctx *h, const double *values) {
  const size_t nb = h->plan.nnz * sizeof(double);
  CK(cudaMemcpyAsync(h->d_values.p, values, nb, is_device_ptr(values) ? cudaMemcpyDeviceToDevice
                                                                       : cudaMemcpyHostToDevice, h->stream));
}

// after the sweep's final synchronisation: the ranks a rank-predicted sweep
// logged against the prediction it was built with
bool replay_check(lorasp_ctx *h, const std::vector<RankLog> &rlog) {
  for (const RankLog &rl : rlog)
    for (size_t q = 0; q < rl.comp.size(); ++q)
      if (h->h_ranklog[rl.pos + q] != h->rank_cache[rl.level][rl.comp[q]]) {
        ++h->replay_misses;
        return false;
      }
  ++h->replay_hits;
  return true;
}

void status_check(lorasp_ctx *h) {
  if (h->h_status[0] == LORASP_NEED_PIVOT)
    throw Err(LORASP_NEED_PIVOT, "LU without pivoting unstable at node " + std::to_string(h->h_status[1]));
  if (h->h_status[0] != 0)
    throw Err(h->h_status[0], std::string(h->h_status[0] == LORASP_E_EIG_NOCONV
                                              ? "Jacobi eigen-solver did not converge"
                                              : "singular pivot (signed Cholesky failed)") +
                                  " at node " + std::to_string(h->h_status[1]));
}

// Returns false only in replay mode when the predicted ranks were wrong (the
// caller then re-runs with replay = false).
bool factor_impl(lorasp_ctx *h, const double *values, bool replay, bool capture = false) {
  ensure_mem(h);
  const Plan &pl = h->plan;
  cudaStream_t st = h->stream;
  const int L = pl.depth;
  const bool sym = (pl.flags & LORASP_SPD) != 0;
  const bool dist = h->dist_world > 1 && (h->dist_fn || h->nccl);
  if (dist && replay) return false;
  h->dist_bytes = 0;
  h->dist_calls = 0;
  h->piv_maxn_hint = 0;
  h->piv_cnt_hint = 0;
  h->launches_factor = 0;
  h->split_nodes = 0;
  h->flops_model = 0;
  h->t_host_ms = 0;
  h->t_sync_ms = 0;
  h->factored = false;
  // values -> device (a capture's caller copies them before the capture)
  if (!capture) copy_values(h, values);
  CK(cudaMemsetAsync(h->d_status.p, 0, 64, st));
  if (dist && h->slot_readers.size() != (size_t)L + 1) build_slot_readers(h);
  if (pl.flags & LORASP_FROBENIUS) {
    h->d_frob.ensure(64, st);
    CK(cudaMemsetAsync(h->d_frob.p, 0, 8, st));
  }
  h->fpool.reset();
  h->recs.clear();
  h->msz.assign(L + 2, {});
  h->rnk.assign(L + 2, {});
  std::vector<int64_t> prev_soff;
  std::vector<int> prev_sld;
  if (!capture) {
    h->stg.reset();
    h->stg.total = 0;
    CK(cudaStreamSynchronize(st));
  } else {
    h->s1_pending = false;   // the previous sweep's stream2 work is complete (caller synchronised)
  }
  std::vector<RankLog> rlog;
  size_t rlog_pos = 0;
  if (replay) {
    size_t need = 0;
    for (int i = 1; i <= L; ++i) need += (size_t)pl.lev[i].K;
    if (h->ranklog_cap < need) {
      if (h->h_ranklog) CK(cudaFreeHost(h->h_ranklog));
      CK(cudaMallocHost(&h->h_ranklog, std::max<size_t>(need, 64) * sizeof(int)));
      h->ranklog_cap = std::max<size_t>(need, 64);
    }
  }

  for (int i = L; i >= 1; --i) {
    const SymLevel &lv = pl.lev[i];
    const int K = lv.K;
    std::vector<int> &m = h->msz[i];
    std::vector<int> &r = h->rnk[i];
    m.assign(K, 0);
    r.assign(K, 0);
    for (int c = 0; c < K; ++c)
      m[c] = (i == L) ? pl.leaf_size[2 * c] + pl.leaf_size[2 * c + 1]
                      : h->rnk[i + 1][2 * c] + h->rnk[i + 1][2 * c + 1];
    auto bound = [&](int id) { return id < K ? m[id] : (lv.node[id - K].aux ? m[id - K] : 0); };
    auto size = [&](int id) { return id < K ? m[id] : r[id - K]; };
    // slot layout (bound sizes; P-node ranks are not known yet)
    std::vector<int64_t> soff(lv.slots.size()), slen(lv.slots.size());
    std::vector<int> sld(lv.slots.size());
    int64_t tot = 0;
    for (size_t s = 0; s < lv.slots.size(); ++s) {
      int rows = bound(lv.slots[s].row), cols = bound(lv.slots[s].col);
      sld[s] = std::max(1, rows);
      soff[s] = tot;
      slen[s] = (int64_t)rows * cols;
      tot += ((int64_t)rows * cols + 31) & ~int64_t(31);
    }
    DevBuf &ar = h->arena[i & 1];
    ar.ensure(std::max<int64_t>(tot, 32) * sizeof(double), st);
    CK(cudaMemsetAsync(ar.p, 0, tot * sizeof(double), st));
    double *base = ar.as<double>();
    auto slot_ptr = [&](int s) { return base + soff[s]; };
    // distributed mode: the owner of each node of this level (include/lorasp.h)
    if (dist && K != (1 << (i - 1)))
      throw Err(LORASP_E_ARG, "distributed factorization needs 2^(i-1) clusters at level i");
    auto owner = [&](int c) { return dist ? dist_owner_of(i, c, h->dist_l0) : 0; };
    auto own = [&](int c) { return !dist || owner(c) == h->dist_rank; };

    // ---- MergeRedNodes ------------------------------------------------------
    if (i == L) {
      if (!h->dest_ready || h->leaf_soff != soff) {
        std::vector<int64_t> dest(pl.nnz, -1);
        for (int64_t k = 0; k < pl.nnz; ++k)
          if (pl.nnz_slot[k] >= 0)
            dest[k] = soff[pl.nnz_slot[k]] + pl.nnz_r[k] + (int64_t)pl.nnz_c[k] * sld[pl.nnz_slot[k]];
        h->d_dest.ensure(std::max<int64_t>(1, pl.nnz) * sizeof(int64_t), st);
        h2d_sync(h->d_dest.p, dest.data(), pl.nnz * sizeof(int64_t), st);
        h->leaf_soff = soff;
        h->dest_ready = true;
      }
      int ev = tbeg(h, K_SCATTER);
      launch_k(k_leaf_scatter, grid1(pl.nnz), 256, 0, st, h->d_values.as<double>(), h->d_dest.as<int64_t>(),
                                                    pl.nnz, base);
      tend(h, ev, 0, 24.0 * pl.nnz);
      ++h->launches_factor;
      CK(cudaGetLastError());
    } else {
      const std::vector<int> &rp = h->rnk[i + 1];  // sizes of the level-i reds
      double *pbase = h->arena[(i + 1) & 1].as<double>();
      std::vector<CopyTask> ct;
      for (const MergeSrc &ms : lv.merge) {
        int rows = rp[ms.src_cluster_r], cols = rp[ms.src_cluster_c];
        if (rows == 0 || cols == 0) continue;
        int ro = (ms.src_cluster_r & 1) ? rp[ms.src_cluster_r - 1] : 0;
        int co = (ms.src_cluster_c & 1) ? rp[ms.src_cluster_c - 1] : 0;
        CopyTask t{};
        t.src = pbase + prev_soff[ms.src_slot];
        t.lds = prev_sld[ms.src_slot];
        t.dst = slot_ptr(ms.dst_slot) + ro + (int64_t)co * sld[ms.dst_slot];
        t.ldd = sld[ms.dst_slot];
        t.rows = rows;
        t.cols = cols;
        t.mode = 0;
        t.trans = ms.trans ? 1 : 0;
        t.alpha = 1.0;
        ct.push_back(t);
      }
      launch_copy(h, ct, K_MERGE);
    }
    // ---- f2: ||all levels below||_F^2 += every super-node block of this level right
    // after MergeRedNodes (reading F2; the other slots are still zero here).  SPD
    // path: an off-diagonal slot stands for both orientations, a self slot's lower
    // triangle for the symmetric block.
    if (pl.flags & LORASP_FROBENIUS) {
      std::vector<FrobTask> ft;
      for (size_t q = 0; q < lv.slots.size(); ++q) {
        const int rows = bound(lv.slots[q].row), cols = bound(lv.slots[q].col);
        if (rows == 0 || cols == 0) continue;
        const bool self = lv.slots[q].row == lv.slots[q].col;
        ft.push_back(FrobTask{slot_ptr((int)q), sld[q], rows, cols, sym ? (self ? 1 : 2) : 0});
      }
      if (!ft.empty()) {
        h->d_frobpart.ensure(ft.size() * sizeof(double), st);
        FrobTask *dft = push(h, ft);
        launch_k(k_frob_part, (unsigned)ft.size(), 256, 0, st, dft, h->d_frobpart.as<double>());
        launch_k(k_frob_final, 1, 256, 0, st, h->d_frobpart.as<double>(), (int)ft.size(), h->d_frob.as<double>());
        h->launches_factor += 2;
      }
    }

    // ---- colour waves ---------------------------------------------------------
    // rank / size ratio seen so far (this level, else the level below): predicts
    // the fused pivot size n = m + r before the rank sync
    double rho_pred = 0.0;
    for (int c = 0; c < (int)h->rnk[i + 1].size() && i < L; ++c)
      if (h->msz[i + 1][c] > 0) rho_pred = std::max(rho_pred, (double)h->rnk[i + 1][c] / h->msz[i + 1][c]);
    for (size_t w = 0; w + 1 < lv.wave_begin.size(); ++w) {
      std::vector<int> comp, elim;
      for (int t = lv.wave_begin[w]; t < lv.wave_begin[w + 1]; ++t) {
        int c = lv.order[t];
        const SymNode &nd = lv.node[c];
        if (!nd.exists || m[c] == 0) continue;
        elim.push_back(c);
        if (nd.aux) comp.push_back(c);
      }
      if (elim.empty()) continue;
      // --- split pivot, part 1 (SPD): S -> L11^{-1} for the super-nodes of the
      // wave on stream2, overlapped with the compress below (S is final: only
      // earlier waves' Schur updates touch it).  K = [[S, V], [V^T, 0]] =
      // L diag(I, -I) L^T has L11 = chol(S); the V-dependent rest follows the
      // rank sync (part 2).  Nodes with m > PIVB_MAXN keep the fused pivot.
      std::vector<int64_t> s_off(K, -1);
      std::vector<CopyTask> s_ct;
      std::vector<PivTask> s_pt, s_big;
      BlockedPlan s_plan;
      int s_max = 0;
      if (!comp.empty() && !h->no_split && (sym || !h->lu_pivot)) {
        int64_t stot2 = 0;
        // A node is split when that pays: in waves wider than the GPU (the S
        // pivots then fill the sync gaps), or when its fused pivot would likely
        // exceed PIVB_MAXN (rank predicted from the largest r / m seen so far
        // at this level or the one below) and so take the launch-heavy blocked
        // path.  Otherwise the single fused k_pivot_blk is cheaper.
        const bool wide = elim.size() > 148;
        const int pmax = sym ? PIVB_MAXN : PIVLU_MAXN;
        // SPD nodes with m > PIVB_MAXN: part 1 is the blocked path on S (stream2,
        // hidden behind the compress), part 2 the rank-sized rest
        for (int c : elim)
          if ((m[c] <= pmax && (wide || m[c] + (int)std::ceil(rho_pred * m[c]) > pmax)) || (sym && m[c] > pmax)) {
            s_off[c] = stot2;
            stot2 += (sym ? 1 : 2) * (int64_t)m[c] * m[c];   // LU: L11^{-1} and U11^{-T}
          }
        if (stot2 > 0) {
          h->ws_S.ensure(stot2 * 8 + 256, st);
          for (int c : elim)
            if (s_off[c] >= 0 && m[c] <= pmax) s_max = std::max(s_max, m[c]);   // launch shape of the whole wave
          for (int c : elim) {
            if (s_off[c] < 0 || !own(c)) continue;
            const SymNode &nd = lv.node[c];
            CopyTask t{};
            t.src = slot_ptr(nd.self_slot);
            t.lds = sld[nd.self_slot];
            t.dst = h->ws_S.as<double>() + s_off[c];
            t.ldd = m[c];
            t.rows = m[c];
            t.cols = m[c];
            t.mode = 0;
            t.alpha = 1.0;
            s_ct.push_back(t);
            if (m[c] <= pmax) s_pt.push_back(PivTask{h->ws_S.as<double>() + s_off[c], m[c], m[c], 0, c});
            else s_big.push_back(PivTask{h->ws_S.as<double>() + s_off[c], m[c], m[c], 0, c});
            ++h->split_nodes;
          }
          if (!s_big.empty()) {
            h->ws_piv2.ensure(blocked_ws_bytes(s_big), st);
            build_blocked_plan(s_big, h->ws_piv2.as<double>(), s_plan);
          }
          CK(cudaEventRecord(h->ev_s0, st));   // S is final here; stream2 starts after it
        }
      }
      split_copies(s_ct);
      // part 1 is enqueued on stream2 once the compress kernels are queued
      auto enqueue_split_part1 = [&]() {
        if (s_pt.empty() && s_big.empty()) return;
        CK(cudaStreamWaitEvent(h->stream2, h->ev_s0, 0));
        const CopyTask *dct;
        const PivTask *dpt;
        const char *dplan = nullptr;
        if (capture) {   // descriptors resident in the graph's buffer
          dct = static_cast<const CopyTask *>(h->stg.push_deferred(s_ct.data(), s_ct.size() * sizeof(CopyTask), st));
          dpt = static_cast<const PivTask *>(h->stg.push_deferred(s_pt.data(), s_pt.size() * sizeof(PivTask), st));
          if (!s_big.empty())
            dplan = static_cast<const char *>(h->stg.push_deferred(s_plan.blob.data(), s_plan.blob.size(), st));
        } else {
          if (h->s1_pending) CK(cudaEventSynchronize(h->ev_s1));   // pinned task buffer reuse
          const size_t n0 = s_ct.size() * sizeof(CopyTask) + s_pt.size() * sizeof(PivTask);
          const size_t poff = (n0 + 255) & ~size_t(255);
          const size_t nbytes = poff + s_plan.blob.size();
          if (h->h_sp_cap < nbytes) {
            if (h->h_sp) CK(cudaFreeHost(h->h_sp));
            h->h_sp_cap = std::max<size_t>(nbytes * 2, 1 << 16);
            CK(cudaMallocHost(&h->h_sp, h->h_sp_cap));
          }
          char *hb = reinterpret_cast<char *>(h->h_sp);
          std::memcpy(hb, s_ct.data(), s_ct.size() * sizeof(CopyTask));
          std::memcpy(hb + s_ct.size() * sizeof(CopyTask), s_pt.data(), s_pt.size() * sizeof(PivTask));
          if (!s_plan.blob.empty()) std::memcpy(hb + poff, s_plan.blob.data(), s_plan.blob.size());
          h->d_sp.ensure(nbytes + 64, st);
          CK(cudaMemcpyAsync(h->d_sp.p, hb, nbytes, cudaMemcpyHostToDevice, h->stream2));
          dct = h->d_sp.as<CopyTask>();
          dpt = reinterpret_cast<const PivTask *>(h->d_sp.as<char>() + s_ct.size() * sizeof(CopyTask));
          dplan = h->d_sp.as<char>() + poff;
        }
        launch_k(k_copy, (unsigned)s_ct.size(), 256, 0, h->stream2, dct);
        if (!s_big.empty()) run_blocked_plan(h, s_plan, dplan, h->ws_piv2.as<double>(), h->stream2);
        if (s_pt.empty()) {
        } else if (sym) {
          const size_t smem = pivb_smem_bytes(s_max);
          launch_k(k_pivot_blk, (unsigned)s_pt.size(), 512, smem, h->stream2, dpt, h->d_status.as<int>());
        } else {   // no-pivot LU of S: L11^{-1} and U11^{-T} side by side in ws_S
          const size_t smem = pivb_smem_bytes(s_max);
          launch_k(k_pivot_lu_blk, (unsigned)s_pt.size(), 512, smem, h->stream2, dpt, h->d_status.as<int>());
        }
        h->launches_factor += 2;
        CK(cudaGetLastError());
        CK(cudaEventRecord(h->ev_s1, h->stream2));
        h->s1_pending = true;
      };
      // --- Compress: Gram + Jacobi + rank ---
      std::vector<int64_t> goff(K, 0);
      if (!comp.empty()) {
        int64_t gtot = 0, stot = 0, xtot = 0;
        for (int c : comp) {
          goff[c] = gtot;
          gtot += (int64_t)m[c] * m[c];
          stot += m[c];
          xtot += 7 * (int64_t)m[c] * m[c];  // eigen-solver scratch
        }
        h->ws_G.ensure(gtot * 8 + 256, st);
        h->ws_V.ensure(gtot * 8 + 256, st);
        h->ws_sig.ensure(stot * 8 + 256, st);
        h->ws_X.ensure(xtot * 8 + 256, st);
        h->d_ranks.ensure(comp.size() * sizeof(int) + 64, st);
        std::vector<GemmTask> gt, gt2;
        std::vector<GemmSeg> gs, gs2;
        std::vector<EigTask> et;
        int64_t soff_sig = 0, xoff = 0;
        int max_m = 0;
        double f_gram = 0, b_gram = 0, f_eig = 0, b_eig = 0;
        h->eig_clmax_hint = h->eig_bigmax_hint = h->eig_regmax_hint = h->eig_reg_wave_n = 0;
        for (int &x : h->eig_cl_wave_n) x = 0;
        h->eig_all_wave_n = dist ? (int)comp.size() : 0;
        if (dist) {
          CK(cudaMemsetAsync(h->d_ranks.p, 0, comp.size() * sizeof(int), st));
          // launch-shape choices from the whole wave, so that every rank runs
          // the single-GPU kernel variants (bit-identical results)
          for (int c : comp) {
            const int mc = m[c];
            if (mc >= EIG_REG_MIN && mc <= EIG_REG_M) {
              h->eig_regmax_hint = std::max(h->eig_regmax_hint, mc);
              ++h->eig_reg_wave_n;
              continue;
            }
            if (const int k = eig_cl_class(mc)) {
              h->eig_clmax_hint = std::max(h->eig_clmax_hint, mc);
              ++h->eig_cl_wave_n[k];
            }
            else h->eig_bigmax_hint = std::max(h->eig_bigmax_hint, mc);
          }
        }
        for (size_t q = 0; q < comp.size(); ++q) {
          const int c = comp[q];
          if (!own(c)) continue;   // distributed: the owner compresses (ranks exchanged below)
          const SymNode &nd = lv.node[c];
          const int mc = m[c];
          max_m = std::max(max_m, mc);
          GemmTask b{};
          b.C = h->ws_G.as<double>() + goff[c];
          b.ldc = mc;
          b.M = b.N = mc;
          b.ta = 0;
          b.tb = 1;
          b.tc = 0;
          b.beta = 0;
          b.seg0 = (int)gs.size();
          int R = 0;
          for (size_t k = 0; k < nd.partners.size(); ++k) {
            int p = nd.partners[k], sl = nd.pslot_src[k];
            int mk = size(p);
            if (mk == 0) continue;
            // SPD: sum X X^T with X = {S_c, p} (rows S_c) = A_k^T;  LU: the same for
            // X = Mat(p -> s) = B_k^T, plus A_k^T A_k from Mat(s -> p) (rows p) below
            GemmSeg g{};
            g.A = slot_ptr(sl);
            g.B = slot_ptr(sl);
            g.lda = g.ldb = sld[sl];
            g.K = mk;
            g.alpha = 1.0;
            gs.push_back(g);
            R += mk;
          }
          b.nseg = (int)gs.size() - b.seg0;
          add_tiles(gt, b);
          if (!sym) {   // second task set (ta = 1, tb = 0) for the A_k^T A_k part, accumulated
            GemmTask b2 = b;
            b2.ta = 1;
            b2.tb = 0;
            b2.beta = 1;
            b2.seg0 = (int)gs2.size();
            for (size_t k = 0; k < nd.partners.size(); ++k) {
              int p = nd.partners[k], sl = nd.pslot_src2[k];
              int mk = size(p);
              if (mk == 0) continue;
              gs2.push_back(GemmSeg{slot_ptr(sl), slot_ptr(sl), sld[sl], sld[sl], mk, 1.0});
              R += mk;
            }
            b2.nseg = (int)gs2.size() - b2.seg0;
            add_tiles(gt2, b2);
          }
          f_gram += (double)R * mc * mc;
          b_gram += 8.0 * R * mc + 8.0 * mc * mc;
          f_eig += 9.0 * mc * (double)mc * mc;
          b_eig += 16.0 * mc * mc;
          EigTask e{};
          e.G = b.C;
          e.V = h->ws_V.as<double>() + goff[c];
          e.sig = h->ws_sig.as<double>() + soff_sig;
          soff_sig += mc;
          e.work = h->ws_X.as<double>() + xoff;
          xoff += 7 * (int64_t)mc * mc;
          e.m = mc;
          e.node = c;
          e.rank_out = h->d_ranks.as<int>() + q;
          if (pl.flags & LORASP_FROBENIUS) {   // f2: Eq. curOff6 against ||all levels below||_F
            e.frob = h->d_frob.as<double>();
            e.frob_w = sym ? 2.0 : 1.0;
          }
          et.push_back(e);
        }
        h->stg.reserve(vbytes(gt) + vbytes(gs) + vbytes(gt2) + vbytes(gs2) + 4 * vbytes(et), st);
        GemmTask *d_gt = pushd(h, gt), *d_gt2 = pushd(h, gt2);
        GemmSeg *d_gs = pushd(h, gs), *d_gs2 = pushd(h, gs2);
        EigTask *de = pushd(h, et);
        h->stg.flush(st);
        launch_gemm_dev(h, d_gt, d_gs, gt.size(), K_GRAM, f_gram, b_gram);
        launch_gemm_dev(h, d_gt2, d_gs2, gt2.size(), K_GRAM, 0, 0);   // LU: A_k^T A_k half of the Gram
        int64_t want = (int64_t)max_m * max_m + 6 * (max_m + 8) + std::max(max_m, 512);
        int cap = (int)std::min<int64_t>(want, SMEM_LIMIT / 8);
        cap = std::max(cap, 6 * (max_m + 8) + std::max(max_m, 512));
        int ev = tbeg(h, K_JACOBI);
        cudaEvent_t dbg_e0 = nullptr, dbg_e1 = nullptr;
        if (h->debug) {
          cudaEventCreate(&dbg_e0);
          cudaEventCreate(&dbg_e1);
          cudaEventRecord(dbg_e0, st);
        }
        launch_eig(h, et, de, max_m, cap);
        enqueue_split_part1();
        if (h->debug) {
          cudaEventRecord(dbg_e1, st);
          cudaEventSynchronize(dbg_e1);
          float ms = 0;
          cudaEventElapsedTime(&ms, dbg_e0, dbg_e1);
          int mmin = 1 << 30, mmax = 0;
          for (auto &e : et) {
            mmin = std::min(mmin, e.m);
            mmax = std::max(mmax, e.m);
          }
          fprintf(stderr, "[lorasp] level %d wave %zu eig: %zu tasks m in [%d, %d]: %.3f ms\n", i, w, et.size(), mmin,
                  mmax, ms);
          cudaEventDestroy(dbg_e0);
          cudaEventDestroy(dbg_e1);
        }
        tend(h, ev, f_eig, b_eig);
        ++h->launches_factor;
        CK(cudaGetLastError());
        if (replay) {
          // predicted ranks; the computed ones are logged (stream order) and
          // compared after the final synchronisation
          CK(cudaMemcpyAsync(h->h_ranklog + rlog_pos, h->d_ranks.p, comp.size() * sizeof(int),
                             cudaMemcpyDeviceToHost, st));
          rlog.push_back(RankLog{i, rlog_pos, comp});
          rlog_pos += comp.size();
          for (size_t q = 0; q < comp.size(); ++q) {
            const int c = comp[q];
            r[c] = h->rank_cache[i][c];
            if (m[c] > 0) rho_pred = std::max(rho_pred, (double)r[c] / m[c]);
          }
        } else {
        auto ts0 = std::chrono::steady_clock::now();
        if (dist) {
          dist_allmax_ints(h, h->d_ranks.as<int>(), comp.size(), h->h_ranks);
        } else {
          CK(cudaMemcpyAsync(h->h_ranks, h->d_ranks.p, comp.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
          CK(cudaMemcpyAsync(h->h_status, h->d_status.p, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
          CK(cudaStreamSynchronize(st));
        }
        h->t_sync_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ts0).count();
        h->stg.reset();
        if (h->h_status[0] != 0) {
          throw Err(h->h_status[0], std::string(h->h_status[0] == LORASP_E_EIG_NOCONV
                                                    ? "Jacobi eigen-solver did not converge"
                                                    : "singular pivot") +
                                        " at level " + std::to_string(i) + " node " +
                                        std::to_string(h->h_status[1]));
        }
        for (size_t q = 0; q < comp.size(); ++q) {
          r[comp[q]] = h->h_ranks[q];
          if (m[comp[q]] > 0) rho_pred = std::max(rho_pred, (double)r[comp[q]] / m[comp[q]]);
        }
        }
      }
      // --- project, assemble, pivot, Z, Schur ---
      auto th0 = std::chrono::steady_clock::now();
      std::vector<GemmTask> pt, zt, stt;
      std::vector<GemmSeg> ps, zs, ss;
      std::vector<CopyTask> ct;
      std::vector<PivTask> pv;
      int64_t ctr_tot = 0;
      std::vector<int64_t> ctr_off(elim.size());
      std::vector<int> Wn(elim.size());
      for (size_t e = 0; e < elim.size(); ++e) {
        const int c = elim[e];
        const SymNode &nd = lv.node[c];
        int W = 0;
        for (int u : nd.n1) W += size(u);
        if (nd.aux) W += r[c];
        Wn[e] = W;
        ctr_off[e] = ctr_tot;
        ctr_tot += ((int64_t)(m[c] + r[c]) * W * (sym ? 1 : 2) + 31) & ~int64_t(31);
      }
      h->ws_ctr.ensure(std::max<int64_t>(ctr_tot, 32) * 8, st);
      // split-pivot scratch: Y (m x r) and T1 (r x m) per split node
      std::vector<GemmTask> sy_t, sg_t, sx_t;
      std::vector<GemmSeg> sy_s, sg_s, sx_s;
      std::vector<int64_t> split_off(elim.size(), 0);
      {
        int64_t yt = 0;
        for (size_t e = 0; e < elim.size(); ++e) {
          const int c = elim[e];
          split_off[e] = yt;
          if (s_off[c] >= 0) yt += (sym ? 1 : 2) * (((int64_t)m[c] * r[c] + 31) & ~int64_t(31));
        }
        if (yt > 0) {
          h->ws_Y.ensure(yt * 8 + 256, st);
          h->ws_T1.ensure(yt * 8 + 256, st);
        }
      }
      int max_n = 0, pv_max_small = 0, pv_max_all = 0, pv_cnt_small = 0, pv_cnt_all = 0;
      double f_proj = 0, b_proj = 0, f_piv = 0, b_piv = 0, f_z = 0, b_z = 0, f_s = 0, b_s = 0;
      // neighbour push (dist): the blocks each node writes, their reader masks, the writer
      std::vector<DirtyList> wr_blocks;
      std::vector<uint32_t> wr_masks;
      std::vector<int> wr_writer;
      for (size_t e = 0; e < elim.size(); ++e) {
        const int c = elim[e];
        const SymNode &nd = lv.node[c];
        const int mc = m[c], rc = r[c], n = mc + rc, W = Wn[e];
        max_n = std::max(max_n, n);
        // distributed: every rank lays out every node (same records and host
        // state); the tasks of nodes it does not own are dropped at the end
        const size_t n_pt = pt.size(), n_ps = ps.size(), n_ct = ct.size(), n_pv = pv.size(), n_zt = zt.size(),
                     n_zs = zs.size(), n_stt = stt.size(), n_ss = ss.size(), n_syt = sy_t.size(),
                     n_sys = sy_s.size(), n_sgt = sg_t.size(), n_sgs = sg_s.size(), n_sxt = sx_t.size(),
                     n_sxs = sx_s.size();
        std::vector<int> wslots;   // slots this node writes (projection + Schur targets)
        double *V = h->ws_V.as<double>() + goff[c];
        // project: R_k = A_k V  into  P(b) <-> p_k  (edge rules 2/3, P:l.385-386)
        int R = 0;
        if (nd.aux && rc > 0) {
          for (size_t k = 0; k < nd.partners.size(); ++k) {
            int p = nd.partners[k];
            int mk = size(p);
            R += mk;
            if (mk == 0) continue;
            // SPD: R_k = (A_k^T)^T V from {S_c, p} into {P_c, p}.
            // LU:  R_k = A_k V (Mat(s->p)) into Mat(P->p);  Q_k = B_k V (Mat(p->s)^T V)
            //      stored transposed into Mat(p->P) = Q_k^T
            int s1 = sym ? nd.pslot_src[k] : nd.pslot_src2[k], s2 = nd.pslot_dst[k];
            wslots.push_back(s2);
            if (!sym) wslots.push_back(nd.pslot_dst2[k]);
            GemmTask b{};
            b.C = slot_ptr(s2);
            b.ldc = sld[s2];
            b.M = mk;
            b.N = rc;
            b.ta = sym ? 1 : 0;
            b.tb = 0;
            b.tc = (lv.slots[s2].row == p) ? 0 : 1;
            b.beta = 0;
            b.seg0 = (int)ps.size();
            b.nseg = 1;
            GemmSeg g{};
            g.A = slot_ptr(s1);
            g.lda = sld[s1];
            g.B = V;
            g.ldb = mc;
            g.K = mc;
            g.alpha = 1.0;
            ps.push_back(g);
            add_tiles(pt, b);
            if (!sym) {
              const int s3 = nd.pslot_src[k], s4 = nd.pslot_dst2[k];
              GemmTask q2 = b;
              q2.C = slot_ptr(s4);
              q2.ldc = sld[s4];
              q2.ta = 1;
              q2.tc = 1;   // Mat(p -> P) has rows P: store Q_k^T
              q2.seg0 = (int)ps.size();
              ps.push_back(GemmSeg{slot_ptr(s3), V, sld[s3], mc, mc, 1.0});
              add_tiles(pt, q2);
            }
          }
        } else if (nd.aux) {
          for (int p : nd.partners) R += size(p);
        }
        // record F = [L^{-1} | Z]  (n x (n + W), leading dimension ldF = n rounded up to
        // even so that every column starts 16-byte aligned for the bulk-copy apply)
        // LU: F = [L^{-1} | U^{-T} | X = L^{-1} C | Y^T = U^{-T} R^T]
        const int ldF = n + (n & 1);
        const int64_t fcols = sym ? (int64_t)(n + W) : (int64_t)(2 * n + 2 * W);
        double *F = h->fpool.alloc((size_t)ldF * fcols + 2);  // +16 B: bulk copies round up
        double *ctr = h->ws_ctr.as<double>() + ctr_off[e];
        double *rtr = sym ? nullptr : ctr + (int64_t)n * W;   // LU: R (W x n, ld W)
        h->f_doubles += (int64_t)ldF * fcols;
        const int64_t offX = sym ? (int64_t)ldF * n : 2 * (int64_t)ldF * n;
        const int64_t offY = offX + (int64_t)ldF * W;
        NodeRec rec;
        rec.level = i;
        rec.c = c;
        rec.m = mc;
        rec.r = rc;
        rec.W = W;
        rec.F = F;
        rec.ld = ldF;
        rec.zf_off = sym ? offX : offY;   // forward: Z (SPD) / Y^T (LU)
        rec.zb_off = offX;                // backward: Z / X
        rec.lb_off = sym ? 0 : (int64_t)ldF * n;   // backward triangle: L^{-1} / U^{-T}
        // assemble pivot K = [[S, V], [V^T, 0]] (lower part used); split nodes:
        // L11^{-1} from part 1 (upper triangle zero) and a zero upper-right block
        const bool split = s_off[c] >= 0;
        CopyTask t{};
        t.src = split ? h->ws_S.as<double>() + s_off[c] : slot_ptr(nd.self_slot);
        t.lds = split ? mc : sld[nd.self_slot];
        t.dst = F;
        t.ldd = ldF;
        t.rows = mc;
        t.cols = mc;
        t.mode = 0;
        t.trans = 0;
        t.alpha = 1.0;
        ct.push_back(t);
        if (split && rc > 0) {
          t = CopyTask{};
          t.dst = F + (int64_t)mc * ldF;
          t.ldd = ldF;
          t.rows = mc;
          t.cols = rc;
          t.mode = 1;
          t.alpha = 0.0;
          ct.push_back(t);
        }
        if (split && !sym) {   // LU: region 1 (1,1) = U11^{-T} from part 1, (1,2) = 0
          double *R1 = F + (int64_t)ldF * n;
          t = CopyTask{};
          t.src = h->ws_S.as<double>() + s_off[c] + (int64_t)mc * mc;
          t.lds = mc;
          t.dst = R1;
          t.ldd = ldF;
          t.rows = mc;
          t.cols = mc;
          t.mode = 0;
          t.alpha = 1.0;
          ct.push_back(t);
          if (rc > 0) {
            t = CopyTask{};
            t.dst = R1 + (int64_t)mc * ldF;
            t.ldd = ldF;
            t.rows = mc;
            t.cols = rc;
            t.mode = 1;
            t.alpha = 0.0;
            ct.push_back(t);
          }
        }
        if (!split && rc > 0) {
          t = CopyTask{};
          t.src = V;
          t.lds = mc;
          t.dst = F + mc;
          t.ldd = ldF;
          t.rows = rc;
          t.cols = mc;
          t.mode = 0;
          t.trans = 1;
          t.alpha = 1.0;
          ct.push_back(t);  // V^T (s -> b, rule 4)
          t = CopyTask{};
          t.dst = F + mc + (int64_t)mc * ldF;
          t.ldd = ldF;
          t.rows = rc;
          t.cols = rc;
          t.mode = 1;
          t.alpha = 0.0;
          ct.push_back(t);  // b has no self block (reading Z13)
          if (!sym) {
            t = CopyTask{};
            t.src = V;
            t.lds = mc;
            t.dst = F + (int64_t)mc * ldF;
            t.ldd = ldF;
            t.rows = mc;
            t.cols = rc;
            t.mode = 0;
            t.alpha = 1.0;
            ct.push_back(t);  // Mat(b -> s) = V (rule 4), upper-right of the LU pivot
          }
        }
        // coupling C: rows (s; b), columns T = N1(s) + [P(b)]
        int zc = 0;
        for (size_t k = 0; k < nd.n1.size(); ++k) {
          int u = nd.n1[k], wu = size(u);
          rec.T.push_back(u);
          rec.w.push_back(wu);
          if (wu > 0) {
            t = CopyTask{};
            t.src = slot_ptr(nd.n1_slot[k]);
            t.lds = sld[nd.n1_slot[k]];
            t.dst = ctr + (int64_t)zc * n;
            t.ldd = n;
            t.rows = mc;
            t.cols = wu;
            t.mode = 0;
            t.alpha = 1.0;
            ct.push_back(t);
            if (!sym) {   // R rows of n: Mat(s -> n) (wu x m), b columns stay zero
              t = CopyTask{};
              t.src = slot_ptr(nd.n1_slot2[k]);
              t.lds = sld[nd.n1_slot2[k]];
              t.dst = rtr + zc;
              t.ldd = W;
              t.rows = wu;
              t.cols = mc;
              t.mode = 0;
              t.alpha = 1.0;
              ct.push_back(t);
              if (rc > 0) {
                t = CopyTask{};
                t.dst = rtr + zc + (int64_t)mc * W;
                t.ldd = W;
                t.rows = wu;
                t.cols = rc;
                t.mode = 1;
                t.alpha = 0.0;
                ct.push_back(t);
              }
            }
          }
          zc += wu;
        }
        if (rc > 0 && zc > 0) {
          t = CopyTask{};
          t.dst = ctr + mc;
          t.ldd = n;
          t.rows = rc;
          t.cols = zc;
          t.mode = 1;
          t.alpha = 0.0;
          ct.push_back(t);
        }
        if (nd.aux) {
          rec.T.push_back(K + c);
          rec.w.push_back(rc);
          if (rc > 0) {
            t = CopyTask{};
            t.dst = ctr + (int64_t)zc * n;
            t.ldd = n;
            t.rows = mc;
            t.cols = rc;
            t.mode = 1;
            t.alpha = 0.0;
            ct.push_back(t);
            t = CopyTask{};
            t.dst = ctr + (int64_t)zc * n + mc;
            t.ldd = n;
            t.rows = rc;
            t.cols = rc;
            t.mode = 2;
            t.alpha = -1.0;
            ct.push_back(t);  // b <-> P(b): -I_r (rule 5)
            if (!sym) {       // R rows of P(b): Mat(s -> P) = 0, Mat(b -> P) = -I
              t = CopyTask{};
              t.dst = rtr + zc;
              t.ldd = W;
              t.rows = rc;
              t.cols = mc;
              t.mode = 1;
              t.alpha = 0.0;
              ct.push_back(t);
              t = CopyTask{};
              t.dst = rtr + zc + (int64_t)mc * W;
              t.ldd = W;
              t.rows = rc;
              t.cols = rc;
              t.mode = 2;
              t.alpha = -1.0;
              ct.push_back(t);
            }
          }
        }
        // pivot
        if (!split) {
          pv.push_back(PivTask{F, ldF, mc, rc, c});
        } else if (rc > 0 && !sym) {
          // LU part 2 (K = [[S, V], [V^T, 0]] = L U, S = L11 U11 from part 1):
          // Y = L11^{-1} V (= U12), Zt = U11^{-T} V (= L21^T), L22 U22 = -Zt^T Y;
          // (L^{-1})21 = -L22^{-1} (Zt^T L11^{-1}), (U^{-T})21 = -U22^{-T} (Y^T U11^{-T})
          double *R1 = F + (int64_t)ldF * n;
          double *Yb = h->ws_Y.as<double>() + split_off[e];
          double *Zt = Yb + (((int64_t)mc * rc + 31) & ~int64_t(31));
          double *T1 = h->ws_T1.as<double>() + split_off[e];
          double *T2 = T1 + (((int64_t)mc * rc + 31) & ~int64_t(31));
          auto gt = [&](std::vector<GemmTask> &tl, std::vector<GemmSeg> &sl, double *C, int ldc, int M, int N, int ta,
                        GemmSeg g) {
            GemmTask q{};
            q.C = C;
            q.ldc = ldc;
            q.M = M;
            q.N = N;
            q.ta = ta;
            q.beta = 0;
            q.seg0 = (int)sl.size();
            q.nseg = 1;
            sl.push_back(g);
            add_tiles(tl, q);
          };
          gt(sy_t, sy_s, Yb, mc, mc, rc, 0, GemmSeg{F, V, ldF, mc, mc, 1.0});
          gt(sy_t, sy_s, Zt, mc, mc, rc, 0, GemmSeg{R1, V, ldF, mc, mc, 1.0});
          gt(sg_t, sg_s, F + mc + (int64_t)mc * ldF, ldF, rc, rc, 1, GemmSeg{Zt, Yb, mc, mc, mc, -1.0});
          gt(sg_t, sg_s, T1, rc, rc, mc, 1, GemmSeg{Zt, F, mc, ldF, mc, 1.0});
          gt(sg_t, sg_s, T2, rc, rc, mc, 1, GemmSeg{Yb, R1, mc, ldF, mc, 1.0});
          pv.push_back(PivTask{F + mc + (int64_t)mc * ldF, ldF, rc, 0, c, R1 + mc + (int64_t)mc * ldF});
          gt(sx_t, sx_s, F + mc, ldF, rc, mc, 0, GemmSeg{F + mc + (int64_t)mc * ldF, T1, ldF, rc, rc, -1.0});
          gt(sx_t, sx_s, R1 + mc, ldF, rc, mc, 0, GemmSeg{R1 + mc + (int64_t)mc * ldF, T2, ldF, rc, rc, -1.0});
        } else if (rc > 0) {
          // part 2: Y = L11^{-1} V, L21 = Y^T, L22 = chol(Y^T Y) (K22 = 0 and
          // D2 = -I), X21 = -L22^{-1} Y^T L11^{-1}
          double *Yb = h->ws_Y.as<double>() + split_off[e];
          double *T1 = h->ws_T1.as<double>() + split_off[e];
          GemmTask g{};
          g.C = Yb;
          g.ldc = mc;
          g.M = mc;
          g.N = rc;
          g.beta = 0;
          g.seg0 = (int)sy_s.size();
          g.nseg = 1;
          sy_s.push_back(GemmSeg{F, V, ldF, mc, mc, 1.0});
          add_tiles(sy_t, g);
          g = GemmTask{};
          g.C = F + mc + (int64_t)mc * ldF;
          g.ldc = ldF;
          g.M = rc;
          g.N = rc;
          g.ta = 1;
          g.beta = 0;
          g.seg0 = (int)sg_s.size();
          g.nseg = 1;
          sg_s.push_back(GemmSeg{Yb, Yb, mc, mc, mc, 1.0});
          add_tiles(sg_t, g);
          g = GemmTask{};
          g.C = T1;
          g.ldc = rc;
          g.M = rc;
          g.N = mc;
          g.ta = 1;
          g.beta = 0;
          g.seg0 = (int)sg_s.size();
          g.nseg = 1;
          sg_s.push_back(GemmSeg{Yb, F, mc, ldF, mc, 1.0});
          add_tiles(sg_t, g);
          pv.push_back(PivTask{F + mc + (int64_t)mc * ldF, ldF, rc, 0, c});
          g = GemmTask{};
          g.C = F + mc;
          g.ldc = ldF;
          g.M = rc;
          g.N = mc;
          g.beta = 0;
          g.seg0 = (int)sx_s.size();
          g.nseg = 1;
          sx_s.push_back(GemmSeg{F + mc + (int64_t)mc * ldF, T1, ldF, rc, rc, -1.0});
          add_tiles(sx_t, g);
        }
        // Z = L^{-1} C  (L^{-1} lower triangular: row tile tm needs k < tm + 64)
        if (W > 0) {
          for (int tn = 0; tn < W; tn += GT)
            for (int tm = 0; tm < n; tm += GT) {
              GemmTask b{};
              b.C = F + offX;
              b.ldc = ldF;
              b.M = n;
              b.N = W;
              b.tm = tm;
              b.tn = tn;
              b.beta = 0;
              b.seg0 = (int)zs.size();
              b.nseg = 1;
              GemmSeg g{};
              g.A = F;
              g.lda = ldF;
              g.B = ctr;
              g.ldb = n;
              g.K = (!sym && h->lu_pivot) ? n : std::min(n, tm + GT);   // L^{-1} P is not triangular
              g.alpha = 1.0;
              zs.push_back(g);
              zt.push_back(b);
              if (!sym) {   // Y^T = U^{-T} R^T  (U^{-T} lower triangular)
                GemmTask y = b;
                y.C = F + offY;
                y.tb = 1;
                y.seg0 = (int)zs.size();
                zs.push_back(GemmSeg{F + (int64_t)ldF * n, rtr, ldF, W, std::min(n, tm + GT), 1.0});
                zt.push_back(y);
              }
            }
        }
        // Schur: T_a,b -= Z_a^T D Z_b   (D = diag(I_m, -I_r))
        {
          const std::vector<int> &T = rec.T;
          std::vector<int> zoff(T.size() + 1, 0);
          for (size_t a = 0; a < T.size(); ++a) zoff[a + 1] = zoff[a] + rec.w[a];
          const double *Z = F + offX;
          if (!sym) {   // LU: Mat(T_b -> T_a) -= Y_a X_b for every ordered pair
            const double *Yt = F + offY;
            for (size_t a = 0; a < T.size(); ++a)
              for (size_t bb = 0; bb < T.size(); ++bb) {
                const int wa = rec.w[a], wb = rec.w[bb];
                if (wa == 0 || wb == 0) continue;
                const int sl = nd.tslot[a * T.size() + bb];
                wslots.push_back(sl);
                GemmTask b{};
                b.C = slot_ptr(sl);
                b.ldc = sld[sl];
                b.M = wa;
                b.N = wb;
                b.ta = 1;
                b.tb = 0;
                b.tc = 0;
                b.beta = 1;
                b.seg0 = (int)ss.size();
                b.nseg = 1;
                ss.push_back(GemmSeg{Yt + (int64_t)zoff[a] * ldF, Z + (int64_t)zoff[bb] * ldF, ldF, ldF, n, -1.0});
                add_tiles(stt, b);
              }
          }
          size_t idx = 0;
          for (size_t a = 0; sym && a < T.size(); ++a)
            for (size_t bb = 0; bb <= a; ++bb, ++idx) {
              int wa = rec.w[a], wb = rec.w[bb];
              if (wa == 0 || wb == 0) continue;
              int sl = nd.tslot[idx];
              wslots.push_back(sl);
              GemmTask b{};
              b.C = slot_ptr(sl);
              b.ldc = sld[sl];
              b.M = wa;
              b.N = wb;
              b.ta = 1;
              b.tb = 0;
              b.tc = (a != bb && lv.slots[sl].row != T[a]) ? 1 : 0;
              b.beta = 1;
              b.seg0 = (int)ss.size();
              GemmSeg g{};
              g.A = Z + (int64_t)zoff[a] * ldF;
              g.B = Z + (int64_t)zoff[bb] * ldF;
              g.lda = g.ldb = ldF;
              g.K = mc;
              g.alpha = -1.0;
              ss.push_back(g);
              if (rc > 0) {
                g.A += mc;
                g.B += mc;
                g.K = rc;
                g.alpha = 1.0;
                ss.push_back(g);
              }
              b.nseg = (int)ss.size() - b.seg0;
              add_tiles(stt, b);
            }
        }
        h->flops_model += node_flops(mc, rc, nd.aux ? R : 0, W, sym);
        f_proj += 2.0 * R * mc * rc;
        b_proj += 8.0 * ((double)R * mc + (double)R * rc + (double)mc * rc);
        f_piv += ((double)mc * mc * mc + (double)rc * rc * rc) / 3.0;
        b_piv += 16.0 * n * n;
        f_z += ((double)mc * mc + (double)rc * rc) * W;
        b_z += 8.0 * ((double)n * n + 2.0 * n * W);
        f_s += (double)(mc + rc) * W * W;
        b_s += 8.0 * (2.0 * n * W + (double)W * W);
        if (dist) {
          for (size_t q = n_pv; q < pv.size(); ++q) {   // the pivot batch as one GPU would see it
            const int pn = pv[q].m + pv[q].r;
            pv_max_all = std::max(pv_max_all, pn);
            ++pv_cnt_all;
            if (pn <= PIV_SMALL_N) {
              pv_max_small = std::max(pv_max_small, pn);
              ++pv_cnt_small;
            }
          }
          // the record F stays on its owner (distributed apply); each written
          // block goes to the ranks that read or update it later
          std::sort(wslots.begin(), wslots.end());
          wslots.erase(std::unique(wslots.begin(), wslots.end()), wslots.end());
          for (int sl : wslots)
            if (slen[sl] > 0) {
              wr_blocks.push_back(DirtyList{{slot_ptr(sl), slen[sl]}});
              wr_masks.push_back(h->slot_readers[i][sl]);
              wr_writer.push_back(owner(c));
            }
          if (!own(c)) {
            pt.resize(n_pt);
            ps.resize(n_ps);
            ct.resize(n_ct);
            pv.resize(n_pv);
            zt.resize(n_zt);
            zs.resize(n_zs);
            stt.resize(n_stt);
            ss.resize(n_ss);
            sy_t.resize(n_syt);
            sy_s.resize(n_sys);
            sg_t.resize(n_sgt);
            sg_s.resize(n_sgs);
            sx_t.resize(n_sxt);
            sx_s.resize(n_sxs);
          }
        }
        h->recs.push_back(std::move(rec));
      }
      h->piv_maxn_hint = dist ? (sym ? pv_max_small : pv_max_all) : 0;
      h->piv_cnt_hint = dist ? (sym ? pv_cnt_small : pv_cnt_all) : 0;
      // all descriptors of the wave travel in one H2D copy
      // descriptors in two groups: the pivot section below pushes its own task
      // lists, and a staging-ring wrap there (which reuses the ring after
      // synchronising) would overwrite descriptors pushed earlier but consumed
      // later — so Z / Schur descriptors are pushed after the pivots
      split_copies(ct);
      h->stg.reserve(vbytes(pt) + vbytes(ps) + vbytes(ct), st);
      GemmTask *d_pt = pushd(h, pt);
      GemmSeg *d_ps = pushd(h, ps);
      CopyTask *d_ct = pushd(h, ct);
      h->stg.flush(st);
      h->t_host_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - th0).count();
      launch_gemm_dev(h, d_pt, d_ps, pt.size(), K_PROJECT, f_proj, b_proj);
      if (h->s1_pending) CK(cudaStreamWaitEvent(st, h->ev_s1, 0));   // part 1 done (L11^{-1} in ws_S)
      launch_copy_dev(h, d_ct, ct, K_ASSEMBLE);
      if (!sy_t.empty()) {
        launch_gemm(h, sy_t, sy_s, K_PIVOT, 0, 0);
        launch_gemm(h, sg_t, sg_s, K_PIVOT, 0, 0);
      }
      if (sym) {
        cudaEvent_t pe0 = nullptr, pe1 = nullptr;
        if (h->debug) {
          cudaEventCreate(&pe0);
          cudaEventCreate(&pe1);
          cudaEventRecord(pe0, st);
        }
        pivots(h, pv, f_piv, b_piv);
        if (h->debug) {
          cudaEventRecord(pe1, st);
          cudaEventSynchronize(pe1);
          float ms = 0;
          cudaEventElapsedTime(&ms, pe0, pe1);
          int nmin = 1 << 30, nmax = 0;
          for (auto &t : pv) {
            nmin = std::min(nmin, t.m + t.r);
            nmax = std::max(nmax, t.m + t.r);
          }
          fprintf(stderr, "[lorasp] level %d wave %zu pivot: %zu tasks n in [%d, %d]: %.3f ms\n", i, w, pv.size(), nmin,
                  nmax, ms);
          cudaEventDestroy(pe0);
          cudaEventDestroy(pe1);
        }
        if (!sx_t.empty()) launch_gemm(h, sx_t, sx_s, K_PIVOT, 0, 0);
      } else {
        cudaEvent_t pe0 = nullptr, pe1 = nullptr;
        if (h->debug) {
          cudaEventCreate(&pe0);
          cudaEventCreate(&pe1);
          cudaEventRecord(pe0, st);
        }
        pivots_lu(h, pv, f_piv, b_piv);
        if (!sx_t.empty()) launch_gemm(h, sx_t, sx_s, K_PIVOT, 0, 0);
        if (h->debug) {
          cudaEventRecord(pe1, st);
          cudaEventSynchronize(pe1);
          float ms = 0;
          cudaEventElapsedTime(&ms, pe0, pe1);
          int nmin = 1 << 30, nmax = 0;
          for (auto &t : pv) {
            nmin = std::min(nmin, t.m + t.r);
            nmax = std::max(nmax, t.m + t.r);
          }
          fprintf(stderr, "[lorasp] level %d wave %zu pivot: %zu tasks n in [%d, %d]: %.3f ms\n", i, w, pv.size(), nmin,
                  nmax, ms);
          cudaEventDestroy(pe0);
          cudaEventDestroy(pe1);
        }
      }
      h->stg.reserve(vbytes(zt) + vbytes(zs) + vbytes(stt) + vbytes(ss), st);
      GemmTask *d_zt = pushd(h, zt), *d_stt = pushd(h, stt);
      GemmSeg *d_zs = pushd(h, zs), *d_ss = pushd(h, ss);
      h->stg.flush(st);
      launch_gemm_dev(h, d_zt, d_zs, zt.size(), K_ZGEMM, f_z, b_z);
      launch_gemm_dev(h, d_stt, d_ss, stt.size(), K_SCHUR, f_s, b_s);
      if (dist) dist_push(h, wr_blocks, wr_masks, wr_writer);
      if (h->debug) {
        CK(cudaStreamSynchronize(st));
        CK(cudaMemcpy(h->h_status, h->d_status.p, 4 * sizeof(int), cudaMemcpyDeviceToHost));
        fprintf(stderr, "[lorasp] level %d wave %zu: %zu nodes, %zu compressed, status %d (node %d); ranks:",
                i, w, elim.size(), comp.size(), h->h_status[0], h->h_status[1]);
        for (int c : elim) fprintf(stderr, " %d:%d/%d", c, r[c], m[c]);
        fprintf(stderr, "\n");
      }
    }
    prev_soff.swap(soff);
    prev_sld.swap(sld);
  }
  if (capture) {   // the caller ends the capture, launches and verifies
    CK(cudaMemcpyAsync(h->h_status, h->d_status.p, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
    h->fg_rlog = std::move(rlog);
    return true;
  }
  if (dist) {
    dist_allmax_ints(h, nullptr, 0, nullptr);
  } else {
    CK(cudaMemcpyAsync(h->h_status, h->d_status.p, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  h->stg.reset();
  tflush(h);
  if (replay && !replay_check(h, rlog)) return false;
  status_check(h);
  if (replay) {
    // same ranks => same record layout (the pool is bump-allocated in the same
    // order): the apply plan of the previous factorization is still valid
    h->factored = true;
    return true;
  }

  // ---- apply plan: vector layout over red nodes of every level --------------
  std::vector<std::vector<int64_t>> voff(L + 1);
  int64_t tot = 0;
  for (int k = L; k >= 0; --k) {
    int ncl = 1 << k;
    voff[k].assign(ncl, 0);
    for (int c = 0; c < ncl; ++c) {
      voff[k][c] = tot;
      tot += (k == L) ? pl.leaf_size[c] : h->rnk[k + 1][c];
    }
  }
  h->vec_len = tot;
  std::vector<ApNode> an;
  std::vector<ApSeg> as;
  int64_t ytot = 0;
  std::vector<int64_t> yoff;
  for (auto &rc : h->recs) {
    yoff.push_back(ytot);
    ytot += ((int64_t)(rc.m + rc.r) + 3) & ~int64_t(3);
  }
  h->d_y.ensure(std::max<int64_t>(ytot, 8) * 8, st);
  h->ap_wave_begin.clear();
  size_t fwd = 0, bwd = 0, max_col = 0;
  // waves in recs order; distributed: a wave's owned nodes first (the apply
  // launches only those), every rank's written vector segments recorded
  std::vector<size_t> order;
  {
    std::vector<size_t> wb;
    int pl_ = -1, pw_ = -1;
    for (size_t q = 0; q < h->recs.size(); ++q) {
      const int wv = pl.lev[h->recs[q].level].node[h->recs[q].c].wave;
      if (h->recs[q].level != pl_ || wv != pw_) wb.push_back(q);
      pl_ = h->recs[q].level;
      pw_ = wv;
    }
    wb.push_back(h->recs.size());
    h->ap_wave_nown.assign(wb.size() - 1, 0);
    h->ap_dirty_f.assign(dist ? wb.size() - 1 : 0, std::vector<std::vector<std::pair<int64_t, int64_t>>>(h->dist_world));
    h->ap_dirty_b.assign(dist ? wb.size() - 1 : 0, std::vector<std::vector<std::pair<int64_t, int64_t>>>(h->dist_world));
    for (size_t w = 0; w + 1 < wb.size(); ++w) {
      for (int pass = 0; pass < 2; ++pass)
        for (size_t q = wb[w]; q < wb[w + 1]; ++q) {
          const bool mine = !dist || dist_owner_of(h->recs[q].level, h->recs[q].c, h->dist_l0) == h->dist_rank;
          if (mine == (pass == 0)) order.push_back(q);
          if (mine && pass == 0) ++h->ap_wave_nown[w];
        }
    }
  }
  int prev_level = -1, prev_wave = -1;
  for (size_t qq = 0; qq < order.size(); ++qq) {
    const size_t q = order[qq];
    const NodeRec &rc = h->recs[q];
    const SymLevel &lv = pl.lev[rc.level];
    int wv = lv.node[rc.c].wave;
    if (rc.level != prev_level || wv != prev_wave) h->ap_wave_begin.push_back((int)qq);
    prev_level = rc.level;
    prev_wave = wv;
    ApNode a{};
    a.F = rc.F;
    a.y = h->d_y.as<double>() + yoff[q];
    a.off_s = voff[rc.level][2 * rc.c];
    a.m = rc.m;
    a.r = rc.r;
    a.W = rc.W;
    a.ld = rc.ld;
    a.zf_off = rc.zf_off;
    a.zb_off = rc.zb_off;
    a.lb_off = rc.lb_off;
    a.sym = (pl.flags & LORASP_SPD) ? 1 : 0;
    a.full = (!a.sym && h->lu_pivot) ? 1 : 0;
    a.seg0 = (int)as.size();
    int zc = 0;
    const int K = lv.K;
    for (size_t k = 0; k < rc.T.size(); ++k) {
      int u = rc.T[k];
      ApSeg sgm{};
      sgm.voff = (u < K) ? voff[rc.level][2 * u] : voff[rc.level - 1][u - K];
      sgm.w = rc.w[k];
      sgm.zc = zc;
      zc += rc.w[k];
      if (sgm.w > 0) as.push_back(sgm);
    }
    a.nseg = (int)as.size() - a.seg0;
    if (dist) {
      const int wi = (int)h->ap_wave_begin.size() - 1;
      const int g = dist_owner_of(rc.level, rc.c, h->dist_l0);
      for (int k = a.seg0; k < a.seg0 + a.nseg; ++k) h->ap_dirty_f[wi][g].push_back({as[k].voff, (int64_t)as[k].w});
      h->ap_dirty_b[wi][g].push_back({a.off_s, (int64_t)rc.m});
    }
    an.push_back(a);
    int n = rc.m + rc.r;
    fwd = std::max(fwd, (size_t)(rc.m + n + 2 * rc.W + 258));   // rhs, y, Z^T D y, target prefetch, partials
    bwd = std::max(bwd, (size_t)(n + rc.W + 258));               // u, x_T, partials
    max_col = std::max(max_col, (size_t)rc.ld);
  }
  h->ap_wave_begin.push_back((int)h->recs.size());
  // split apply: waves of few nodes (the upper levels) are latency-bound when one
  // CTA streams a whole record; their Z columns are spread over CTAs (~64 KB of
  // Z each), y = L^{-1} rhs over 64-row slabs and x = L^{-T} u over 32-column
  // slabs
  std::vector<ApPart> parts;
  h->ap_part_begin.clear();
  h->ap_ypart_begin.clear();
  h->ap_lpart_begin.clear();
  h->ap_part_end.clear();
  h->ap_wave_split.assign(h->ap_wave_begin.size() - 1, 0);
  int64_t utot = 0;
  for (size_t w = 0; w + 1 < h->ap_wave_begin.size(); ++w) {
    const int b0 = h->ap_wave_begin[w], b1 = h->ap_wave_begin[w + 1], cnt = b1 - b0;
    std::vector<int> ns(cnt, 1);
    bool split = false;
    if (!h->no_split_apply && !dist && cnt <= 64) {
      double zmax = 0;
      for (int q = b0; q < b1; ++q) zmax = std::max(zmax, 8.0 * (an[q].m + an[q].r) * an[q].W);
      if (zmax >= 64.0 * 1024) {
        const int cap = std::max(1, std::min(32, 444 / std::max(cnt, 1)));
        for (int q = b0; q < b1; ++q) {
          const double zbytes = 8.0 * (an[q].m + an[q].r) * an[q].W;
          int k = (int)std::ceil(zbytes / (64.0 * 1024));
          k = std::max(1, std::min({k, cap, std::max(1, an[q].W)}));
          ns[q - b0] = k;
          split = split || k > 1;
        }
      }
    }
    h->ap_wave_split[w] = split;
    h->ap_part_begin.push_back((int)parts.size());
    if (split) {
      for (int q = b0; q < b1; ++q) {
        const int k = ns[q - b0], n = an[q].m + an[q].r, W = an[q].W;
        an[q].nsplit = k;
        an[q].upart = utot;
        utot += (int64_t)k * n;
        for (int pp = 0; pp < k; ++pp)
          parts.push_back(ApPart{q, (int)((int64_t)W * pp / k), (int)((int64_t)W * (pp + 1) / k), pp});
      }
      h->ap_ypart_begin.push_back((int)parts.size());
      for (int q = b0; q < b1; ++q)
        for (int i0 = 0; i0 < an[q].m + an[q].r; i0 += 64)
          parts.push_back(ApPart{q, i0, std::min(an[q].m + an[q].r, i0 + 64), 0});
      h->ap_lpart_begin.push_back((int)parts.size());
      for (int q = b0; q < b1; ++q)
        for (int i0 = 0; i0 < an[q].m; i0 += 32) parts.push_back(ApPart{q, i0, std::min(an[q].m, i0 + 32), 0});
    } else {
      for (int q = b0; q < b1; ++q) an[q].nsplit = 1;
      h->ap_ypart_begin.push_back((int)parts.size());
      h->ap_lpart_begin.push_back((int)parts.size());
    }
    h->ap_part_end.push_back((int)parts.size());
  }
  h->d_apparts.ensure(std::max<size_t>(1, parts.size()) * sizeof(ApPart), st);
  if (!parts.empty())
    h2d_sync(h->d_apparts.p, parts.data(), parts.size() * sizeof(ApPart), st);
  h->d_upart.ensure(std::max<int64_t>(utot, 8) * 8, st);
  h->ap_wave_flops.assign(h->ap_wave_begin.size() - 1, 0.0);
  h->ap_wave_bytes.assign(h->ap_wave_begin.size() - 1, 0.0);
  for (size_t w = 0; w + 1 < h->ap_wave_begin.size(); ++w)
    for (int q = h->ap_wave_begin[w]; q < h->ap_wave_begin[w + 1]; ++q) {
      const NodeRec &rc = h->recs[q];
      double n = rc.m + rc.r;
      // one pass reads L^{-1} (lower half) and Z once: 2 flops / element read
      double elems = n * (n + 1) / 2 + n * rc.W;
      h->ap_wave_flops[w] += 2.0 * elems;
      h->ap_wave_bytes[w] += 8.0 * elems + 8.0 * 2 * (n + rc.W);
    }
  // 2-stage streaming ring: as large as fits (<= 2 x 48 KB), >= 2 columns per stage
  {
    size_t fixed = std::max(fwd, bwd) * 8 + 256;
    size_t room = fixed < (size_t)SMEM_LIMIT ? ((size_t)SMEM_LIMIT - fixed) / 2 : 0;
    size_t ch = std::min<size_t>(room, 48 * 1024) / 8;
    ch &= ~size_t(1);
    if (ch < 2 * max_col + 2)
      throw Err(LORASP_E_ARG, "apply: node record too large for the shared-memory apply kernel");
    h->ap_chunk = (int)ch;
    h->ap_fwd_smem = fwd * 8 + 2 * ch * 8 + 64;
    h->ap_y_smem = (fwd + 256) * 8;
    h->ap_bwd_smem = bwd * 8 + 2 * ch * 8 + 64;
    const size_t nwv = h->ap_wave_begin.size() - 1;
    h->ap_wave_ch.assign(nwv, (int)ch);
    h->ap_wave_fsm.assign(nwv, h->ap_fwd_smem);
    h->ap_wave_bsm.assign(nwv, h->ap_bwd_smem);
    for (size_t w = 0; w < nwv; ++w) {
        size_t wf = 0, wb = 0, wc = 2;
        for (int q = h->ap_wave_begin[w]; q < h->ap_wave_begin[w + 1]; ++q) {
          const NodeRec &rc = h->recs[q];
          const size_t n = rc.m + rc.r;
          wf = std::max(wf, (size_t)(rc.m + n + 2 * rc.W + 258));
          wb = std::max(wb, (size_t)(n + rc.W + 258));
          // one stage holds a whole part of the record (L^{-1} columns or Z)
          wc = std::max(wc, std::max<size_t>(2 * (size_t)rc.ld + 2,
                                             (size_t)rc.ld * std::max<size_t>(n, (size_t)rc.W)));
        }
        wc = std::min(wc, ch);
        // wide waves: smaller stages so that several CTAs share an SM (each
        // CTA's chain of bulk copies is latency bound; more of them in flight)
        {
          const int cnt = h->ap_wave_begin[w + 1] - h->ap_wave_begin[w];
          const int target = std::min(5, (cnt + 147) / 148);
          size_t ldmax = 2;
          for (int q = h->ap_wave_begin[w]; q < h->ap_wave_begin[w + 1]; ++q)
            ldmax = std::max(ldmax, (size_t)h->recs[q].ld);
          if (target > 2) {
            const size_t room = (size_t)SMEM_LIMIT / target;
            const size_t fix = std::max(wf, wb) * 8 + 256;
            if (room > fix) wc = std::min(wc, std::max<size_t>((room - fix) / 16, 2 * ldmax + 2));
          }
        }
        wc = (wc + 1) & ~size_t(1);
        if (h->debug) {
          double avg = 0;
          size_t mx = 0;
          for (int q = h->ap_wave_begin[w]; q < h->ap_wave_begin[w + 1]; ++q) {
            const NodeRec &rc = h->recs[q];
            const size_t e = (size_t)rc.ld * (rc.m + rc.r + rc.W);
            avg += e;
            mx = std::max(mx, e);
          }
          const int cnt = h->ap_wave_begin[w + 1] - h->ap_wave_begin[w];
          fprintf(stderr, "[lorasp] apply wave %zu: %d nodes, record doubles avg %.0f max %zu, chunk %zu, smem %zu / %zu\n",
                  w, cnt, avg / cnt, mx, wc, wf * 8 + 2 * wc * 8 + 64, wb * 8 + 2 * wc * 8 + 64);
        }
        h->ap_wave_ch[w] = (int)wc;
        h->ap_wave_fsm[w] = wf * 8 + 2 * wc * 8 + 64;
        h->ap_wave_bsm[w] = wb * 8 + 2 * wc * 8 + 64;
      }
  }
  // dataflow apply plan: the reader of every forward segment (the node whose RHS
  // range contains it), per reader its contributions in writer order, per node
  // the distinct readers / writers to notify
  h->ap_df_ok = false;
  if (!dist && !h->no_df && !an.empty()) {
    // the dataflow part: every node before the first split wave
    // (the top of the tree -- from the first wave holding a record of >= 1 MB of
    // Z after which every wave has <= 64 nodes -- stays wave launches, whose
    // split kernels spread such records over CTAs; one CTA would stream them)
    const int nwv = (int)h->ap_wave_split.size();
    int S = nwv;
    {
      int few = nwv;   // first wave of the suffix with <= 64 nodes per wave
      while (few > 0 && h->ap_wave_begin[few] - h->ap_wave_begin[few - 1] <= 64) --few;
      for (int w = few; w < nwv; ++w) {
        double zmax = 0;
        for (int q = h->ap_wave_begin[w]; q < h->ap_wave_begin[w + 1]; ++q)
          zmax = std::max(zmax, 8.0 * (an[q].m + an[q].r) * an[q].W);
        if (zmax >= 1024.0 * 1024) {
          S = w;
          break;
        }
      }
    }
    h->ap_df_wave = S;
    const int NA = (int)an.size();
    const int N = h->ap_wave_begin[S];
    std::vector<std::pair<int64_t, int>> rng;
    for (int q = 0; q < NA; ++q)
      if (an[q].m > 0) rng.push_back({an[q].off_s, q});
    std::sort(rng.begin(), rng.end());
    std::vector<int64_t> zoff(N);
    int64_t ztot = 0;
    for (int q = 0; q < N; ++q) {
      zoff[q] = ztot;
      ztot += an[q].W;
    }
    // task index of a reader: a dataflow node itself, or the flush task of a
    // wave-launched reader (indices N, N + 1, ...)
    std::vector<int> task_of(NA, -1), flush_node;
    for (int q = 0; q < N; ++q) task_of[q] = q;
    std::vector<std::vector<int>> Rl(N), Wl;
    std::vector<std::vector<ApContrib>> CT(N);
    Wl.resize(N);
    std::vector<int> nreal(N, 0);   // distinct dataflow readers (backward waits)
    bool ok = true;
    for (int p = 0; p < N && ok; ++p)
      for (int k = an[p].seg0; k < an[p].seg0 + an[p].nseg; ++k) {
        const ApSeg &Sg = as[k];
        auto it = std::upper_bound(rng.begin(), rng.end(), std::make_pair(Sg.voff, INT32_MAX));
        if (it == rng.begin()) { ok = false; break; }
        const int q = std::prev(it)->second;
        if (q <= p || Sg.voff + Sg.w > an[q].off_s + an[q].m) { ok = false; break; }
        if (task_of[q] < 0) {
          task_of[q] = N + (int)flush_node.size();
          flush_node.push_back(q);
          CT.emplace_back();
          Wl.emplace_back();
        }
        const int tq = task_of[q];
        CT[tq].push_back(ApContrib{zoff[p] + Sg.zc, (int)(Sg.voff - an[q].off_s), Sg.w});
        if (std::find(Rl[p].begin(), Rl[p].end(), tq) == Rl[p].end()) {
          Rl[p].push_back(tq);
          if (tq < N) ++nreal[p];
        }
        if (Wl[tq].empty() || Wl[tq].back() != p) Wl[tq].push_back(p);   // writers arrive in order
      }
    const int NT = N + (int)flush_node.size();
    if (ok && N > 0) {
      std::vector<ApDf> df(NT);
      std::vector<ApContrib> cl;
      std::vector<int> dl;
      size_t fmx = 0, bmx = 0;
      for (int q = 0; q < NT; ++q) {
        ApDf &d = df[q];
        d.node = q < N ? q : flush_node[q - N];
        d.fin = (int)Wl[q].size();
        if (q >= N) {
          d.c0 = (int)cl.size();
          d.nc = (int)CT[q].size();
          cl.insert(cl.end(), CT[q].begin(), CT[q].end());
          continue;
        }
        d.bin = nreal[q];
        d.c0 = (int)cl.size();
        d.nc = (int)CT[q].size();
        cl.insert(cl.end(), CT[q].begin(), CT[q].end());
        d.r0 = (int)dl.size();
        d.nr = (int)Rl[q].size();
        dl.insert(dl.end(), Rl[q].begin(), Rl[q].end());
        d.w0 = (int)dl.size();
        d.nwr = (int)Wl[q].size();
        dl.insert(dl.end(), Wl[q].begin(), Wl[q].end());
        d.zo = zoff[q];
        const size_t n = (size_t)an[q].m + an[q].r;
        fmx = std::max(fmx, (size_t)an[q].m + n + 258);   // rhs, y, partials
        bmx = std::max(bmx, n + (size_t)an[q].W + 258);   // u, x_T, partials
      }
      h->d_apdf.ensure(NT * sizeof(ApDf), st);
      h->d_apcontr.ensure(std::max<size_t>(1, cl.size()) * sizeof(ApContrib), st);
      h->d_apdfl.ensure(std::max<size_t>(1, dl.size()) * sizeof(int), st);
      h2d_sync(h->d_apdf.p, df.data(), NT * sizeof(ApDf), st);
      if (!cl.empty()) h2d_sync(h->d_apcontr.p, cl.data(), cl.size() * sizeof(ApContrib), st);
      if (!dl.empty()) h2d_sync(h->d_apdfl.p, dl.data(), dl.size() * sizeof(int), st);
      h->d_zob.ensure(std::max<int64_t>(ztot, 8) * 8, st);
      h->d_dfcnt.ensure((NT + 8) * sizeof(int), st);
      h->ap_df_nt = NT;
      // 2-stage ring per CTA sized for ~3 CTAs per SM (>= 2 columns per stage)
      // CTAs per SM: 4 when the leaf waves are several times wider than the GPU
      // (throughput: more bulk copies in flight), else 2 (larger stages, shorter
      // per-node chains) -- measured: cfg4 / cfg5 Krylov -6 % / -5 % at 4 vs 3,
      // cfg2 / cfg3 -6 % / -3 % at 2
      int wmax = 0;
      for (int w = 0; w < S; ++w) wmax = std::max(wmax, h->ap_wave_begin[w + 1] - h->ap_wave_begin[w]);
      const int dfo = wmax >= 4 * 148 ? 4 : 2;
      size_t ch = ((size_t)SMEM_LIMIT / dfo > std::max(fmx, bmx) * 8 + 256)
                      ? ((size_t)SMEM_LIMIT / dfo - std::max(fmx, bmx) * 8 - 256) / 16 : 0;
      ch = std::max(ch, 2 * max_col + 2);
      ch = std::min<size_t>(ch, 48 * 1024 / 8);
      ch = std::max(ch, 2 * max_col + 2);
      ch = (ch + 1) & ~size_t(1);
      h->ap_df_ch = (int)ch;
      h->ap_df_fsm = fmx * 8 + 2 * ch * 8 + 64;
      h->ap_df_bsm = bmx * 8 + 2 * ch * 8 + 64;
      if (h->ap_df_fsm <= (size_t)SMEM_LIMIT && h->ap_df_bsm <= (size_t)SMEM_LIMIT) {
        int dev = 0, nsm = 148, of = 1, ob = 1;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&of, k_apply_fwd_df, 256, h->ap_df_fsm));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ob, k_apply_bwd_df, 256, h->ap_df_bsm));
        h->ap_df_gf = std::max(1, std::min(NT, nsm * std::max(1, of)));
        h->ap_df_gb = std::max(1, std::min(N, nsm * std::max(1, ob)));
        h->ap_df_n = N;
        h->ap_df_ok = true;
      }
    }
    if (h->debug && !h->ap_df_ok) fprintf(stderr, "[lorasp] dataflow apply plan not built (ok=%d)\n", (int)ok);
  }
  h->d_apnodes.ensure(std::max<size_t>(1, an.size()) * sizeof(ApNode), st);
  h->d_apsegs.ensure(std::max<size_t>(1, as.size()) * sizeof(ApSeg), st);
  h2d_sync(h->d_apnodes.p, an.data(), an.size() * sizeof(ApNode), st);
  h2d_sync(h->d_apsegs.p, as.data(), as.size() * sizeof(ApSeg), st);
  std::vector<int64_t> perm(pl.n);
  for (int64_t q = 0; q < pl.n; ++q) perm[q] = voff[L][pl.leaf_of[q]] + pl.leaf_pos[q];
  h->d_perm.ensure(pl.n * sizeof(int64_t), st);
  h2d_sync(h->d_perm.p, perm.data(), pl.n * sizeof(int64_t), st);
  h->d_vec.ensure(std::max<int64_t>(tot, 8) * 8, st);
  h->d_b.ensure(pl.n * 8, st);
  h->d_x.ensure(pl.n * 8, st);
  h->factored = true;
  h->rank_cache = h->rnk;
  h->cache_valid = true;
  return true;
}

// One wave of Alg. 3 (fwd) or Alg. 4 (bwd): fused one-CTA-per-node kernel, or
// the split kernels (y / L part per node + Z column slices over CTAs).
void apply_wave(lorasp_ctx *h, int w, bool fwd, cudaStream_t s) {
  const ApNode *nodes = h->d_apnodes.as<ApNode>();
  const ApSeg *segs = h->d_apsegs.as<ApSeg>();
  const int b0 = h->ap_wave_begin[w], b1 = h->ap_wave_begin[w + 1];
  double *vec = h->d_vec.as<double>();
  if (!h->ap_wave_split[w]) {
    if (fwd) launch_k(k_apply_fwd, b1 - b0, 256, h->ap_wave_fsm[w], s, nodes + b0, segs, vec, h->ap_wave_ch[w]);
    else launch_k(k_apply_bwd, b1 - b0, 256, h->ap_wave_bsm[w], s, nodes + b0, segs, vec, h->ap_wave_ch[w]);
    return;
  }
  const ApPart *pall = h->d_apparts.as<ApPart>();
  const ApPart *parts = pall + h->ap_part_begin[w], *yparts = pall + h->ap_ypart_begin[w],
               *lparts = pall + h->ap_lpart_begin[w];
  const int np = h->ap_ypart_begin[w] - h->ap_part_begin[w], ny = h->ap_lpart_begin[w] - h->ap_ypart_begin[w],
            nl = h->ap_part_end[w] - h->ap_lpart_begin[w];
  if (fwd) {
    launch_k(k_apply_fwd_y, ny, 256, h->ap_y_smem, s, nodes, yparts, vec);
    launch_k(k_apply_fwd_z, np, 256, h->ap_fwd_smem, s, nodes, parts, segs, vec, h->ap_chunk);
  } else {
    launch_k(k_apply_bwd_z, np, 256, h->ap_bwd_smem, s, nodes, parts, segs, vec, h->d_upart.as<double>(), h->ap_chunk);
    launch_k(k_apply_bwd_l, nl, 256, h->ap_bwd_smem, s, nodes, lparts, h->d_upart.as<double>(), vec);
  }
}

// Alg. 3 (fwd) or Alg. 4 (bwd) as one persistent dataflow launch (single GPU)
void apply_df(lorasp_ctx *h, bool fwd, cudaStream_t s) {
  const int N = h->ap_df_n, NT = h->ap_df_nt, nw = (int)h->ap_wave_begin.size() - 1;
  int *cnt = h->d_dfcnt.as<int>(), *work = cnt + NT;
  if (fwd) {
    CK(cudaMemsetAsync(cnt, 0, (NT + 1) * sizeof(int), s));
    launch_k(k_apply_fwd_df, h->ap_df_gf, 256, h->ap_df_fsm, s, h->d_apnodes.as<ApNode>(), h->d_apdf.as<ApDf>(),
             h->d_apcontr.as<ApContrib>(), h->d_apdfl.as<int>(), N, NT, h->d_vec.as<double>(),
             h->d_zob.as<double>(), cnt, work, h->ap_df_ch);
    for (int w = h->ap_df_wave; w < nw; ++w) apply_wave(h, w, true, s);
  } else {
    for (int w = nw - 1; w >= h->ap_df_wave; --w) apply_wave(h, w, false, s);
    CK(cudaMemsetAsync(cnt, 0, (NT + 1) * sizeof(int), s));
    launch_k(k_apply_bwd_df, h->ap_df_gb, 256, h->ap_df_bsm, s, h->d_apnodes.as<ApNode>(), h->d_apdf.as<ApDf>(),
             h->d_apsegs.as<ApSeg>(), h->d_apdfl.as<int>(), N, h->d_vec.as<double>(), cnt, work, h->ap_df_ch);
  }
}

// x = Ã b on device buffers
void apply_dev(lorasp_ctx *h, const double *b, double *x, int64_t *counter) {
  cudaStream_t st = h->stream;
  const Plan &pl = h->plan;
  CK(cudaMemsetAsync(h->d_vec.p, 0, h->vec_len * 8, st));
  int ev = tbeg(h, K_VEC);
  launch_k(k_set_rhs, grid1(pl.n), 256, 0, st, b, h->d_perm.as<int64_t>(), pl.n, h->d_vec.as<double>());
  tend(h, ev, 0, 24.0 * pl.n);
  const ApNode *nodes = h->d_apnodes.as<ApNode>();
  const ApSeg *segs = h->d_apsegs.as<ApSeg>();
  const int nw = (int)h->ap_wave_begin.size() - 1;
  if (h->dist_world > 1) {
    // distributed apply: each rank runs the nodes it owns (their
    // records never left it); after every wave the vector segments written
    // there travel to every rank (distance-2 colouring: one writer per segment
    // per wave), so each rank enters the next wave with the full vector
    double *vec = h->d_vec.as<double>();
    auto exch = [&](const std::vector<std::vector<std::pair<int64_t, int64_t>>> &dl) {
      std::vector<DirtyList> dirty(h->dist_world);
      int64_t any = 0;
      for (int g = 0; g < h->dist_world; ++g)
        for (auto &pr : dl[g]) {
          dirty[g].push_back({vec + pr.first, pr.second});
          any += pr.second;
        }
      if (!any) return;
      const int64_t b0 = h->dist_bytes, c0 = h->dist_calls;
      dist_exchange(h, dirty);
      h->dist_apply_bytes += h->dist_bytes - b0;
      h->dist_apply_calls += h->dist_calls - c0;
      h->dist_bytes = b0;
      h->dist_calls = c0;
    };
    for (int w = 0; w < nw; ++w) {
      const int b0 = h->ap_wave_begin[w], no = h->ap_wave_nown[w];
      ev = tbeg(h, K_APPLY_FWD);
      if (no > 0) launch_k(k_apply_fwd, no, 256, h->ap_wave_fsm[w], st, nodes + b0, segs, vec, h->ap_wave_ch[w]);
      tend(h, ev, h->ap_wave_flops[w], h->ap_wave_bytes[w]);
      exch(h->ap_dirty_f[w]);
    }
    for (int w = nw - 1; w >= 0; --w) {
      const int b0 = h->ap_wave_begin[w], no = h->ap_wave_nown[w];
      ev = tbeg(h, K_APPLY_BWD);
      if (no > 0) launch_k(k_apply_bwd, no, 256, h->ap_wave_bsm[w], st, nodes + b0, segs, vec, h->ap_wave_ch[w]);
      tend(h, ev, h->ap_wave_flops[w], h->ap_wave_bytes[w]);
      exch(h->ap_dirty_b[w]);
    }
  } else if (!h->no_graph && nw > 0) {
    // Alg. 3 / Alg. 4 wave launches as one CUDA graph (per-class timing, when
    // requested for the apply classes, uses the launch-by-launch path below)
    // the graph stays valid across re-factorizations as long as every launch
    // parameter is unchanged (the node descriptors live in device memory)
    std::vector<int64_t> sig(h->ap_wave_begin.begin(), h->ap_wave_begin.end());
    sig.push_back((int64_t)h->ap_fwd_smem);
    sig.push_back((int64_t)h->ap_bwd_smem);
    sig.push_back(h->ap_chunk);
    sig.push_back((int64_t)(intptr_t)nodes);
    sig.push_back((int64_t)(intptr_t)segs);
    sig.push_back((int64_t)(intptr_t)h->d_vec.p);
    sig.insert(sig.end(), h->ap_part_begin.begin(), h->ap_part_begin.end());
    sig.insert(sig.end(), h->ap_ypart_begin.begin(), h->ap_ypart_begin.end());
    sig.insert(sig.end(), h->ap_lpart_begin.begin(), h->ap_lpart_begin.end());
    sig.insert(sig.end(), h->ap_part_end.begin(), h->ap_part_end.end());
    sig.insert(sig.end(), h->ap_wave_split.begin(), h->ap_wave_split.end());
    sig.insert(sig.end(), h->ap_wave_ch.begin(), h->ap_wave_ch.end());
    for (size_t v : h->ap_wave_fsm) sig.push_back((int64_t)v);
    for (size_t v : h->ap_wave_bsm) sig.push_back((int64_t)v);
    sig.push_back((int64_t)(intptr_t)h->d_apparts.p);
    sig.push_back((int64_t)(intptr_t)h->d_upart.p);
    sig.push_back(h->ap_df_ok);
    sig.push_back(h->ap_df_n);
    sig.push_back(h->ap_df_nt);
    sig.push_back(h->ap_df_wave);
    sig.push_back(h->ap_df_ch);
    sig.push_back(h->ap_df_gf);
    sig.push_back(h->ap_df_gb);
    sig.push_back((int64_t)h->ap_df_fsm);
    sig.push_back((int64_t)h->ap_df_bsm);
    for (DevBuf *b : {&h->d_apdf, &h->d_apcontr, &h->d_apdfl, &h->d_zob, &h->d_dfcnt})
      sig.push_back((int64_t)(intptr_t)b->p);
    if (h->ap_graph && sig != h->ap_graph_sig) {
      CK(cudaGraphExecDestroy(h->ap_graph));
      h->ap_graph = nullptr;
    }
    if (!h->ap_graph) {
      h->ap_graph_sig = sig;
      // captured on a private stream (the library stream may be the legacy
      // default stream, which cannot be captured); launched on the library stream
      cudaStream_t cs;
      CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      if (h->ap_df_ok) {
        apply_df(h, true, cs);
        apply_df(h, false, cs);
      } else {
        for (int w = 0; w < nw; ++w) apply_wave(h, w, true, cs);
        for (int w = nw - 1; w >= 0; --w) apply_wave(h, w, false, cs);
      }
      const cudaError_t ce = cudaStreamEndCapture(cs, &g);
      cudaStreamDestroy(cs);
      CK(ce);
      CK(cudaGraphInstantiate(&h->ap_graph, g, 0));
      CK(cudaGraphDestroy(g));
    }
    // timing: one event pair around the graph, accounted to apply_fwd as 2 nw
    // launches (both passes; per-launch averages stay meaningful)
    int evg = -1;
    if (h->timing && (((h->timing_mask >> K_APPLY_FWD) & 1u) || ((h->timing_mask >> K_APPLY_BWD) & 1u)))
      evg = tbeg_force(h, K_APPLY_FWD);
    CK(cudaGraphLaunch(h->ap_graph, st));
    if (evg >= 0) {
      double fl = 0, by = 0;
      for (int w = 0; w < nw; ++w) {
        fl += 2 * h->ap_wave_flops[w];
        by += 2 * h->ap_wave_bytes[w];
      }
      tend(h, evg, fl, by);
      int nl = 2 * nw;
      if (h->ap_df_ok) {   // two dataflow launches + the trailing waves' launches
        nl = 2;
        for (int w = h->ap_df_wave; w < nw; ++w) nl += h->ap_wave_split[w] ? 4 : 2;
      }
      h->pend[evg].nl = nl;
    }
  } else if (h->ap_df_ok) {
    double fl = 0, by = 0;
    for (int w = 0; w < nw; ++w) {
      fl += h->ap_wave_flops[w];
      by += h->ap_wave_bytes[w];
    }
    ev = tbeg(h, K_APPLY_FWD);
    apply_df(h, true, st);
    tend(h, ev, fl, by);
    ev = tbeg(h, K_APPLY_BWD);
    apply_df(h, false, st);
    tend(h, ev, fl, by);
  } else {
  for (int w = 0; w < nw; ++w) {
    ev = tbeg(h, K_APPLY_FWD);
    apply_wave(h, w, true, st);
    tend(h, ev, h->ap_wave_flops[w], h->ap_wave_bytes[w]);
  }
  for (int w = nw - 1; w >= 0; --w) {
    ev = tbeg(h, K_APPLY_BWD);
    apply_wave(h, w, false, st);
    tend(h, ev, h->ap_wave_flops[w], h->ap_wave_bytes[w]);
  }
  }
  ev = tbeg(h, K_VEC);
  launch_k(k_get_x, grid1(pl.n), 256, 0, st, h->d_vec.as<double>(), h->d_perm.as<int64_t>(), pl.n, x);
  tend(h, ev, 0, 24.0 * pl.n);
  *counter += 2 * nw + 2;
  CK(cudaGetLastError());
}

double dot_dev(lorasp_ctx *h, const double *a, const double *b) {
  cudaStream_t st = h->stream;
  int ev = tbeg(h, K_DOT);
  launch_k(k_dot_partial, DOT_BLOCKS, 256, 0, st, h->plan.n, a, b, h->d_dotpart.as<double>());
  launch_k(k_dot_final, 1, 256, 0, st, h->d_dotpart.as<double>(), DOT_BLOCKS,
                                 h->d_dotpart.as<double>() + DOT_BLOCKS);
  tend(h, ev, 2.0 * h->plan.n, 16.0 * h->plan.n);
  CK(cudaMemcpyAsync(h->h_dot, h->d_dotpart.as<double>() + DOT_BLOCKS, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  h->launches_krylov += 2;
  return h->h_dot[0];
}

// dot product into a device scalar (no host round trip)
void dot_dev_to(lorasp_ctx *h, const double *a, const double *b, double *out) {
  cudaStream_t st = h->stream;
  int ev = tbeg(h, K_DOT);
  launch_k(k_dot_partial, DOT_BLOCKS, 256, 0, st, h->plan.n, a, b, h->d_dotpart.as<double>());
  launch_k(k_dot_final, 1, 256, 0, st, h->d_dotpart.as<double>(), DOT_BLOCKS, out);
  tend(h, ev, 2.0 * h->plan.n, 16.0 * h->plan.n);
  h->launches_krylov += 2;
}

void spmv_dev(lorasp_ctx *h, const double *x, double *y) {
  const Plan &pl = h->plan;
  int ev = tbeg(h, K_SPMV);
  launch_k(k_spmv, grid1(pl.n), 256, 0, h->stream, pl.n, h->d_rowptr.as<int64_t>(), h->d_colidx.as<int64_t>(),
                                            h->d_values.as<double>(), x, y);
  tend(h, ev, 2.0 * pl.nnz, 20.0 * pl.nnz + 16.0 * pl.n);
  ++h->launches_krylov;
}

void axpby(lorasp_ctx *h, double a, const double *x, double b, double *y) {
  int ev = tbeg(h, K_VEC);
  launch_k(k_axpby, grid1(h->plan.n), 256, 0, h->stream, h->plan.n, a, x, b, y);
  tend(h, ev, 3.0 * h->plan.n, 24.0 * h->plan.n);
  ++h->launches_krylov;
}

// preconditioned CG (P:l.652; readings Z21/Z24/Z27); device vectors b, x
int pcg_dev(lorasp_ctx *h, const double *b, double *x, double tol, int maxit, int *iters, double *relres) {
  const int64_t n = h->plan.n;
  h->d_kry.ensure(4 * n * 8, h->stream);
  double *r = h->d_kry.as<double>(), *z = r + n, *p = z + n, *q = p + n;
  cudaStream_t st = h->stream;
  CK(cudaMemsetAsync(x, 0, n * 8, st));
  CK(cudaMemcpyAsync(r, b, n * 8, cudaMemcpyDeviceToDevice, st));
  double nb = std::sqrt(dot_dev(h, b, b));
  if (nb == 0.0) {
    if (iters) *iters = 0;
    if (relres) *relres = 0;
    return LORASP_OK;
  }
  apply_dev(h, r, z, &h->launches_krylov);
  CK(cudaMemcpyAsync(p, z, n * 8, cudaMemcpyDeviceToDevice, st));
  // device scalars: rz (two slots, alternating), pq, rr, breakdown flag
  double *sc = h->d_dotpart.as<double>() + DOT_BLOCKS + 8;
  double *rz_cur = sc, *rz_nxt = sc + 1, *d_pq = sc + 2, *d_rr = sc + 3, *d_flag = sc + 4;
  CK(cudaMemsetAsync(d_flag, 0, 8, st));
  dot_dev_to(h, r, z, rz_cur);
  int it = 0;
  bool conv = false;
  for (it = 1; it <= maxit; ++it) {
    spmv_dev(h, p, q);
    dot_dev_to(h, p, q, d_pq);
    int ev = tbeg(h, K_VEC);
    k_pcg_update<<<grid1(n), 256, 0, st>>>(n, rz_cur, d_pq, p, q, x, r, d_flag);   // plain launch (see gmres)
    tend(h, ev, 4.0 * n, 48.0 * n);
    ++h->launches_krylov;
    dot_dev_to(h, r, r, d_rr);
    CK(cudaMemcpyAsync(h->h_dot, d_pq, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));   // pq, rr, flag
    CK(cudaStreamSynchronize(st));
    if (h->h_dot[2] != 0.0) {
      it -= 1;
      break;  // breakdown (reading Z24): x, r were left unchanged
    }
    const double rel = std::sqrt(h->h_dot[1]) / nb;
    if (rel <= tol) {
      conv = true;
      break;
    }
    apply_dev(h, r, z, &h->launches_krylov);
    dot_dev_to(h, r, z, rz_nxt);
    ev = tbeg(h, K_VEC);
    k_pcg_dir<<<grid1(n), 256, 0, st>>>(n, rz_nxt, rz_cur, z, p);   // plain launch (see gmres)
    tend(h, ev, 2.0 * n, 24.0 * n);
    ++h->launches_krylov;
    std::swap(rz_cur, rz_nxt);
  }
  if (it > maxit) it = maxit;
  // true residual
  spmv_dev(h, x, q);
  launch_k(k_sub, grid1(n), 256, 0, st, n, b, q, r);
  ++h->launches_krylov;
  double rr = std::sqrt(dot_dev(h, r, r)) / nb;
  if (iters) *iters = it;
  if (relres) *relres = rr;
  return (conv || rr <= tol) ? LORASP_OK : LORASP_NOT_CONVERGED;
}

// right-preconditioned GMRES(restart) with MGS + Givens (reading Z21)
int gmres_dev(lorasp_ctx *h, const double *b, double *x, double tol, int restart, int maxit, int *iters,
              double *relres) {
  const int64_t n = h->plan.n;
  cudaStream_t st = h->stream;
  h->d_kry.ensure((size_t)(2 * restart + 3) * n * 8, h->stream);
  double *Vb = h->d_kry.as<double>();            // (restart+1) x n
  double *Zb = Vb + (int64_t)(restart + 1) * n;  // restart x n
  double *w = Zb + (int64_t)restart * n;         // n
  double *r = w + n;                             // n
  CK(cudaMemsetAsync(x, 0, n * 8, st));
  double nb = std::sqrt(dot_dev(h, b, b));
  if (nb == 0.0) {
    if (iters) *iters = 0;
    if (relres) *relres = 0;
    return LORASP_OK;
  }
  int it = 0;
  bool conv = false;
  std::vector<double> H((restart + 1) * restart), cs(restart), sn(restart), g(restart + 1);
  while (it < maxit && !conv) {
    spmv_dev(h, x, w);
    launch_k(k_sub, grid1(n), 256, 0, st, n, b, w, r);
    ++h->launches_krylov;
    double beta = std::sqrt(dot_dev(h, r, r));
    if (beta / nb <= tol) {
      conv = true;
      break;
    }
    axpby(h, 1.0 / beta, r, 0.0, Vb);
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int k_used = 0;
    for (int k = 0; k < restart && it < maxit; ++k) {
      apply_dev(h, Vb + (int64_t)k * n, Zb + (int64_t)k * n, &h->launches_krylov);
      spmv_dev(h, Zb + (int64_t)k * n, w);
      // modified Gram-Schmidt with the coefficients kept on the device; one
      // host round trip per iteration for the Hessenberg column
      double *hcol = h->d_dotpart.as<double>() + DOT_BLOCKS + 16;   // k + 2 <= 1002 slots
      for (int j = 0; j <= k; ++j) {
        dot_dev_to(h, w, Vb + (int64_t)j * n, hcol + j);
        int ev = tbeg(h, K_VEC);
        // plain launch (no PDL): a PDL launch of this device-scalar consumer right
        // after k_dot_final produced wrong Gram-Schmidt updates (measured; cause
        // not isolated), so the scalar consumers are fully stream-ordered
        k_axpy_dev<<<grid1(n), 256, 0, st>>>(n, hcol + j, -1.0, Vb + (int64_t)j * n, w);
        tend(h, ev, 2.0 * n, 24.0 * n);
        ++h->launches_krylov;
      }
      dot_dev_to(h, w, w, hcol + k + 1);
      CK(cudaMemcpyAsync(h->h_dot, hcol, (size_t)(k + 2) * sizeof(double), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (int j = 0; j <= k; ++j) H[j + k * (restart + 1)] = h->h_dot[j];
      double hn = std::sqrt(h->h_dot[k + 1]);
      H[k + 1 + k * (restart + 1)] = hn;
      for (int j = 0; j < k; ++j) {
        double a = H[j + k * (restart + 1)], bb = H[j + 1 + k * (restart + 1)];
        H[j + k * (restart + 1)] = cs[j] * a + sn[j] * bb;
        H[j + 1 + k * (restart + 1)] = -sn[j] * a + cs[j] * bb;
      }
      double a = H[k + k * (restart + 1)], bb = H[k + 1 + k * (restart + 1)];
      double den = std::hypot(a, bb);
      cs[k] = den == 0 ? 1.0 : a / den;
      sn[k] = den == 0 ? 0.0 : bb / den;
      H[k + k * (restart + 1)] = cs[k] * a + sn[k] * bb;
      H[k + 1 + k * (restart + 1)] = 0;
      g[k + 1] = -sn[k] * g[k];
      g[k] = cs[k] * g[k];
      ++it;
      k_used = k + 1;
      if (std::fabs(g[k + 1]) / nb <= tol) {
        conv = true;
        break;
      }
      if (hn == 0) break;
      if (k + 1 < restart || true) axpby(h, 1.0 / hn, w, 0.0, Vb + (int64_t)(k + 1) * n);
    }
    // y = H^{-1} g (upper triangular)
    std::vector<double> y(k_used);
    for (int j = k_used - 1; j >= 0; --j) {
      double s = g[j];
      for (int q = j + 1; q < k_used; ++q) s -= H[j + q * (restart + 1)] * y[q];
      y[j] = s / H[j + j * (restart + 1)];
    }
    for (int j = 0; j < k_used; ++j) axpby(h, y[j], Zb + (int64_t)j * n, 1.0, x);
  }
  spmv_dev(h, x, w);
  launch_k(k_sub, grid1(n), 256, 0, st, n, b, w, r);
  ++h->launches_krylov;
  double rr = std::sqrt(dot_dev(h, r, r)) / nb;
  if (iters) *iters = it;
  if (relres) *relres = rr;
  return (rr <= tol) ? LORASP_OK : LORASP_NOT_CONVERGED;
}


// Rank-predicted re-factorization.  Once a predicted sweep has been verified
// (replay_hits > 0), the next one is captured into a CUDA graph with its task
// descriptors resident in fg_desc; later calls copy the values and launch the
// graph (no host task building, no staging copies, no launch gaps), then
// verify the logged ranks as usual.  A capture that cannot complete (a buffer
// would grow, an API refuses capture) falls back to the plain predicted sweep.
bool graph_launch(lorasp_ctx *h, const double *values) {
  copy_values(h, values);
  CK(cudaGraphLaunch(h->fgraph, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  ++h->fg_launches;
  h->fgraph_used = true;
  h->f_doubles = h->fg_fdoubles;
  h->t_host_ms = 0;
  h->t_sync_ms = 0;
  h->pend.insert(h->pend.end(), h->fg_pend.begin(), h->fg_pend.end());
  tflush(h);
  if (!replay_check(h, h->fg_rlog)) {
    cudaGraphExecDestroy(h->fgraph);
    h->fgraph = nullptr;
    return false;
  }
  status_check(h);
  h->factored = true;
  return true;
}

bool factor_replay(lorasp_ctx *h, const double *values) {
  h->fgraph_used = false;
  const unsigned tsig = h->timing ? h->timing_mask : 0u;
  const bool want = !h->no_fgraph && !h->debug && h->replay_hits > 0 && h->fg_failures < 2;
  if (want && h->fgraph && h->fg_gen == g_alloc_gen.load() && h->fg_timing == tsig) return graph_launch(h, values);
  if (!want) return factor_impl(h, values, true);
  if (h->fgraph) {
    cudaGraphExecDestroy(h->fgraph);
    h->fgraph = nullptr;
  }
  // record
  CK(cudaStreamSynchronize(h->stream));
  h->fg_desc.ensure(h->stg.total + h->stg.total / 8 + (size_t(1) << 20), h->stream);
  h->stg.gd = h->fg_desc.as<char>();
  h->stg.gd_cap = h->fg_desc.cap;
  h->stg.blob.clear();
  h->stg.cap_overflow = false;
  h->pend.clear();
  cudaGraph_t g = nullptr;
  bool ok = false;
  CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeRelaxed));
  h->stg.cap_mode = true;
  try {
    ok = factor_impl(h, values, true, true);
  } catch (const CaptureAbort &) {
    ok = false;
  } catch (const Err &) {   // an API that refuses capture: the plain sweep below decides
    ok = false;
  } catch (...) {
    h->stg.cap_mode = false;
    cudaStreamEndCapture(h->stream, &g);
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    h->s1_pending = false;
    h->pend.clear();
    throw;
  }
  h->stg.cap_mode = false;
  h->s1_pending = false;   // the capture's events only ordered nodes
  cudaError_t e = cudaStreamEndCapture(h->stream, &g);
  if (e == cudaSuccess && ok && !h->stg.cap_overflow && g) e = cudaGraphInstantiate(&h->fgraph, g, 0);
  else if (e == cudaSuccess) e = cudaErrorUnknown;
  if (g) cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    cudaGetLastError();
    h->fgraph = nullptr;
    ++h->fg_failures;
    h->pend.clear();
    return factor_impl(h, values, true);
  }
  h2d_sync(h->fg_desc.p, h->stg.blob.data(), h->stg.blob.size(), h->stream);
  h->fg_gen = g_alloc_gen.load();
  h->fg_timing = tsig;
  h->fg_pend = h->pend;
  h->pend.clear();
  ++h->fg_captures;
  h->fg_fdoubles = h->f_doubles;
  return graph_launch(h, values);
}

template <class F>
int guarded(lorasp_ctx *h, F &&f) {
  if (!h) return LORASP_E_ARG;
  try {
    return f();
  } catch (const Err &e) {
    h->last_error = e.msg;
    return e.code;
  } catch (const std::exception &e) {
    h->last_error = e.what();
    return LORASP_E_ARG;
  }
}

}  // namespace

extern "C" {

// forget everything a previous sweep cached for the current plan / pivot mode
void reset_sweep_state(lorasp_ctx *h) {
  CK(cudaDeviceSynchronize());
  h->cache_valid = false;
  h->factored = false;
  if (h->fgraph) {
    cudaGraphExecDestroy(h->fgraph);
    h->fgraph = nullptr;
  }
  if (h->ap_graph) {
    cudaGraphExecDestroy(h->ap_graph);
    h->ap_graph = nullptr;
  }
  h->ap_graph_sig.clear();
  h->s1_pending = false;
  h->pend.clear();
  h->stg.reset();
  CK(cudaMemsetAsync(h->d_status.p, 0, 64, h->stream));
  CK(cudaStreamSynchronize(h->stream));
}

// reading Z12: the SPD path's signed Cholesky met a non-positive pivot (the
// approximation broke definiteness).  The handle is re-planned on the general
// path (both block orientations, stacks [A; B]) with partial pivoting, and the
// sweep re-runs there; counted in the stats (spd_fallbacks).
void replan_general(lorasp_ctx *h, const char *why) {
  const Plan &old = h->plan;
  Plan np;
  std::string err;
  const int rc = build_plan(np, old.n, old.row_ptr.data(), old.col_idx.data(), h->an_dim,
                            h->an_coords.empty() ? nullptr : h->an_coords.data(), h->an_leaf, old.depth, old.eps,
                            old.flags & ~(unsigned)LORASP_SPD, err);
  if (rc != 0) throw Err(LORASP_E_PATTERN, "re-plan for the LU fallback failed: " + err);
  h->plan = std::move(np);
  h->dest_ready = false;
  h->leaf_soff.clear();
  h->piv_maxn_hint = 0;
  h->piv_cnt_hint = 0;
  h->eig_clmax_hint = h->eig_bigmax_hint = h->eig_regmax_hint = 0;
  for (int &x : h->eig_cl_wave_n) x = 0;
  h->rank_cache.clear();
  h->lu_pivot = true;
  ++h->spd_fallbacks;
  h->spd_fallback_node = why;
}

int lorasp_analyze(int64_t n, const int64_t *row_ptr, const int64_t *col_idx, int dim, const double *coords,
                   int leaf_size, int depth, double eps, unsigned flags, int device, lorasp_handle *out) {
  if (!out) return LORASP_E_ARG;
  *out = nullptr;
  if ((flags & LORASP_FROBENIUS) && (flags & LORASP_RRQR)) return LORASP_E_ARG;   // f2 is an SVD rule
  auto *h = new lorasp_ctx();
  h->device = device;
  std::string err;
  int rc = build_plan(h->plan, n, row_ptr, col_idx, dim, coords, leaf_size, depth, eps, flags, err);
  if (rc != 0) {
    delete h;
    return rc == -1 ? LORASP_E_ARG : LORASP_E_PATTERN;
  }
  if (coords && dim > 0) h->an_coords.assign(coords, coords + n * dim);
  h->an_dim = dim;
  h->an_leaf = leaf_size;
  *out = h;
  return LORASP_OK;
}

int lorasp_factor(lorasp_handle h, const double *values) {
  return guarded(h, [&]() {
    if (!values) return (int)LORASP_E_ARG;
    CK(cudaSetDevice(h->device));
    auto t0 = std::chrono::steady_clock::now();
    h->f_doubles = 0;
    // the sweep runs on the library's high-priority stream (ordered after the
    // caller's stream), so that the low-priority overlap work (split pivots)
    // only takes SMs the sweep leaves idle; the call returns synchronised
    ensure_mem(h);
    cudaStream_t user = h->stream;
    CK(cudaEventRecord(h->ev_u, user));
    CK(cudaStreamWaitEvent(h->stream_hi, h->ev_u, 0));
    h->stream = h->stream_hi;
    try {
      for (int attempt = 0;; ++attempt) {
        try {
          bool ok = false;
          h->replay_used = false;
          if (h->cache_valid && !h->no_replay && h->dist_world == 1) {
            ok = factor_replay(h, values);
            h->replay_used = ok;
          }
          if (!ok) {
            if (h->fgraph) {   // built for the old ranks
              cudaGraphExecDestroy(h->fgraph);
              h->fgraph = nullptr;
            }
            h->fgraph_used = false;
            factor_impl(h, values, false);
          }
          break;
        } catch (const Err &e) {
          if (attempt >= 2) throw;
          const bool lu = !(h->plan.flags & LORASP_SPD);
          if (e.code == LORASP_NEED_PIVOT && lu && !h->lu_pivot) {
            h->lu_pivot = true;   // re-run the sweep with partial pivoting
            ++h->lu_pivot_switches;
          } else if (e.code == LORASP_E_SINGULAR_PIVOT && !lu && h->dist_world == 1) {
            replan_general(h, e.msg.c_str());   // Z12: signed Cholesky failed -> LU path
          } else {
            throw;
          }
          reset_sweep_state(h);
        }
      }
    } catch (...) {
      h->cache_valid = false;
      cudaStreamSynchronize(h->stream_hi);
      h->stream = user;
      throw;
    }
    h->stream = user;
    h->t_factor_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return (int)LORASP_OK;
  });
}

int lorasp_apply(lorasp_handle h, const double *b, double *x) {
  return guarded(h, [&]() {
    if (!b || !x || b == x) return (int)LORASP_E_ARG;
    if (!h->factored) return (int)LORASP_E_STATE;
    CK(cudaSetDevice(h->device));
    const int64_t n = h->plan.n;
    h->launches_apply = 0;
    if (is_device_ptr(b)) {
      apply_dev(h, b, x, &h->launches_apply);
      CK(cudaStreamSynchronize(h->stream));
    } else {
      CK(cudaMemcpyAsync(h->d_b.p, b, n * 8, cudaMemcpyHostToDevice, h->stream));
      apply_dev(h, h->d_b.as<double>(), h->d_x.as<double>(), &h->launches_apply);
      CK(cudaMemcpyAsync(x, h->d_x.p, n * 8, cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
    }
    tflush(h);
    return (int)LORASP_OK;
  });
}

int lorasp_krylov_ex(lorasp_handle h, const double *b, double *x, double tol, int method, int restart,
                     int max_it, int *iters, double *relres) {
  return guarded(h, [&]() {
    if (!b || !x || b == x || tol < 0 || max_it < 0) return (int)LORASP_E_ARG;
    if (!h->factored) return (int)LORASP_E_STATE;
    CK(cudaSetDevice(h->device));
    if (restart <= 0) restart = 50;
    if (restart > 1000) return (int)LORASP_E_ARG;
    const int64_t n = h->plan.n;
    h->launches_krylov = 0;
    bool dev = is_device_ptr(b);
    const double *bd = b;
    double *xd = x;
    if (!dev) {
      CK(cudaMemcpyAsync(h->d_b.p, b, n * 8, cudaMemcpyHostToDevice, h->stream));
      bd = h->d_b.as<double>();
      xd = h->d_x.as<double>();
    }
    int rc = (method == LORASP_CG) ? pcg_dev(h, bd, xd, tol, max_it, iters, relres)
                                   : gmres_dev(h, bd, xd, tol, restart, max_it, iters, relres);
    if (!dev) CK(cudaMemcpyAsync(x, xd, n * 8, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    tflush(h);
    return rc;
  });
}

// Eq. GMRES_residual (P:l.665-669): ||Ã b - Ã A x||_2 / ||Ã b||_2, all on the device
// (SpMV, two preconditioner applications, dot products in the library's kernels)
int lorasp_paper_residual(lorasp_handle h, const double *b, const double *x, double *out) {
  return guarded(h, [&]() {
    if (!b || !x || !out) return (int)LORASP_E_ARG;
    if (!h->factored) return (int)LORASP_E_STATE;
    CK(cudaSetDevice(h->device));
    const int64_t n = h->plan.n;
    h->d_kry.ensure(6 * n * 8, h->stream);
    double *w = h->d_kry.as<double>(), *ab = w + n, *aax = ab + n, *bd = aax + n, *xd = bd + n, *ax = xd + n;
    cudaStream_t st = h->stream;
    const bool dev = is_device_ptr(b) && is_device_ptr(x);
    if (!dev) {
      CK(cudaMemcpyAsync(bd, b, n * 8, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(xd, x, n * 8, cudaMemcpyHostToDevice, st));
      b = bd;
      x = xd;
    }
    h->launches_krylov = 0;
    apply_dev(h, b, ab, &h->launches_krylov);            // Ã b
    spmv_dev(h, x, ax);                                  // A x
    apply_dev(h, ax, aax, &h->launches_krylov);          // Ã A x
    launch_k(k_sub, grid1(n), 256, 0, st, n, ab, aax, w);
    const double num = dot_dev(h, w, w), den = dot_dev(h, ab, ab);
    *out = den > 0.0 ? std::sqrt(num / den) : 0.0;
    tflush(h);
    return (int)LORASP_OK;
  });
}

int lorasp_gmres(lorasp_handle h, const double *b, double *x, double tol) {
  return lorasp_krylov_ex(h, b, x, tol, LORASP_GMRES, 50, 500, nullptr, nullptr);
}

int lorasp_set_stream(lorasp_handle h, void *s) {
  if (!h) return LORASP_E_ARG;
  h->stream = reinterpret_cast<cudaStream_t>(s);
  return LORASP_OK;
}

int lorasp_set_dist(lorasp_handle h, int rank, int world, lorasp_coll_fn fn, void *user) {
  if (!h) return LORASP_E_ARG;
  if (world < 1 || world > 32 || (world & (world - 1)) != 0 || rank < 0 || rank >= world) return LORASP_E_ARG;
  int l0 = 0;
  while ((1 << l0) < world) ++l0;
  if (world > 1 && (!fn || h->plan.depth - 1 < l0)) return LORASP_E_ARG;
  h->dist_rank = world > 1 ? rank : 0;
  h->dist_world = world;
  h->dist_l0 = l0;
  h->dist_fn = world > 1 ? fn : nullptr;
  h->dist_user = user;
  h->cache_valid = false;
  h->slot_readers.clear();
  if (h->nccl) {
    if (const NcclApi *api = nccl_api()) api->CommDestroy(h->nccl);
    h->nccl = nullptr;
  }
  return LORASP_OK;
}

int lorasp_nccl_unique_id(void *id_out) {
  if (!id_out) return LORASP_E_ARG;
  const NcclApi *api = nccl_api();
  if (!api) return LORASP_E_NCCL;
  ncclUniqueId id;
  if (api->GetUniqueId(&id) != ncclSuccess) return LORASP_E_NCCL;
  std::memcpy(id_out, &id, sizeof(id));
  return LORASP_OK;
}

int lorasp_set_dist_nccl(lorasp_handle h, int rank, int world, const void *unique_id) {
  return guarded(h, [&]() {
    if (world < 1 || world > 32 || (world & (world - 1)) != 0 || rank < 0 || rank >= world || !unique_id)
      return (int)LORASP_E_ARG;
    int l0 = 0;
    while ((1 << l0) < world) ++l0;
    if (world > 1 && h->plan.depth - 1 < l0) return (int)LORASP_E_ARG;
    const NcclApi *api = nccl_api();
    if (!api) return (int)LORASP_E_NCCL;
    CK(cudaSetDevice(h->device));
    if (h->nccl) {
      api->CommDestroy(h->nccl);
      h->nccl = nullptr;
    }
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    ncclComm_t comm = nullptr;
    NCK(api->CommInitRank(&comm, world, id, rank));
    h->nccl = comm;
    h->dist_rank = world > 1 ? rank : 0;
    h->dist_world = world;
    h->dist_l0 = l0;
    h->dist_fn = nullptr;
    h->dist_user = nullptr;
    h->dist_send = h->dist_recv = nullptr;
    h->dist_send_cap = h->dist_recv_cap = 0;
    h->cache_valid = false;
    h->slot_readers.clear();
    return (int)LORASP_OK;
  });
}

// NCCL plumbing check on one device: a 1-rank communicator from a fresh unique
// id, all-gather and int32 max-reduce of `n` values through the library's
// transport calls; returns LORASP_OK when the results are the inputs.
int lorasp_test_nccl(int device, int n) {
  try {
    const NcclApi *api = nccl_api();
    if (!api || n <= 0) return LORASP_E_NCCL;
    CK(cudaSetDevice(device));
    ncclUniqueId id;
    NCK(api->GetUniqueId(&id));
    ncclComm_t comm;
    NCK(api->CommInitRank(&comm, 1, id, 0));
    int *d;
    CK(cudaMalloc(&d, 3 * (size_t)n * sizeof(int)));
    std::vector<int> hv(n);
    for (int i = 0; i < n; ++i) hv[i] = 3 * i - 7;
    CK(cudaMemcpy(d, hv.data(), n * sizeof(int), cudaMemcpyHostToDevice));
    NCK(api->AllGather(d, d + n, (size_t)n * sizeof(int), ncclUint8, comm, 0));
    NCK(api->AllReduce(d, d + 2 * n, (size_t)n, ncclInt32, ncclMax, comm, 0));
    CK(cudaDeviceSynchronize());
    std::vector<int> out(3 * (size_t)n);
    CK(cudaMemcpy(out.data(), d, 3 * (size_t)n * sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(d);
    api->CommDestroy(comm);
    for (int i = 0; i < n; ++i)
      if (out[n + i] != hv[i] || out[2 * n + i] != hv[i]) return LORASP_E_NCCL;
    return LORASP_OK;
  } catch (const Err &e) {
    return e.code;
  }
}

int lorasp_dist_counts(lorasp_handle h, int64_t *counts, int cap) {
  if (!h || !counts) return LORASP_E_ARG;
  const int n = (int)h->a2a_counts.size();
  if (cap < n) return LORASP_E_ARG;
  std::copy(h->a2a_counts.begin(), h->a2a_counts.end(), counts);
  return n;
}

int lorasp_set_dist_buffers(lorasp_handle h, void *send, int64_t send_cap, void *recv, int64_t recv_cap) {
  if (!h || send_cap < 0 || recv_cap < 0) return LORASP_E_ARG;
  h->dist_send = send;
  h->dist_send_cap = send ? send_cap : 0;
  h->dist_recv = recv;
  h->dist_recv_cap = recv ? recv_cap : 0;
  return LORASP_OK;
}

int lorasp_dist_owner(int level, int c, int world) {
  if (level < 1 || c < 0 || world < 1 || (world & (world - 1)) != 0) return -1;
  int l0 = 0;
  while ((1 << l0) < world) ++l0;
  return dist_owner_of(level, c, l0);
}

int lorasp_set_timing(lorasp_handle h, int enable) {
  return guarded(h, [&]() {
    CK(cudaSetDevice(h->device));
    h->timing = enable != 0;
    h->timing_mask = (unsigned)enable;
    for (auto &k : h->kst) k = KStat();
    h->pend.clear();
    return (int)LORASP_OK;
  });
}

int lorasp_get_depth(lorasp_handle h, int *depth) {
  if (!h || !depth) return LORASP_E_ARG;
  *depth = h->plan.depth;
  return LORASP_OK;
}

int lorasp_get_level_order(lorasp_handle h, int level, int *order, int *wave, int cap) {
  if (!h || level < 1 || level > h->plan.depth) return LORASP_E_ARG;
  const SymLevel &lv = h->plan.lev[level];
  if (cap < lv.K) return LORASP_E_ARG;
  for (int t = 0; t < lv.K; ++t) {
    if (order) order[t] = lv.order[t];
    if (wave) wave[lv.order[t]] = lv.node[lv.order[t]].wave;
  }
  return LORASP_OK;
}

int lorasp_get_node_counts(lorasp_handle h, int level, int *partners, int *n1, int cap) {
  if (!h || level < 1 || level > h->plan.depth) return LORASP_E_ARG;
  const SymLevel &lv = h->plan.lev[level];
  if (cap < lv.K) return LORASP_E_ARG;
  for (int c = 0; c < lv.K; ++c) {
    if (partners) partners[c] = (int)lv.node[c].partners.size();
    if (n1) n1[c] = (int)lv.node[c].n1.size() + (lv.node[c].aux ? 1 : 0);   // + b
  }
  return LORASP_OK;
}

int lorasp_get_ranks(lorasp_handle h, int level, int *ranks, int cap) {
  if (!h || !ranks || level < 1 || level > h->plan.depth) return LORASP_E_ARG;
  if (!h->factored) return LORASP_E_STATE;
  const auto &r = h->rnk[level];
  if (cap < (int)r.size()) return LORASP_E_ARG;
  std::copy(r.begin(), r.end(), ranks);
  return LORASP_OK;
}

int lorasp_get_sizes(lorasp_handle h, int level, int *sizes, int cap) {
  if (!h || !sizes || level < 1 || level > h->plan.depth) return LORASP_E_ARG;
  if (!h->factored) return LORASP_E_STATE;
  const auto &m = h->msz[level];
  if (cap < (int)m.size()) return LORASP_E_ARG;
  std::copy(m.begin(), m.end(), sizes);
  return LORASP_OK;
}

int lorasp_get_stats(lorasp_handle h, char *buf, size_t cap, size_t *len) {
  if (!h) return LORASP_E_ARG;
  std::ostringstream o;
  o.precision(17);
  const Plan &pl = h->plan;
  o << "{\"n\":" << pl.n << ",\"nnz\":" << pl.nnz << ",\"depth\":" << pl.depth << ",\"eps\":" << pl.eps
    << ",\"waves\":" << pl.total_waves << ",\"max_edge_distance\":" << pl.max_edge_distance
    << ",\"factored\":" << (h->factored ? "true" : "false");
  if (h->factored) {
    o << ",\"flops_model\":" << h->flops_model << ",\"factor_bytes\":" << h->f_doubles * 8
      << ",\"t_factor_host_ms\":" << h->t_factor_ms << ",\"t_task_build_ms\":" << h->t_host_ms
      << ",\"t_rank_sync_wait_ms\":" << h->t_sync_ms << ",\"launches_factor\":" << h->launches_factor
      << ",\"schedule_rank_predicted\":" << (h->replay_used ? "true" : "false")
      << ",\"rank_prediction_hits\":" << h->replay_hits << ",\"rank_prediction_misses\":" << h->replay_misses
      << ",\"split_pivot_nodes\":" << h->split_nodes << ",\"factor_graph\":" << (h->fgraph_used ? "true" : "false") << ",\"apply_dataflow\":" << (h->ap_df_ok ? "true" : "false")
      << ",\"factor_graph_captures\":" << h->fg_captures << ",\"factor_graph_launches\":" << h->fg_launches
      << ",\"factor_graph_failures\":" << h->fg_failures << ",\"dist_world\":" << h->dist_world
      << ",\"dist_rank\":" << h->dist_rank << ",\"dist_exchange_calls\":" << h->dist_calls
      << ",\"dist_allgather_bytes\":" << h->dist_bytes << ",\"dist_apply_bytes\":" << h->dist_apply_bytes
      << ",\"dist_apply_calls\":" << h->dist_apply_calls << ",\"dist_transport\":\""
      << (h->nccl ? "nccl" : (h->dist_world > 1 ? "callback" : "none")) << "\""
      << ",\"lu_partial_pivoting\":" << (h->lu_pivot ? "true" : "false")
      << ",\"lu_pivot_switches\":" << h->lu_pivot_switches << ",\"spd_fallbacks\":" << h->spd_fallbacks
      << ",\"path\":\"" << ((pl.flags & LORASP_SPD) ? "spd" : "lu") << "\"";
    {
      double g = 0;
      std::memcpy(&g, h->h_status + 2, sizeof(double));
      o << ",\"lu_max_multiplier\":" << g;
    }
    o << ",\"aux_vars\":";
    int64_t aux = 0;
    for (int i = 1; i <= pl.depth; ++i)
      for (int r : h->rnk[i]) aux += 2 * r;
    o << aux << ",\"levels\":[";
    // FactorStats (P:l.527-558, P:l.729-733): d_i, <rank>, compression ratio,
    // kappa1 / kappa2; alpha_hat = max_{i<l} (d_i / d_l)^(1/(l-i))
    int kap1 = 0, kap2 = 0;
    double alpha_hat = 0;
    const int dl = *std::max_element(h->msz[pl.depth].begin(), h->msz[pl.depth].end());
    for (int i = pl.depth; i >= 1; --i) {
      int64_t rs = 0, ms = 0, rs_c = 0, ms_c = 0;
      int rmax = 0, mmax = 0, nr = 0, k1 = 0, k2 = 0;
      for (size_t c = 0; c < h->rnk[i].size(); ++c) {
        const SymNode &nd = pl.lev[i].node[c];
        rs += h->rnk[i][c];
        rmax = std::max(rmax, h->rnk[i][c]);
        ms += h->msz[i][c];
        mmax = std::max(mmax, h->msz[i][c]);
        nr += nd.aux;
        if (nd.aux) {
          rs_c += h->rnk[i][c];
          ms_c += h->msz[i][c];
        }
        k1 = std::max(k1, (int)nd.n1.size() + (nd.aux ? 1 : 0));
        k2 = std::max(k2, (int)nd.partners.size());
      }
      kap1 = std::max(kap1, k1);
      kap2 = std::max(kap2, k2);
      if (i < pl.depth && dl > 0 && mmax > 0)
        alpha_hat = std::max(alpha_hat, std::pow((double)mmax / dl, 1.0 / (pl.depth - i)));
      o << "{\"level\":" << i << ",\"supers\":" << h->rnk[i].size() << ",\"compressed\":" << nr
        << ",\"rank_sum\":" << rs << ",\"rank_max\":" << rmax << ",\"size_sum\":" << ms
        << ",\"size_max\":" << mmax << ",\"d_max\":" << mmax
        << ",\"d_avg\":" << (double)ms / std::max<size_t>(1, h->msz[i].size())
        << ",\"rank_avg\":" << (nr ? (double)rs_c / nr : 0.0)
        << ",\"compression_ratio\":" << (ms_c ? (double)rs_c / ms_c : 0.0) << ",\"kappa1\":" << k1
        << ",\"kappa2\":" << k2 << ",\"waves\":" << pl.lev[i].wave_begin.size() - 1
        << ",\"lattice\":" << (pl.lev[i].lattice ? "true" : "false") << "}" << (i > 1 ? "," : "");
    }
    o << "],\"kappa1\":" << kap1 << ",\"kappa2\":" << kap2 << ",\"alpha_hat\":" << alpha_hat;
  }
  o << ",\"kernels\":{";
  bool first = true;
  for (int c = 0; c < K_NCLASS; ++c) {
    const KStat &k = h->kst[c];
    if (k.launches == 0) continue;
    o << (first ? "" : ",") << "\"" << KNAME[c] << "\":{\"class\":" << c << ",\"kernel\":\"" << KKERNEL[c]
      << "\",\"ms\":" << k.ms
      << ",\"launches\":" << k.launches << ",\"alg_flops\":" << k.flops << ",\"alg_bytes\":" << k.bytes << "}";
    first = false;
  }
  o << "}}";
  std::string s = o.str();
  if (len) *len = s.size() + 1;
  if (buf && cap > 0) {
    size_t k = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), k);
    buf[k] = 0;
  }
  return LORASP_OK;
}

int lorasp_get_launch_count(lorasp_handle h, int64_t *f, int64_t *a, int64_t *k) {
  if (!h) return LORASP_E_ARG;
  if (f) *f = h->launches_factor;
  if (a) *a = h->launches_apply;
  if (k) *k = h->launches_krylov;
  return LORASP_OK;
}

int lorasp_test_eig(int device, const double *G, int m, double eps, double *V, double *sigma, int *rank) {
  if (!G || !V || !sigma || !rank || m <= 0) return LORASP_E_ARG;
  try {
    CK(cudaSetDevice(device));
    set_eig_attrs();
    double *dG, *dV, *dS, *dW;
    int *dr, *dst;
    size_t mm = (size_t)m * m;
    CK(cudaMalloc(&dG, mm * 8));
    CK(cudaMalloc(&dV, mm * 8));
    CK(cudaMalloc(&dS, m * 8));
    CK(cudaMalloc(&dW, 7 * mm * 8));
    CK(cudaMalloc(&dr, 64));
    dst = dr + 4;
    CK(cudaMemset(dr, 0, 64));
    CK(cudaMemset(dV, 0, mm * 8));
    CK(cudaMemcpy(dG, G, mm * 8, cudaMemcpyHostToDevice));
    EigTask e{};
    e.G = dG;
    e.V = dV;
    e.sig = dS;
    e.work = dW;
    e.m = m;
    e.node = 0;
    e.rank_out = dr;
    long long *ddbg = nullptr;
    if (getenv("LORASP_EIG_PROFILE")) {
      CK(cudaMalloc(&ddbg, 4096));
      CK(cudaMemset(ddbg, 0, 4096));
    }
    e.dbg = ddbg;
    EigTask *de;
    CK(cudaMalloc(&de, sizeof(EigTask)));
    CK(cudaMemcpy(de, &e, sizeof(EigTask), cudaMemcpyHostToDevice));
    if (m <= EIGW_M && !getenv("LORASP_EIG_GENERIC")) {   // the production path for m <= 32
      // test hook: the warp count of the production variant (LORASP_TEST_EIGW_NW = 1 / 4 / 8)
      const char *nwe = getenv("LORASP_TEST_EIGW_NW");
      const int nw = nwe ? atoi(nwe) : 4;
      if (nw == 1) k_eig_warp<1><<<1, 32, EIGW_SMEM_DOUBLES * sizeof(double)>>>(de, eps, dst);
      else if (nw == 4) k_eig_warp<4><<<1, 128, EIGW_SMEM_DOUBLES * sizeof(double)>>>(de, eps, dst);
      else k_eig_warp<8><<<1, 256, EIGW_SMEM_DOUBLES * sizeof(double)>>>(de, eps, dst);
    } else {
      if (m >= EIG_REG_MIN && m <= EIG_REG_M && !getenv("LORASP_EIG_GENERIC")) {
        if (ddbg) {
          long long *dprof;
          CK(cudaMalloc(&dprof, 16 * 8 * 8));
          k_tridiag_reg<true><<<1, EIG_REG_THREADS>>>(de, eps, dprof);
          long long hp[128];
          CK(cudaMemcpy(hp, dprof, sizeof(hp), cudaMemcpyDeviceToHost));
          const char *nm[6] = {"ph2", "bar2", "ph3", "bar3", "ph4", "bar1"};
          for (int w = 0; w < 16; ++w) {
            fprintf(stderr, "  warp %2d:", w);
            for (int i = 0; i < 6; ++i) fprintf(stderr, " %s %lld", nm[i], hp[w * 8 + i]);
            fprintf(stderr, "\n");
          }
          cudaFree(dprof);
          k_tridiag_reg<false><<<1, EIG_REG_THREADS>>>(de, eps, nullptr);   // warm-up (timing below)
          CK(cudaDeviceSynchronize());
        }
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        launch_eig_reg(0, de, 1, m <= 32 ? 0 : (m <= 64 ? 1 : 2), eps, dst, 1);
        cudaEventRecord(e1);
        if (ddbg) {
          float ms = 0;
          cudaEventSynchronize(e1);
          cudaEventElapsedTime(&ms, e0, e1);
          fprintf(stderr, "[k_tridiag_reg m=%d] %.1f us\n", m, 1e3 * ms);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
      } else if (eig_cl_class(m) && !getenv("LORASP_EIG_GENERIC")) {
        if (ddbg) {
          long long *dprof, hp[8];
          CK(cudaMalloc(&dprof, 64));
          launch_tridiag_cl(0, de, 1, eig_cl_class(m), eps, dprof);
          CK(cudaMemcpy(hp, dprof, 64, cudaMemcpyDeviceToHost));
          cudaFree(dprof);
          fprintf(stderr, "  [cl phases, cycles/step] A %.0f bar %.0f B %.0f clsync1 %.0f C %.0f (bar+)D %.0f clsync2 %.0f pull %.0f\n",
                  hp[0] / (m - 2.0), hp[1] / (m - 2.0), hp[2] / (m - 2.0), hp[3] / (m - 2.0), hp[4] / (m - 2.0),
                  hp[5] / (m - 2.0), hp[6] / (m - 2.0), hp[7] / (m - 2.0));
        }
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        launch_tridiag_cl(0, de, 1, eig_cl_class(m), eps);
        cudaEventRecord(e1);
        cudaEvent_t pev[4];
        for (auto &x : pev) cudaEventCreate(&x);
        launch_pre_post(0, de, 1, m, eps, dst, ddbg ? pev : nullptr);
        cudaEventRecord(pev[3]);
        if (ddbg) {
          float ms = 0, a = 0, b = 0, c = 0, d = 0;
          cudaEventSynchronize(pev[3]);
          cudaEventElapsedTime(&ms, e0, e1);
          cudaEventElapsedTime(&a, e1, pev[0]);
          cudaEventElapsedTime(&b, pev[0], pev[1]);
          cudaEventElapsedTime(&c, pev[1], pev[2]);
          cudaEventElapsedTime(&d, pev[2], pev[3]);
          fprintf(stderr, "[k_tridiag_cl m=%d class %d] %.1f us | eigvals %.1f invit %.1f orth %.1f backtr %.1f us\n", m,
                  eig_cl_class(m), 1e3 * ms, 1e3 * a, 1e3 * b, 1e3 * c, 1e3 * d);
          long long ob[8];
          CK(cudaMemcpy(ob, ddbg + 20, sizeof(ob), cudaMemcpyDeviceToHost));
          fprintf(stderr, "  [orth CTA 1 cycles] intra-tail %lld cluster-sync %lld stage %lld project %lld | norm+barA %lld "
                  "normalise+barD %lld update %lld\n", ob[0], ob[1], ob[2], ob[3], ob[4], ob[5], ob[6]);
        }
        for (auto &x : pev) cudaEventDestroy(x);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
      } else {
        k_eig_t<false><<<1, EIG_THREADS, (size_t)eig_generic_cap(m) * 8>>>(de, eps, eig_generic_cap(m), dst);
      }
    }
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    int st[2];
    CK(cudaMemcpy(rank, dr, sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(st, dst, 2 * sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(sigma, dS, m * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(V, dV, (size_t)m * (*rank) * 8, cudaMemcpyDeviceToHost));
    if (ddbg) {
      long long tt[16];
      CK(cudaMemcpy(tt, ddbg, sizeof(tt), cudaMemcpyDeviceToHost));
      fprintf(stderr, "[tridiag phases] v %lld  matvec %lld  update %lld | invit %lld mgs %lld backtr %lld\n", tt[5],
              tt[6], tt[7], tt[8] - tt[2], tt[9] - tt[8], tt[3] - tt[9]);
      fprintf(stderr, "[eigvals] lambda0 %lld  rest %lld\n", tt[10] - tt[1], tt[2] - tt[10]);
      fprintf(stderr, "[eig m=%d r=%d] tridiag %lld  eigvals %lld  invit %lld  backtr %lld cycles\n", m, *rank,
              tt[1] - tt[0], tt[2] - tt[1], tt[3] - tt[2], tt[4] - tt[3]);
      cudaFree(ddbg);
    }
    cudaFree(dG); cudaFree(dV); cudaFree(dS); cudaFree(dW); cudaFree(dr); cudaFree(de);
    return st[0];
  } catch (const Err &e) {
    fprintf(stderr, "lorasp_test_eig: %s\n", e.msg.c_str());
    return e.code;
  }
}

// GEMM kernel comparison hook (north_star item 3, DMMA vs DFMA per block
// shape): `reps` independent copies of C = op(A) op(B) (a wave of equal GEMMs)
// through k_gemm2 (variant 0, FP64 FMA pipe) or k_gemm2_dmma (variant 1, FP64
// tensor cores); *ms = CUDA-event time of one launch (after a warm-up); C of
// the first copy returned.  A: M x K (ld M) or, ta, K x M (ld K); B: K x N (ld K)
// or, tb, N x K (ld N); C: M x N (ld M), host buffers.
int lorasp_test_gemm(int device, int variant, int M, int N, int K, int ta, int tb, int reps, const double *A,
                     const double *B, double *C, double *ms) {
  if (!A || !B || !C || M <= 0 || N <= 0 || K <= 0 || reps <= 0 || variant < 0 || variant > 1) return LORASP_E_ARG;
  try {
    CK(cudaSetDevice(device));
    double *dA, *dB, *dC;
    CK(cudaMalloc(&dA, (size_t)M * K * 8 * reps));
    CK(cudaMalloc(&dB, (size_t)K * N * 8 * reps));
    CK(cudaMalloc(&dC, (size_t)M * N * 8 * reps));
    for (int q = 0; q < reps; ++q) {
      CK(cudaMemcpy(dA + (size_t)q * M * K, A, (size_t)M * K * 8, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(dB + (size_t)q * K * N, B, (size_t)K * N * 8, cudaMemcpyHostToDevice));
    }
    std::vector<GemmTask> tasks;
    std::vector<GemmSeg> segs;
    for (int q = 0; q < reps; ++q) {
      GemmTask g{};
      g.C = dC + (size_t)q * M * N;
      g.ldc = M;
      g.M = M;
      g.N = N;
      g.ta = ta;
      g.tb = tb;
      g.beta = 0;
      g.seg0 = (int)segs.size();
      g.nseg = 1;
      segs.push_back(GemmSeg{dA + (size_t)q * M * K, dB + (size_t)q * K * N, ta ? K : M, tb ? N : K, K, 1.0});
      add_tiles(tasks, g);
    }
    GemmTask *dt;
    GemmSeg *ds;
    CK(cudaMalloc(&dt, tasks.size() * sizeof(GemmTask)));
    CK(cudaMalloc(&ds, segs.size() * sizeof(GemmSeg)));
    CK(cudaMemcpy(dt, tasks.data(), tasks.size() * sizeof(GemmTask), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ds, segs.data(), segs.size() * sizeof(GemmSeg), cudaMemcpyHostToDevice));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int it = 0; it < 4; ++it) {
      CK(cudaEventRecord(e0));
      if (variant == 0) k_gemm2<<<(unsigned)tasks.size(), 128>>>(dt, ds);
      else k_gemm2_dmma<<<(unsigned)tasks.size(), 128>>>(dt, ds);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float t = 0;
      CK(cudaEventElapsedTime(&t, e0, e1));
      if (it > 0) best = std::min(best, t);
    }
    CK(cudaGetLastError());
    *ms = best;
    CK(cudaMemcpy(C, dC, (size_t)M * N * 8, cudaMemcpyDeviceToHost));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(dt); cudaFree(ds);
    return LORASP_OK;
  } catch (const Err &e) {
    return e.code;
  }
}

int lorasp_test_pivot(int device, double *K, int m, int r) {
  if (!K || m < 0 || r < 0 || m + r == 0) return LORASP_E_ARG;
  try {
    CK(cudaSetDevice(device));
    CK(cudaFuncSetAttribute(k_pivot, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT));
    const int n = m + r;
    double *dK;
    int *dst;
    CK(cudaMalloc(&dK, (size_t)n * n * 8));
    CK(cudaMalloc(&dst, 64));
    CK(cudaMemset(dst, 0, 64));
    CK(cudaMemcpy(dK, K, (size_t)n * n * 8, cudaMemcpyHostToDevice));
    PivTask t{dK, n, m, r, 0};
    PivTask *dt;
    CK(cudaMalloc(&dt, sizeof(PivTask)));
    CK(cudaMemcpy(dt, &t, sizeof(PivTask), cudaMemcpyHostToDevice));
    if (n <= PIVW_MAXN) {   // the production kernel for n <= 32
      k_pivot_warp<1><<<1, 32 * PivW<1>::WARPS, PivW<1>::SMEM>>>(dt, 1, dst);
    } else if (n <= PIVB_MAXN) {
      CK(cudaFuncSetAttribute(k_pivot_blk, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
      k_pivot_blk<<<1, 512, pivb_smem_bytes(n)>>>(dt, dst);
    } else {
      int cap = (int)std::min<int64_t>((int64_t)n * n + n, SMEM_LIMIT / 8);
      cap = std::max(cap, n);
      k_pivot<<<1, 512, cap * 8>>>(dt, cap, dst);
    }
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    int st[2];
    CK(cudaMemcpy(st, dst, 2 * sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(K, dK, (size_t)n * n * 8, cudaMemcpyDeviceToHost));
    cudaFree(dK); cudaFree(dst); cudaFree(dt);
    return st[0];
  } catch (const Err &e) {
    return e.code;
  }
}

const char *lorasp_last_error(lorasp_handle h) { return h ? h->last_error.c_str() : "null handle"; }

void lorasp_destroy(lorasp_handle h) {
  if (!h) return;
  if (h->mem_ready) {
    cudaSetDevice(h->device);
    // every library stream drains before any buffer is released (a factorization
    // that threw may have left split-pivot / eigen work in flight)
    cudaStreamSynchronize(h->stream);
    for (cudaStream_t s : {h->stream2, h->stream_hi, h->stream_eig, h->stream_cl[0], h->stream_cl[1], h->stream_cl[2]})
      if (s) cudaStreamSynchronize(s);
    DevBuf *bufs[] = {&h->d_values, &h->d_rowptr, &h->d_colidx, &h->d_dest, &h->arena[0], &h->arena[1],
                      &h->ws_G, &h->ws_V, &h->ws_sig, &h->ws_X, &h->ws_ctr, &h->ws_piv, &h->d_ranks,
                      &h->d_status,
                      &h->d_vec, &h->d_y, &h->d_perm, &h->d_b, &h->d_x, &h->d_kry, &h->d_apnodes,
                      &h->d_apsegs, &h->d_dotpart};
    for (DevBuf *b : bufs) b->release();
    for (cudaEvent_t e : h->evpool) cudaEventDestroy(e);
    if (h->ap_graph) cudaGraphExecDestroy(h->ap_graph);
    if (h->nccl) {
      if (const NcclApi *api = nccl_api()) api->CommDestroy(h->nccl);
      h->nccl = nullptr;
    }
    h->nccl_send.release();
    h->nccl_recv.release();
    if (h->fgraph) cudaGraphExecDestroy(h->fgraph);
    h->fg_desc.release();
    if (h->stream2) {
      cudaStreamSynchronize(h->stream2);
      cudaStreamDestroy(h->stream2);
    }
    if (h->stream_hi) {
      cudaStreamSynchronize(h->stream_hi);
      cudaStreamDestroy(h->stream_hi);
    }
    if (h->stream_eig) {
      cudaStreamSynchronize(h->stream_eig);
      cudaStreamDestroy(h->stream_eig);
    }
    for (auto &cs : h->stream_cl)
      if (cs) {
        cudaStreamSynchronize(cs);
        cudaStreamDestroy(cs);
      }
    if (h->ev_cf) cudaEventDestroy(h->ev_cf);
    for (auto &e : h->ev_cj)
      if (e) cudaEventDestroy(e);
    if (h->ev_ef) cudaEventDestroy(h->ev_ef);
    if (h->ev_ej) cudaEventDestroy(h->ev_ej);
    if (h->ev_u) cudaEventDestroy(h->ev_u);
    if (h->ev_s0) cudaEventDestroy(h->ev_s0);
    if (h->ev_s1) cudaEventDestroy(h->ev_s1);
    if (h->h_sp) cudaFreeHost(h->h_sp);
    if (h->h_ranklog) cudaFreeHost(h->h_ranklog);
    h->ws_S.release();
    h->ws_Y.release();
    h->ws_T1.release();
    h->ws_piv2.release();
    h->d_sp.release();
    h->d_apparts.release();
    for (DevBuf *b : {&h->d_apdf, &h->d_apcontr, &h->d_apdfl, &h->d_zob, &h->d_dfcnt}) b->release();
    h->d_upart.release();
    h->fpool.release();
    h->stg.release();
    if (h->h_ranks) cudaFreeHost(h->h_ranks);
    if (h->h_status) cudaFreeHost(h->h_status);
    if (h->h_dot) cudaFreeHost(h->h_dot);
  }
  delete h;
}

}  // extern "C"
