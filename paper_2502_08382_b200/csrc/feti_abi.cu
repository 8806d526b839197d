// Host runtime behind the C-ABI (include/feti_b200.h).
//
// Owns the device memory of one operator context (persistent: packed F~ apply
// tiles, index maps, dual vectors; temporary: factor tiles and X panels of the
// assembly), builds the batched work lists once at finalize (the reference's
// symbolic/prepare stage, dualop.py:212-269), and sequences the kernels of
// preprocess (dualop.py:301-327) and apply (dualop.py:348-388).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/feti_b200.h"
#include "feti_common.cuh"
#include "feti_coarse.h"
#include "feti_exchange.h"
#include "feti_factor.h"
#include "feti_implicit.h"
#include "feti_kernels.h"
#include "feti_pcpg.h"
#include "feti_sparse.h"

using namespace feti;

namespace {

thread_local std::string g_err;
const bool g_debug_sync = getenv("FETI_DEBUG_SYNC") != nullptr;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define FETI_DEBUG_SYNC(st)                                                                   \
  do {                                                                                        \
    if (g_debug_sync) {                                                                       \
      cudaError_t _e = cudaStreamSynchronize(st);                                             \
      if (_e == cudaSuccess) _e = cudaGetLastError();                                         \
      if (_e != cudaSuccess)                                                                  \
        return fail(FETI_ERR_CUDA, "kernel failed at %s:%d: %s", __FILE__, __LINE__,          \
                    cudaGetErrorString(_e));                                                  \
    }                                                                                         \
  } while (0)

#define CUDA_TRY(expr)                                                                          \
  do {                                                                                          \
    cudaError_t _e = (expr);                                                                    \
    if (_e != cudaSuccess) {                                                                    \
      if (_e == cudaErrorMemoryAllocation)                                                      \
        return fail(FETI_ERR_CAPACITY, "device memory exhausted in %s: %s", #expr,              \
                    cudaGetErrorString(_e));                                                    \
      return fail(FETI_ERR_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e));               \
    }                                                                                           \
  } while (0)

struct SubHost {
  int64_t n = 0, m = 0, nnz = 0;
  int T = 0, P = 0, T32 = 0;
  int smin = 0;                      // first block row reached by any X column
  int64_t raw_off = 0;               // first factor value the device needs
  bool dense = true;
  std::vector<int64_t> colperm;      // sorted position -> original local row
  std::vector<int> r_sorted;         // P*128
  std::vector<double> s_sorted;      // P*128
  std::vector<int> gids_sorted;      // T32*32
  std::vector<int> panel_minrow;     // P
  std::vector<int64_t> up, ui;       // sparse pattern (host copy until finalize)
  // device
  double* d_raw_own = nullptr;       // lib-owned upload buffer
  const double* d_raw = nullptr;     // current factor values
  int64_t* d_up = nullptr;
  int64_t* d_ui = nullptr;
  double* d_tiles = nullptr;
  double* d_X = nullptr;
  double* d_F = nullptr;
  double *d_U = nullptr, *d_Y = nullptr, *d_Lt = nullptr;   // path "trsm" only
  double* d_Fp = nullptr;            // lumped preconditioner B~ K B~^T, same tile layout as d_F
  int* d_r = nullptr;
  double* d_s = nullptr;
  int* d_g = nullptr;
  int* d_pmin = nullptr;
  bool factor_set = false;
  bool factor_from_host = false;
  const double* h_values = nullptr;  // host factor awaiting upload at assemble
  int tbase = 0;                     // first stored tile block
  int src = SRC_RAW_DENSE;
  // device factorization inputs (feti_set_stiffness)
  bool stiff_set = false;
  int64_t k_nnz = 0;
  int kr = 0;
  double rho = 0.0;
  double* d_Q = nullptr;
  int64_t *d_perm = nullptr, *d_iperm = nullptr, *d_kptr = nullptr, *d_kind = nullptr;
  double* d_kdata = nullptr;
  cudaEvent_t ev_upload = nullptr;
  // sparse-factor route (feti_set_sparse_pattern): K_s = K + rho E E^T in a
  // block-sparse tile pool, rank-2r correction after the assembly
  bool sp_pattern = false;
  int sp_r = 0;
  int64_t sp_n = 0;                  // DOFs (rows of K); n above counts positions (>= sp_n)
  std::vector<int64_t> sp_perm, sp_iperm, sp_kptr, sp_kind, sp_fix;
  SpPlan sp;
  double* d_pool = nullptr;
  int* d_tmap = nullptr;
  int64_t* d_fix = nullptr;
  double* d_U1 = nullptr;
  double* d_U2W = nullptr;
  int64_t* d_kdiag = nullptr;        // diagonal position of each row of K (rho on the device)
  double *d_fproj = nullptr, *d_qtf = nullptr, *d_U2f = nullptr;   // device dual rhs (feti_enable_dual_rhs)
  std::vector<double> h_qtf;
  double* d_rho = nullptr;
  std::vector<double> h_Q, h_U1;     // last kernel basis handed over and its U1 = B~ Q (async sources)
  int64_t f_tiles() const { return (int64_t)T32 * (T32 + 1) / 2; }
  int64_t l_tiles() const { return (int64_t)(T - tbase) * (T - tbase + 1) / 2; }
  int64_t upload_count() const { return nnz - raw_off; }
};

struct DevBuf {
  void* p = nullptr;
};

}  // namespace

struct feti_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr, copy_stream = nullptr;
  std::vector<SubHost> subs;
  int64_t n_mult = 0;
  bool finalized = false, assembled = false;
  bool implicit = false;             // FETI_STRATEGY_IMPLICIT: no F~, sweeps per apply
  bool path_trsm = false;            // FETI_PATH_TRSM: F = B~ (L^-T X) instead of X^T X
  std::vector<void*> allocs;
  int64_t bytes_persistent = 0, bytes_temporary = 0;
  // device tables
  SubDev* d_subdev = nullptr;
  int4 *d_w_unpack = nullptr, *d_w_diag = nullptr, *d_w_scale = nullptr, *d_w_chain = nullptr,
       *d_w_syrk = nullptr;
  ApplySeg* d_apply_segs = nullptr;
  int n_unpack = 0, n_diag = 0, n_scale = 0, n_chain = 0, n_syrk = 0, n_apply = 0;
  int64_t* d_ridx = nullptr;        // partial positions per (subdomain, multiplier) contribution
  int* d_apply_seg_ptr = nullptr;
  double* d_part = nullptr;
  int* d_cptr = nullptr;
  int4* d_cent = nullptr;
  double *d_p = nullptr, *d_q = nullptr;
  int apply_nw = 8;
  int apply_sb = 32;                 // apply super-block edge (32x32 tiles)
  int apply_cps = 1;                 // apply CTAs per SM
  feti_stats stats{};
  cudaEvent_t ev[8] = {};
  bool subdev_dirty = true;
  // device factorization (feti_enable_device_factorization before finalize)
  bool device_factor = false;
  bool tiles_fresh = false;          // tiles hold L (not yet block-scaled)
  int uniform_T = 0;
  FactorSub* d_fsub = nullptr;
  double* d_dinv = nullptr;
  int* d_bad = nullptr;
  int64_t* d_vec_off = nullptr;
  double *d_sb = nullptr, *d_sx = nullptr;
  // sparse-route solve: growing per-call buffers (b, x, scratch; items)
  double* d_sps = nullptr;
  size_t sps_cap = 0;
  SpSolveItem* d_sps_items = nullptr;
  size_t sps_items_cap = 0;
  int* d_slots = nullptr;
  // implicit apply: per-slot offsets into a partial buffer of sum(m) values
  int64_t* d_impl_off = nullptr;
  double* d_impl_part = nullptr;
  int impl_max_blocks = 0;
  // coarse space (GPU-resident PCPG): G blocks, (G^T G)^-1, work vectors
  int nk = 0;
  CoarseSub* d_coarse = nullptr;
  int2* d_kcols = nullptr;
  double* d_cinv = nullptr;
  double* d_kv = nullptr;
  double* d_kz = nullptr;
  // G flattened by kernel column and cut into pieces (device PCPG's G^T x)
  double* d_gval = nullptr;
  int* d_gidx = nullptr;
  int4* d_pieces = nullptr;
  int npieces = 0;
  double* d_ppart = nullptr;
  // upload/compute pipeline for host factors: subdomains grouped in waves
  // (largest work first); wave w's H2D on copy_stream, its kernels on
  // wave_streams[w % 2] once its copies landed
  static constexpr int kWaveStreams = 2;
  cudaStream_t wave_streams[kWaveStreams] = {};
  cudaEvent_t wave_join[kWaveStreams] = {};
  std::vector<std::vector<int>> waves;
  std::vector<cudaEvent_t> wave_ev;
  // per-wave work lists: [kind][wave] -> (offset, count) into d_wv[kind]
  int4* d_wv[5] = {};
  std::vector<std::pair<int, int>> wv_range[5];
  // sparse-factor route: per block column task ranges into the device lists
  bool sparse_factor = false;
  bool dual_rhs = false;             // factor f' along (appended row) for d = B~ K_reg^-1 f
  SpSub* d_spsub = nullptr;
  SpInit* d_sp_init = nullptr;
  SpTask* d_sp_tasks = nullptr;
  SpPair* d_sp_pairs = nullptr;
  SpDiag* d_sp_diag = nullptr;
  int2* d_sp_panels = nullptr;
  int n_sp_init = 0, n_sp_panels = 0, sp_max_T32 = 0, sp_max_n = 0;
  int sp_u2_cols = 0;                // implicit sparse route: columns of the U2 sweep (max r, +1 for f')
  // subdomains are split into sp_groups groups, each factored on its own
  // stream: one group's latency-bound diagonal factorizations overlap the
  // DMMA tile work of the others.  Ranges are indexed [g * sp_maxTq + j].
  std::vector<std::pair<int, int>> sp_acc_rng, sp_panel_rng, sp_diag_rng;
  int sp_groups = 1, sp_maxTq = 0;
  bool sp_graph_used = false;
  static constexpr int kSpStreams = 16;   // upper bound on factorization groups (FETI_SP_GROUPS, default 8)
  std::vector<std::pair<int, int>> sp_corr_rng, sp_sub_rng;   // per group: panels, subdomains
  cudaEvent_t sp_ev[3] = {};   // factorize start, factorize end, assemble end
  // fused graph: each group's interface assembly + correction captured right
  // behind its column sequence on its stream (FETI_SP_FUSE=0: separate);
  // sp_fend[g] marks group g's factorization end (external event records)
  bool sp_graph_fused = false, sp_assembled_in_graph = false, sp_graph_built = false;
  cudaGraphExec_t sp_gexec[kSpStreams] = {};   // per-group step graphs
  int sp_glaunches[kSpStreams] = {};
  cudaEvent_t k_ready_grp[kSpStreams] = {};    // a group's K values (and Q / forces) landed
  std::vector<int> sp_group_of;                // slot -> factorization group
  std::vector<std::pair<int, int>> sp_init_rng;  // per group: range of d_sp_init
  cudaEvent_t sp_fend[kSpStreams] = {};
  // sparse-route stiffness hand-over: values are copied on copy_stream while
  // the pool is zeroed; k_ready = copies issued so far landed, k_free = the
  // last scatter finished reading the previous values
  cudaEvent_t k_ready = nullptr, k_free = nullptr;
  bool k_pending = false;
  bool k_early = false;              // Q or f' changed: sp_init reads them, so wait before it
  std::vector<int> sp_bad_init;
  bool sp_pending_check = false;   // pivots of the last factorize not yet checked
  // device-native PCPG (feti_pcpg_solve): iteration vectors, coarse scratch,
  // block partials, device scalars (+ a pinned host copy polled per graph)
  double* pc_vec = nullptr;
  double* pc_k = nullptr;
  double* pc_bpart = nullptr;
  PcpgScal* pc_sc = nullptr;
  PcpgScal* pc_sc_host = nullptr;
  cudaGraphExec_t pc_graph[2] = {};
  static constexpr int kPcpgGraphIters = 8;
  // lumped preconditioner (feti_set_preconditioner): a second descriptor table
  // whose F points at the preconditioner tiles, applied by the same kernels
  SubDev* d_subdev_p = nullptr;
  int n_precond_set = 0;
  // fused cross-rank exchange (feti_exchange_setup/connect)
  int x_rank = 0, x_world = 1;
  double* x_slab = nullptr;          // own slab (IPC-exported)
  std::vector<double*> x_open;       // peer slabs opened through IPC (to close)
  double** d_x_peers = nullptr;
  int* d_x_touched = nullptr;
  int x_n_touched = 0;
  unsigned* d_x_done = nullptr;
  int* d_x_error = nullptr;
  int64_t x_epoch = 0;
  bool x_ready = false;
  cudaEvent_t x_sum_done = nullptr;  // end of the last exchange's sum (slab reuse order)
  // end of the last apply enqueued on a caller stream: the next
  // factorization/assembly (which rewrite the tiles and F~) waits for it
  cudaEvent_t apply_done = nullptr;
  bool apply_pending = false;
  std::vector<int> h_cptr;           // host copy of the contribution CSR pointer
  cudaStream_t sp_streams[kSpStreams] = {};
  cudaEvent_t sp_join[kSpStreams] = {};
  double sp_flops = 0.0;
  double sp_flops_scalar = 0.0;
};

extern "C" {
static int sparse_group_assembly(feti_ctx* c, int g, cudaStream_t gs, int* launches);
}

namespace {

int dev_alloc(feti_ctx* c, void** p, size_t bytes, bool persistent) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    return fail(FETI_ERR_CAPACITY,
                "device pool of %zu bytes cannot hold %lld persistent bytes plus a %zu-byte request "
                "(%zu free)",
                tot, (long long)c->bytes_persistent, bytes, fr);
  }
  c->allocs.push_back(*p);
  if (persistent)
    c->bytes_persistent += (int64_t)bytes;
  else
    c->bytes_temporary += (int64_t)bytes;
  return FETI_OK;
}

template <class T>
int upload(feti_ctx* c, T** dst, const std::vector<T>& v, bool persistent = true) {
  int rc = dev_alloc(c, (void**)dst, v.size() * sizeof(T), persistent);
  if (rc) return rc;
  if (!v.empty()) CUDA_TRY(cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return FETI_OK;
}

void fill_subdev(const feti_ctx* c, std::vector<SubDev>& h);

int sync_subdev(feti_ctx* c) {
  std::vector<SubDev> h;
  fill_subdev(c, h);
  if (!h.empty())
    CUDA_TRY(cudaMemcpyAsync(c->d_subdev, h.data(), h.size() * sizeof(SubDev), cudaMemcpyHostToDevice,
                             c->stream));
  c->subdev_dirty = false;
  return FETI_OK;
}

void fill_subdev(const feti_ctx* c, std::vector<SubDev>& h) {
  h.resize(c->subs.size());
  for (size_t i = 0; i < c->subs.size(); ++i) {
    const SubHost& s = c->subs[i];
    SubDev& d = h[i];
    d.raw = s.d_raw;
    d.up = s.dense ? nullptr : s.d_up;
    d.ui = s.dense ? nullptr : s.d_ui;
    d.tiles = s.d_tiles;
    d.X = s.d_X;
    d.F = s.d_F;
    d.U = s.d_U;
    d.Y = s.d_Y;
    d.Lt = s.d_Lt;
    // sparse route, SYRK path: the rank-2r correction rides in the SYRK epilogue
    const bool fused = c->sparse_factor && !c->implicit && !c->path_trsm && s.sp_r > 0 && s.d_U1;
    d.U1 = fused ? s.d_U1 : nullptr;
    d.U2W = fused ? s.d_U2W : nullptr;
    d.kr = fused ? s.sp_r : 0;
    d.r_sorted = s.d_r;
    d.s_sorted = s.d_s;
    d.gids_sorted = s.d_g;
    d.panel_minrow = s.d_pmin;
    d.nnz = s.nnz;
    d.raw_off = s.raw_off;
    d.smin = s.smin;
    d.tbase = s.tbase;
    d.src = s.src;
    d.n = (int)s.n;
    d.m = (int)s.m;
    d.T = s.T;
    d.P = s.P;
    d.T32 = s.T32;
  }
}

// Device task lists of the block-sparse factorization, ordered by block
// column: [acc(j) | potrf(j) | panel(j)] with every subdomain batched in each
// launch (deepest accumulations first).
int build_sparse_tasks(feti_ctx* c) {
  const int ns = (int)c->subs.size();
  int rc;
  if ((rc = dev_alloc(c, (void**)&c->d_dinv, (size_t)ns * TILE * 8, false))) return rc;
  if ((rc = dev_alloc(c, (void**)&c->d_bad, (size_t)ns * sizeof(int), false))) return rc;
  if ((rc = dev_alloc(c, (void**)&c->d_spsub, (size_t)ns * sizeof(SpSub), true))) return rc;
  int maxTq = 0;
  std::vector<SpInit> init;
  std::vector<int2> panels;
  for (int si = 0; si < ns; ++si) {
    SubHost& s = c->subs[si];
    const SpPlan& P = s.sp;
    maxTq = std::max(maxTq, P.Tq);
    c->sp_max_T32 = std::max(c->sp_max_T32, s.T32);
    c->sp_max_n = std::max<int>(c->sp_max_n, (int)s.sp_n);
    c->sp_u2_cols = std::max(c->sp_u2_cols, s.sp_r + (c->dual_rhs ? 1 : 0));
    for (int K = 0; K < P.Tq; ++K)
      for (int L = 0; L <= K; ++L) {
        const int slot = P.tmap[(size_t)K * P.Tq + L];
        if (slot >= 0) init.push_back(SpInit{s.d_pool + (size_t)slot * TILE, K, L, si, 0});
      }
    c->sp_flops += P.flops_exec;
    c->sp_flops_scalar += P.flops_scalar;
  }
  // correction work per group (contiguous subdomain ranges, as the waves)
  c->sp_corr_rng.assign(c->sp_groups, {0, 0});
  c->sp_sub_rng.assign(c->sp_groups, {0, 0});
  for (int g = 0; g < c->sp_groups; ++g) {
    const std::vector<int>& wv = c->waves[g];
    const int b = (int)panels.size();
    for (int si : wv)
      if (c->subs[si].sp_r > 0 || c->dual_rhs)
        for (int p = 0; p < c->subs[si].P; ++p) panels.push_back(make_int2(si, p));
    c->sp_corr_rng[g] = {b, (int)panels.size() - b};
    c->sp_sub_rng[g] = {wv.empty() ? 0 : wv.front(), (int)wv.size()};
  }
  std::vector<SpTask> tasks;
  std::vector<SpPair> pairs;
  std::vector<SpDiag> diag;
  const int G = c->sp_groups;
  c->sp_maxTq = maxTq;
  c->sp_acc_rng.assign((size_t)G * maxTq, {0, 0});
  c->sp_panel_rng.assign((size_t)G * maxTq, {0, 0});
  c->sp_diag_rng.assign((size_t)G * maxTq, {0, 0});
  for (int g = 0; g < G; ++g) {
    CUDA_TRY(cudaStreamCreateWithFlags(&c->sp_streams[g], cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&c->sp_join[g], cudaEventDisableTiming));
  }
  for (auto& e : c->sp_ev) CUDA_TRY(cudaEventCreate(&e));
  for (int g = 0; g < G; ++g) {
    CUDA_TRY(cudaEventCreate(&c->sp_fend[g]));
    CUDA_TRY(cudaEventCreateWithFlags(&c->k_ready_grp[g], cudaEventDisableTiming));
  }
  // contiguous groups of subdomains
  auto group_of = [&](int si) { return (int)((int64_t)si * G / std::max(ns, 1)); };
  c->sp_group_of.assign(ns, 0);
  for (int si = 0; si < ns; ++si) c->sp_group_of[si] = group_of(si);
  // slots of the (P Q)^T block row: their tasks run "thin" (rows < 8 only)
  std::vector<std::vector<char>> qrow(ns);
  for (int si = 0; si < ns; ++si) {
    const SpPlan& P = c->subs[si].sp;
    qrow[si].assign((size_t)P.ntiles, 0);
    if (P.Tq > P.T)
      for (int L = 0; L <= P.T; ++L) {
        const int slot = P.tmap[(size_t)P.T * P.Tq + L];
        if (slot >= 0) qrow[si][slot] = 1;
      }
  }
  for (int g = 0; g < G; ++g)
  for (int j = 0; j < maxTq; ++j) {
    const size_t gj = (size_t)g * maxTq + j;
    int b = (int)tasks.size();
    for (int si = 0; si < ns; ++si) {
      const SubHost& s = c->subs[si];
      if (j >= s.sp.Tq || group_of(si) != g) continue;
      for (const auto& t : s.sp.acc[j]) {
        // one entry per needed k-slice of every product (structurally zero
        // slices of either operand skipped: they add exact zeros)
        const int64_t p0 = (int64_t)pairs.size();
        for (const auto& pr : t.second) {
          const unsigned mk = s.sp.slot_mask[pr.first] & s.sp.slot_mask[pr.second];
          for (int q = 0; q < TB / KS; ++q)
            if (mk >> q & 1)
              pairs.push_back(SpPair{s.d_pool + (size_t)pr.first * TILE + (size_t)q * SLICE,
                                     s.d_pool + (size_t)pr.second * TILE + (size_t)q * SLICE});
        }
        tasks.push_back(SpTask{s.d_pool + (size_t)t.first * TILE, p0, (int)((int64_t)pairs.size() - p0),
                               qrow[si][t.first] ? 2 : 0});
      }
    }
    // largest first (shortest launch tail; keeping the subdomain order for L2
    // locality of shared operand tiles measured the same, 42.6 vs 42.3 ms)
    std::stable_sort(tasks.begin() + b, tasks.end(), [](const SpTask& x, const SpTask& y) {
      return x.npairs * ((x.flags & 2) ? 1 : 4) > y.npairs * ((y.flags & 2) ? 1 : 4);
    });
    c->sp_acc_rng[gj] = {b, (int)tasks.size() - b};
    // inv(L_jj): the subdomain's scratch, or -- in the trailing triangle,
    // where the assembly wants inv(L_jj) in the diagonal tile anyway -- the
    // diagonal tile itself (potrf_invert_128 stores L, then the inverse over it)
    auto dinv_of = [&](int si) -> double* {
      const SubHost& s = c->subs[si];
      return j >= s.smin ? s.d_pool + (size_t)s.sp.tmap[(size_t)j * s.sp.Tq + j] * TILE
                         : c->d_dinv + (size_t)si * TILE;
    };
    const int db = (int)diag.size();
    for (int si = 0; si < ns; ++si) {
      const SubHost& s = c->subs[si];
      if (j >= s.sp.T || group_of(si) != g) continue;
      diag.push_back(SpDiag{s.d_pool + (size_t)s.sp.tmap[(size_t)j * s.sp.Tq + j] * TILE, dinv_of(si), si, j * TB});
    }
    c->sp_diag_rng[gj] = {db, (int)diag.size() - db};
    b = (int)tasks.size();
    for (int si = 0; si < ns; ++si) {
      const SubHost& s = c->subs[si];
      if (j >= s.sp.T || group_of(si) != g) continue;
      for (int slot : s.sp.panel[j]) {
        // L_ij = A_ij inv(L_jj)^T over the k-slices (columns of block j) where A_ij has nonzeros
        double* C = s.d_pool + (size_t)slot * TILE;
        const int64_t p0 = (int64_t)pairs.size();
        const unsigned mk = s.sp.slot_mask[slot];
        for (int q = 0; q < TB / KS; ++q)
          if (mk >> q & 1) pairs.push_back(SpPair{C + (size_t)q * SLICE, dinv_of(si) + (size_t)q * SLICE});
        tasks.push_back(SpTask{C, p0, (int)((int64_t)pairs.size() - p0), qrow[si][slot] ? 3 : 1});
      }
    }
    c->sp_panel_rng[gj] = {b, (int)tasks.size() - b};
  }
  // per group: its subdomains' init entries (the list is in subdomain order)
  c->sp_init_rng.assign(G, {0, 0});
  {
    size_t a = 0;
    for (int g = 0; g < G; ++g) {
      size_t b = a;
      while (b < init.size() && group_of(init[b].sub) == g) ++b;
      c->sp_init_rng[g] = {(int)a, (int)(b - a)};
      a = b;
    }
  }
  if ((rc = upload(c, &c->d_sp_init, init))) return rc;
  if ((rc = upload(c, &c->d_sp_tasks, tasks))) return rc;
  if ((rc = upload(c, &c->d_sp_pairs, pairs))) return rc;
  if ((rc = upload(c, &c->d_sp_diag, diag))) return rc;
  if ((rc = upload(c, &c->d_sp_panels, panels))) return rc;
  c->n_sp_init = (int)init.size();
  c->n_sp_panels = (int)panels.size();
  for (auto& s : c->subs) {   // the plan's task lists live on the device now
    decltype(s.sp.acc)().swap(s.sp.acc);
    decltype(s.sp.panel)().swap(s.sp.panel);
    decltype(s.sp.slot_mask)().swap(s.sp.slot_mask);
  }
  CUDA_TRY(configure_sparse());
  CUDA_TRY(configure_sp_solve());
  return FETI_OK;
}

int factorize_sparse(feti_ctx* c) {
  cudaStream_t st = c->stream;
  const int ns = (int)c->subs.size();
  std::vector<SpSub> ss(ns);
  for (int si = 0; si < ns; ++si) {
    SubHost& s = c->subs[si];
    ss[si] = SpSub{s.d_pool, s.d_tmap, s.d_perm, s.d_iperm, s.d_kptr, s.d_kind, s.d_kdata, s.d_Q, s.d_kdiag,
                   s.d_fix, s.d_U1, s.d_U2W, s.d_rho, s.d_fproj, s.d_qtf, s.d_U2f, c->dual_rhs ? s.sp_r : -1,
                   s.sp.T, s.sp.Tq, (int)s.sp_n, s.sp_r, s.sp_r, (int)s.n};
    s.src = SRC_TILES;
  }
  CUDA_TRY(cudaMemcpyAsync(c->d_spsub, ss.data(), ns * sizeof(SpSub), cudaMemcpyHostToDevice, st));
  int rc;
  c->subdev_dirty = true;
  if ((rc = sync_subdev(c))) return rc;
  c->sp_bad_init.assign(ns, 1 << 30);
  CUDA_TRY(cudaMemcpyAsync(c->d_bad, c->sp_bad_init.data(), ns * sizeof(int), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaEventRecord(c->sp_ev[0], st));
  const int G = c->sp_groups;
  const bool use_graph = !g_debug_sync && !(getenv("FETI_SP_GRAPH") && atoi(getenv("FETI_SP_GRAPH")) == 0);
  int launches = 0;
  if (use_graph) {
    // one CUDA graph per group, replayed on the group's stream: [rho, K scatter,
    // the group's column sequence, its interface assembly + correction].  The
    // group's pool is zeroed on its stream first, and its graph waits only for
    // its own subdomains' K values (k_ready_grp), so with host K values the
    // H2D copy of later groups overlaps the factorization of earlier ones.
    // Each group's assembly overlaps the other groups' factorization.
    if (!c->sp_graph_built)
      c->sp_graph_fused = !(getenv("FETI_SP_FUSE") && atoi(getenv("FETI_SP_FUSE")) == 0);
    CUDA_TRY(cudaEventRecord(c->ev[2], st));
    int nl = 0;
    for (int g = 0; g < G; ++g) {
      cudaStream_t gs = c->sp_streams[g];
      const auto ir = c->sp_init_rng[g], sr = c->sp_sub_rng[g];
      CUDA_TRY(cudaStreamWaitEvent(gs, c->ev[2], 0));
      // a changed kernel basis / force is read by the pool init itself
      if (c->k_pending && c->k_early) CUDA_TRY(cudaStreamWaitEvent(gs, c->k_ready_grp[g], 0));
      launch_sp_init(c->d_sp_init + ir.first, ir.second, c->d_spsub, gs);
      if (c->k_pending) CUDA_TRY(cudaStreamWaitEvent(gs, c->k_ready_grp[g], 0));
      launches += ir.second > 0;
      if (!c->sp_gexec[g]) {
        int gl = 0;
        CUDA_TRY(cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal));
        launch_sp_trace(c->d_spsub + sr.first, sr.second, gs);
        launch_sp_scatter(c->d_spsub, sr.first, sr.second, c->sp_max_n, gs);
        gl += 2 * (sr.second > 0);
        for (int j = 0; j < c->sp_maxTq; ++j) {
          const size_t gj = (size_t)g * c->sp_maxTq + j;
          const auto a = c->sp_acc_rng[gj], d = c->sp_diag_rng[gj], pp = c->sp_panel_rng[gj];
          launch_sp_gemm(c->d_sp_tasks + a.first, a.second, c->d_sp_pairs, gs);
          launch_sp_potrf(c->d_sp_diag + d.first, d.second, c->d_bad, gs);
          launch_sp_gemm(c->d_sp_tasks + pp.first, pp.second, c->d_sp_pairs, gs);
          gl += (a.second > 0) + (d.second > 0) + (pp.second > 0);
        }
        int rc2 = FETI_OK;
        if (c->sp_graph_fused) {
          cudaError_t e = cudaEventRecordWithFlags(c->sp_fend[g], gs, cudaEventRecordExternal);
          rc2 = e != cudaSuccess ? fail(FETI_ERR_CUDA, "%s", cudaGetErrorString(e))
                                 : sparse_group_assembly(c, g, gs, &gl);
        }
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamEndCapture(gs, &graph);
        if (rc2) {
          if (graph) cudaGraphDestroy(graph);
          return rc2;
        }
        CUDA_TRY(e);
        e = cudaGraphInstantiate(&c->sp_gexec[g], graph, 0);
        cudaGraphDestroy(graph);
        CUDA_TRY(e);
        c->sp_glaunches[g] = gl;
      }
      CUDA_TRY(cudaGraphLaunch(c->sp_gexec[g], gs));
      nl += c->sp_glaunches[g];
      CUDA_TRY(cudaEventRecord(c->sp_join[g], gs));
      CUDA_TRY(cudaStreamWaitEvent(st, c->sp_join[g], 0));
    }
    c->sp_graph_built = true;
    c->k_pending = c->k_early = false;
    // the last scatter that read the step's K values ran inside the graphs
    CUDA_TRY(cudaEventRecord(c->k_free, st));
    launches += nl;
  } else {
    // direct launches (FETI_SP_GRAPH=0 or FETI_DEBUG_SYNC): one init + scatter
    // over every subdomain, then the groups' column sequences round-robin on
    // their own streams; feti_assemble runs each group's assembly
    c->sp_graph_fused = false;
    if (c->k_pending && c->k_early) {
      CUDA_TRY(cudaStreamWaitEvent(st, c->k_ready, 0));
      c->k_pending = c->k_early = false;
    }
    launch_sp_init(c->d_sp_init, c->n_sp_init, c->d_spsub, st);
    if (c->k_pending) {
      CUDA_TRY(cudaStreamWaitEvent(st, c->k_ready, 0));
      c->k_pending = false;
    }
    launch_sp_trace(c->d_spsub, ns, st);
    launch_sp_scatter(c->d_spsub, 0, ns, c->sp_max_n, st);
    CUDA_TRY(cudaEventRecord(c->k_free, st));
    CUDA_TRY(cudaGetLastError());
    FETI_DEBUG_SYNC(st);
    launches = 3;
    CUDA_TRY(cudaEventRecord(c->ev[2], st));
    for (int g = 0; g < G; ++g) CUDA_TRY(cudaStreamWaitEvent(c->sp_streams[g], c->ev[2], 0));
    for (int j = 0; j < c->sp_maxTq; ++j)
      for (int g = 0; g < G; ++g) {
        const size_t gj = (size_t)g * c->sp_maxTq + j;
        cudaStream_t gs = c->sp_streams[g];
        const auto a = c->sp_acc_rng[gj], d = c->sp_diag_rng[gj], pp = c->sp_panel_rng[gj];
        launch_sp_gemm(c->d_sp_tasks + a.first, a.second, c->d_sp_pairs, gs);
        launch_sp_potrf(c->d_sp_diag + d.first, d.second, c->d_bad, gs);
        launch_sp_gemm(c->d_sp_tasks + pp.first, pp.second, c->d_sp_pairs, gs);
        launches += (a.second > 0) + (d.second > 0) + (pp.second > 0);
        CUDA_TRY(cudaGetLastError());
        FETI_DEBUG_SYNC(gs);
      }
    for (int g = 0; g < G; ++g) {
      CUDA_TRY(cudaEventRecord(c->sp_join[g], c->sp_streams[g]));
      CUDA_TRY(cudaStreamWaitEvent(st, c->sp_join[g], 0));
    }
  }
  c->sp_graph_used = use_graph;
  c->sp_assembled_in_graph = use_graph && c->sp_graph_fused;
  // the factorization end on the context stream (timing only); no host sync:
  // feti_assemble runs each group's assembly right behind its factorization
  // on the group's stream and checks the pivots once everything finished
  CUDA_TRY(cudaEventRecord(c->sp_ev[1], st));
  c->stats.flops_factor_exec = c->sp_flops;
  c->stats.flops_factor_alg = c->sp_flops_scalar;
  c->stats.launches_factorize = launches;
  for (auto& s : c->subs) s.factor_set = true;
  c->tiles_fresh = true;
  c->sp_pending_check = true;
  return FETI_OK;
}

// An apply reads F~, the shared partial buffer and (implicit) the tiles on a
// caller stream; mark its end so the next factorize/assemble, which rewrite
// them on the library's streams, wait for it (write-after-read).
int mark_apply(feti_ctx* c, cudaStream_t st) {
  CUDA_TRY(cudaEventRecord(c->apply_done, st));
  c->apply_pending = true;
  return FETI_OK;
}

int wait_applies(feti_ctx* c) {
  if (c->apply_pending) {
    CUDA_TRY(cudaStreamWaitEvent(c->stream, c->apply_done, 0));
    c->apply_pending = false;
  }
  return FETI_OK;
}

// Sparse route: queue one slot's K values (and, when it changed, its kernel
// basis + U1 = B~ Q) on copy_stream; factorize_sparse waits for k_ready
// after zeroing the pool.  The caller keeps `data` alive and unchanged
// until feti_assemble returns; Q and U1 are staged in the slot's own host
// buffers.
// the slot's factorization group may start once its copies landed (the
// group's step graph waits for k_ready_grp, recorded after each of its slots)
int mark_group_ready(feti_ctx* c, int slot) {
  if (slot >= 0 && slot < (int)c->sp_group_of.size())
    CUDA_TRY(cudaEventRecord(c->k_ready_grp[c->sp_group_of[slot]], c->copy_stream));
  return FETI_OK;
}

int stiffness_values_async(feti_ctx* c, SubHost& s, const double* data, const double* Q) {
  if (!c->k_pending) {
    CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->k_free, 0));   // the last scatter read the old values
    c->k_pending = true;
  }
  CUDA_TRY(cudaMemcpyAsync(s.d_kdata, data, (size_t)s.k_nnz * 8, cudaMemcpyHostToDevice, c->copy_stream));
  const int64_t n = s.sp_n, r = s.kr;
  if (r > 0 && Q && (s.h_Q.empty() || std::memcmp(s.h_Q.data(), Q, (size_t)(n * r) * 8) != 0)) {
    s.h_Q.assign(Q, Q + n * r);
    // U1 = B~ Q in sorted column order: row a = sign_a Q[dof_a]
    const size_t rows = (size_t)s.P * TB;
    s.h_U1.assign(rows * r, 0.0);
    for (int64_t a = 0; a < s.m; ++a) {
      const int64_t dof = s.sp_perm[s.r_sorted[a]];
      for (int64_t q = 0; q < r; ++q) s.h_U1[a * r + q] = s.s_sorted[a] * Q[dof * r + q];
    }
    if (!s.d_U1) {
      int rc;
      if ((rc = dev_alloc(c, (void**)&s.d_U1, rows * r * 8, true))) return rc;
      if ((rc = dev_alloc(c, (void**)&s.d_U2W, rows * 2 * r * 8, true))) return rc;
    }
    CUDA_TRY(cudaMemcpyAsync(s.d_Q, s.h_Q.data(), (size_t)(n * r) * 8, cudaMemcpyHostToDevice, c->copy_stream));
    c->k_early = true;
    CUDA_TRY(cudaMemcpyAsync(s.d_U1, s.h_U1.data(), rows * r * 8, cudaMemcpyHostToDevice, c->copy_stream));
  } else if (r > 0 && s.h_Q.empty()) {
    return fail(FETI_ERR_ARG, "the first hand-over of a slot needs its kernel basis");
  }
  CUDA_TRY(cudaEventRecord(c->k_ready, c->copy_stream));
  mark_group_ready(c, (int)(&s - c->subs.data()));
  return FETI_OK;
}

}  // namespace

extern "C" {

int feti_abi_version(void) { return FETI_B200_ABI_VERSION; }

const char* feti_last_error(void) { return g_err.c_str(); }

int feti_create(int device, feti_ctx** out) {
  if (!out) return fail(FETI_ERR_ARG, "out is NULL");
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(FETI_ERR_ARG, "device %d out of range (%d devices)", device, ndev);
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(FETI_ERR_CUDA, "device %d is sm_%d%d; this build targets sm_100a", device, prop.major, prop.minor);
  feti_ctx* c = new feti_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  CUDA_TRY(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  for (int i = 0; i < feti_ctx::kWaveStreams; ++i) {
    CUDA_TRY(cudaStreamCreateWithFlags(&c->wave_streams[i], cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&c->wave_join[i], cudaEventDisableTiming));
  }
  for (auto& e : c->ev) CUDA_TRY(cudaEventCreate(&e));
  CUDA_TRY(cudaEventCreateWithFlags(&c->apply_done, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&c->x_sum_done, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&c->k_ready, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&c->k_free, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(c->k_free, c->stream));
  CUDA_TRY(configure_kernels());
  *out = c;
  return FETI_OK;
}

int feti_destroy(feti_ctx* c) {
  if (!c) return FETI_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
  for (void* p : c->allocs) cudaFree(p);
  for (auto& s : c->subs)
    if (s.ev_upload) cudaEventDestroy(s.ev_upload);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->wave_ev)
    if (e) cudaEventDestroy(e);
  for (int i = 0; i < feti_ctx::kWaveStreams; ++i) {
    if (c->wave_join[i]) cudaEventDestroy(c->wave_join[i]);
    if (c->wave_streams[i]) cudaStreamDestroy(c->wave_streams[i]);
  }
  for (auto& e : c->sp_ev)
    if (e) cudaEventDestroy(e);
  for (int g = 0; g < feti_ctx::kSpStreams; ++g) {
    if (c->sp_join[g]) cudaEventDestroy(c->sp_join[g]);
    if (c->sp_fend[g]) cudaEventDestroy(c->sp_fend[g]);
    if (c->k_ready_grp[g]) cudaEventDestroy(c->k_ready_grp[g]);
    if (c->sp_gexec[g]) cudaGraphExecDestroy(c->sp_gexec[g]);
    if (c->sp_streams[g]) cudaStreamDestroy(c->sp_streams[g]);
  }
  for (double* pp : c->x_open) cudaIpcCloseMemHandle(pp);
  if (c->apply_done) cudaEventDestroy(c->apply_done);
  if (c->x_sum_done) cudaEventDestroy(c->x_sum_done);
  if (c->k_ready) cudaEventDestroy(c->k_ready);
  for (auto& ge : c->pc_graph)
    if (ge) cudaGraphExecDestroy(ge);
  if (c->pc_sc_host) cudaFreeHost(c->pc_sc_host);
  if (c->k_free) cudaEventDestroy(c->k_free);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  delete c;
  return FETI_OK;
}

int feti_add_subdomain(feti_ctx* c, int64_t n, int64_t m, const int64_t* first_row, const double* sign,
                       const int64_t* gids, const int64_t* up, const int64_t* ui, int64_t nnz,
                       int64_t* out_slot) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (c->finalized) return fail(FETI_ERR_LIFECYCLE, "prepare was already called on this operator");
  if (n <= 0 || m < 0) return fail(FETI_ERR_ARG, "bad subdomain size n=%lld m=%lld", (long long)n, (long long)m);
  if (n > (1 << 28)) return fail(FETI_ERR_ARG, "subdomain too large");
  if (m > 0 && (!first_row || !sign || !gids)) return fail(FETI_ERR_ARG, "NULL index arrays");
  const bool dense = (up == nullptr);
  if (dense && nnz != n * (n + 1) / 2)
    return fail(FETI_ERR_ARG, "dense factor needs n(n+1)/2 = %lld values, got %lld", (long long)(n * (n + 1) / 2),
                (long long)nnz);
  SubHost s;
  s.n = n;
  s.m = m;
  s.nnz = nnz;
  s.dense = dense;
  s.src = dense ? SRC_RAW_DENSE : SRC_RAW_SPARSE;
  s.T = (int)((n + TB - 1) / TB);
  s.P = (int)((m + TB - 1) / TB);
  s.T32 = (int)((m + AT - 1) / AT);
  for (int64_t j = 0; j < m; ++j) {
    if (first_row[j] < 0 || first_row[j] >= n)
      return fail(FETI_ERR_ARG, "constraint row %lld hits factor row %lld outside [0, %lld)", (long long)j,
                  (long long)first_row[j], (long long)n);
    if (j > 0 && gids[j] <= gids[j - 1]) return fail(FETI_ERR_ARG, "multiplier ids must be strictly ascending");
  }
  if (!dense) {
    if (!ui) return fail(FETI_ERR_ARG, "ui is NULL");
    if (up[0] != 0 || up[n] != nnz) return fail(FETI_ERR_ARG, "pattern pointer does not match nnz");
    for (int64_t j = 0; j < n; ++j) {
      if (up[j + 1] <= up[j] || ui[up[j]] != j)
        return fail(FETI_ERR_SINGULAR, "factor row %lld has no leading diagonal entry", (long long)j);
    }
    s.up.assign(up, up + n + 1);
    s.ui.assign(ui, ui + nnz);
  }
  // sort columns of P B~^T by their first nonzero row (stable)
  s.colperm.resize(m);
  std::iota(s.colperm.begin(), s.colperm.end(), 0);
  std::stable_sort(s.colperm.begin(), s.colperm.end(),
                   [&](int64_t a, int64_t b) { return first_row[a] < first_row[b]; });
  s.r_sorted.assign((size_t)s.P * TB, BIG_ROW);
  s.s_sorted.assign((size_t)s.P * TB, 0.0);
  s.gids_sorted.assign((size_t)s.T32 * AT, -1);
  for (int64_t a = 0; a < m; ++a) {
    const int64_t j = s.colperm[a];
    s.r_sorted[a] = (int)first_row[j];
    s.s_sorted[a] = sign[j];
    s.gids_sorted[a] = (int)gids[j];
  }
  s.panel_minrow.resize(s.P);
  for (int p = 0; p < s.P; ++p) s.panel_minrow[p] = s.r_sorted[(size_t)p * TB];
  // pruning: nothing above the smallest first row is ever read
  s.smin = s.P > 0 ? s.panel_minrow[0] / TB : s.T;
  const int64_t j0 = std::min<int64_t>((int64_t)s.smin * TB, n);
  s.raw_off = dense ? (j0 * n - j0 * (j0 - 1) / 2) : (j0 < n ? up[j0] : nnz);
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaEventCreateWithFlags(&s.ev_upload, cudaEventDisableTiming));
  c->subs.push_back(std::move(s));
  if (out_slot) *out_slot = (int64_t)c->subs.size() - 1;
  return FETI_OK;
}

int feti_set_strategy(feti_ctx* c, int strategy) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (c->finalized) return fail(FETI_ERR_LIFECYCLE, "the strategy must be chosen before finalize");
  if (strategy != FETI_STRATEGY_EXPLICIT && strategy != FETI_STRATEGY_IMPLICIT)
    return fail(FETI_ERR_ARG, "unknown strategy %d", strategy);
  c->implicit = strategy == FETI_STRATEGY_IMPLICIT;
  return FETI_OK;
}

int feti_set_path(feti_ctx* c, int path) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (c->finalized) return fail(FETI_ERR_LIFECYCLE, "the path must be chosen before finalize");
  if (path != FETI_PATH_SYRK && path != FETI_PATH_TRSM) return fail(FETI_ERR_ARG, "unknown path %d", path);
  c->path_trsm = path == FETI_PATH_TRSM;
  return FETI_OK;
}

int feti_finalize(feti_ctx* c, int64_t n_multipliers) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (c->finalized) return fail(FETI_ERR_LIFECYCLE, "prepare was already called on this operator");
  if (n_multipliers < 0 || n_multipliers >= (int64_t)1 << 31) return fail(FETI_ERR_ARG, "bad n_multipliers");
  if (c->sparse_factor && c->dual_rhs)
    for (auto& s : c->subs)
      if (s.sp_r >= 8) return fail(FETI_ERR_ARG, "the device dual rhs needs a kernel dimension < 8");
  CUDA_TRY(cudaSetDevice(c->device));
  c->n_mult = n_multipliers;
  for (auto& s : c->subs)
    for (int a = 0; a < s.m; ++a)
      if (s.gids_sorted[a] >= n_multipliers) return fail(FETI_ERR_ARG, "multiplier id out of range");

  if (c->device_factor) {
    // the factorization and full solves need every tile (tbase = 0) and run
    // one batched launch per block step: every slot is given the largest
    // block count, rows >= n being identity (kreg_fill_kernel) -- decoupled,
    // so L, X and F~ of the real rows are unchanged
    for (auto& s : c->subs) c->uniform_T = std::max(c->uniform_T, s.T);
    for (auto& s : c->subs) {
      s.tbase = 0;
      if (s.P == 0) s.smin = c->uniform_T;
      s.T = c->uniform_T;
    }
  }
  // capacity check before allocating anything large
  size_t need = 0;
  if (c->sparse_factor)
    for (size_t i = 0; i < c->subs.size(); ++i) {
      SubHost& s = c->subs[i];
      if (!s.sp_pattern) return fail(FETI_ERR_LIFECYCLE, "slot %zu has no sparse pattern", i);
      sp_symbolic(s.sp_n, s.sp_kptr.data(), s.sp_kind.data(), s.sp_iperm.data(), s.n, s.sp_r, s.smin, &s.sp,
                  c->dual_rhs);
      need += (size_t)s.sp.ntiles * TILE * 8;
    }
  for (auto& s : c->subs) {
    const int64_t tb = c->device_factor ? 0 : s.smin;
    if (!c->sparse_factor) need += (size_t)(s.T - tb) * (s.T - tb + 1) / 2 * TILE * 8;   // tiles
    if (!c->implicit) {
      need += (size_t)s.P * (s.T - s.smin) * TILE * 8;   // X panels
      need += (size_t)s.f_tiles() * ATILE * 8;          // F~
      if (c->path_trsm)                                  // U, Y panels + transposed trailing tiles
        need += (size_t)(2 * s.P + (s.T - s.smin + 1) / 2) * (s.T - s.smin) * TILE * 8;
    }
  }
  size_t fr = 0, tot = 0;
  CUDA_TRY(cudaMemGetInfo(&fr, &tot));
  if (need > fr)
    return fail(FETI_ERR_CAPACITY,
                "device pool of %zu bytes (%zu free) cannot hold the %zu-byte explicit operator workspace", tot,
                fr, need);

  int rc;
  if (!c->device_factor)
    for (auto& s : c->subs) s.tbase = s.smin;
  for (auto& s : c->subs) {
    if (c->sparse_factor) {
      if ((rc = dev_alloc(c, (void**)&s.d_pool, (size_t)std::max<int64_t>(s.sp.ntiles, 1) * TILE * 8, false)))
        return rc;
      s.d_tiles = s.d_pool + (size_t)s.sp.trail_base * TILE;
      if ((rc = upload(c, &s.d_tmap, s.sp.tmap))) return rc;
      if ((rc = upload(c, &s.d_fix, s.sp_fix))) return rc;
      if (c->dual_rhs) {
        if ((rc = dev_alloc(c, (void**)&s.d_fproj, (size_t)std::max<int64_t>(s.sp_n, 1) * 8, true))) return rc;
        if ((rc = dev_alloc(c, (void**)&s.d_qtf, (size_t)std::max(s.sp_r, 1) * 8, true))) return rc;
        if ((rc = dev_alloc(c, (void**)&s.d_U2f, (size_t)std::max(s.P, 1) * TB * 8, true))) return rc;
        CUDA_TRY(cudaMemset(s.d_fproj, 0, (size_t)std::max<int64_t>(s.sp_n, 1) * 8));
        CUDA_TRY(cudaMemset(s.d_qtf, 0, (size_t)std::max(s.sp_r, 1) * 8));
      }
    } else if ((rc = dev_alloc(c, (void**)&s.d_tiles, (size_t)std::max<int64_t>(s.l_tiles(), 1) * TILE * 8, false))) {
      return rc;
    }
    if (!c->implicit) {
      if ((rc = dev_alloc(c, (void**)&s.d_X, (size_t)std::max(s.P, 1) * std::max(s.T - s.smin, 1) * TILE * 8,
                          false)))
        return rc;
      if ((rc = dev_alloc(c, (void**)&s.d_F, (size_t)std::max<int64_t>(s.f_tiles(), 1) * ATILE * 8, true)))
        return rc;
      if (c->path_trsm) {
        const size_t pb = (size_t)std::max(s.P, 1) * std::max(s.T - s.smin, 1) * TILE * 8;
        const int64_t tt = s.T - s.smin;
        if ((rc = dev_alloc(c, (void**)&s.d_U, pb, false))) return rc;
        if ((rc = dev_alloc(c, (void**)&s.d_Y, pb, false))) return rc;
        if ((rc = dev_alloc(c, (void**)&s.d_Lt, (size_t)std::max<int64_t>(tt * (tt + 1) / 2, 1) * TILE * 8, false)))
          return rc;
      }
    }
    if ((rc = upload(c, &s.d_r, s.r_sorted))) return rc;
    if ((rc = upload(c, &s.d_s, s.s_sorted))) return rc;
    if ((rc = upload(c, &s.d_g, s.gids_sorted))) return rc;
    if ((rc = upload(c, &s.d_pmin, s.panel_minrow))) return rc;
    if (!s.dense) {
      if ((rc = upload(c, &s.d_up, s.up))) return rc;
      if ((rc = upload(c, &s.d_ui, s.ui))) return rc;
      std::vector<int64_t>().swap(s.up);
      std::vector<int64_t>().swap(s.ui);
    }
  }
  if ((rc = dev_alloc(c, (void**)&c->d_subdev, c->subs.size() * sizeof(SubDev), true))) return rc;

  // ---- work lists (largest work first where it varies)
  std::vector<int4> wu, wd, ws, wc, wy;
  double trsm_alg = 0, syrk_alg = 0, trsm_exec = 0, syrk_exec = 0, scale_exec = 0;
  const double tb3 = 2.0 * TB * TB * TB;
  for (int si = 0; si < (int)c->subs.size(); ++si) {
    const SubHost& s = c->subs[si];
    // dense pattern: the kernels read the packed factor directly (no unpack);
    // sparse pattern: zero-fill + scatter into tiles first
    if (!s.dense)
      for (int K = s.smin; K < s.T; ++K)
        for (int L = s.smin; L <= K; ++L) wu.push_back(make_int4(si, K, L, 0));
    // device factorization: every block row is scaled (full solves need it)
    const int k0 = c->device_factor ? 0 : s.smin;
    for (int k = k0; k < s.T; ++k) wd.push_back(make_int4(si, k, 0, 0));
    for (int k = s.T - 1; k > k0; --k) ws.push_back(make_int4(si, k, 0, 0));
    const double tt = s.T - k0;
    scale_exec += tt * (tt - 1) / 2 * 2.0 * (2.0 * 64 * 32 * 32 * (1 + 2 + 3 + 4));
    for (int p = 0; p < s.P && !c->implicit; ++p) {
      wc.push_back(make_int4(si, p, 0, 0));
      const double s0 = s.panel_minrow[p] / TB;
      trsm_exec += tb3 * (s.T - 1 - s0) * (s.T - s0) / 2.0;
      if (c->path_trsm) {   // backward chain over [smin, T) + inv(L_kk)^T per block row
        const double tt = s.T - s.smin;
        trsm_exec += tb3 * (tt * (tt - 1) / 2.0 + tt);
      }
    }
    const int rend = (int)((s.n + KS - 1) / KS * KS);
    for (int I = 0; I < s.P && !c->implicit && !c->path_trsm; ++I)
      for (int J = I; J < s.P; ++J) {
        wy.push_back(make_int4(si, I, J, 0));
        const int rs = std::max(s.panel_minrow[I], s.panel_minrow[J]) & ~(KS - 1);
        syrk_exec += 2.0 * TB * TB * (rend - rs);
      }
    for (int a = 0; a < s.m; ++a) {
      const double d = (double)(s.n - s.r_sorted[a]);
      trsm_alg += d * d;
      syrk_alg += 2.0 * d * (a + 1);
    }
  }
  // chains: longest first so the tail is short
  std::stable_sort(ws.begin(), ws.end(), [&](const int4& a, const int4& b) {
    return a.y - c->subs[a.x].tbase > b.y - c->subs[b.x].tbase;
  });
  std::sort(wc.begin(), wc.end(), [&](const int4& a, const int4& b) {
    const SubHost& sa = c->subs[a.x];
    const SubHost& sb = c->subs[b.x];
    const double la = sa.T - sa.panel_minrow[a.y] / TB, lb = sb.T - sb.panel_minrow[b.y] / TB;
    return la > lb;
  });
  std::sort(wy.begin(), wy.end(), [&](const int4& a, const int4& b) {
    const SubHost& sa = c->subs[a.x];
    const SubHost& sb = c->subs[b.x];
    const int la = (int)sa.n - std::max(sa.panel_minrow[a.y], sa.panel_minrow[a.z]);
    const int lb = (int)sb.n - std::max(sb.panel_minrow[b.y], sb.panel_minrow[b.z]);
    return la > lb;
  });

  // ---- upload/compute waves (host-factor pipeline), largest work first
  {
    std::vector<int> order(c->subs.size());
    std::iota(order.begin(), order.end(), 0);
    std::vector<double> work(c->subs.size(), 0.0);
    for (size_t si = 0; si < c->subs.size(); ++si) {
      const SubHost& s = c->subs[si];
      for (int p = 0; p < s.P; ++p) {
        const double len = s.T - s.panel_minrow[p] / TB;
        work[si] += len * len;
      }
    }
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return work[a] > work[b]; });
    int nw = (int)std::min<size_t>(c->subs.size(), 8);
    if (c->sparse_factor) {
      // sparse route: the waves are the factorization groups (contiguous
      // subdomain ranges), so each group's assembly follows its own
      // factorization on its stream
      const char* genv = getenv("FETI_SP_GROUPS");
      const int ns = (int)c->subs.size();
      int G = genv ? atoi(genv) : 8;
      G = std::max(1, std::min(std::min(G, (int)feti_ctx::kSpStreams), std::max(ns, 1)));
      c->sp_groups = G;
      nw = G;
      c->waves.assign(nw, {});
      for (int si = 0; si < ns; ++si) c->waves[(int)((int64_t)si * G / ns)].push_back(si);
    } else {
      c->waves.assign(nw, {});
      for (size_t k = 0; k < order.size(); ++k) c->waves[k * nw / order.size()].push_back(order[k]);
    }
    std::vector<int> wave_of(c->subs.size());
    for (int w = 0; w < nw; ++w)
      for (int si : c->waves[w]) wave_of[si] = w;
    const std::vector<int4>* lists[5] = {&wu, &wd, &ws, &wc, &wy};
    for (int kind = 0; kind < 5; ++kind) {
      std::vector<int4> v;
      c->wv_range[kind].assign(nw, {0, 0});
      for (int w = 0; w < nw; ++w) {
        const int b = (int)v.size();
        for (const int4& x : *lists[kind])
          if (wave_of[x.x] == w) v.push_back(x);
        c->wv_range[kind][w] = {b, (int)v.size() - b};
      }
      if ((rc = upload(c, &c->d_wv[kind], v))) return rc;
    }
    c->wave_ev.resize(nw);
    for (auto& e : c->wave_ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }

  // ---- apply work: every subdomain's packed upper triangle of 32x32 tiles is
  // split into SB x SB-tile super-blocks (I <= J); the concatenated tile list
  // of all super-blocks is cut into one contiguous, equal range per SM
  // (persistent CTAs), each range into segments at super-block bounds.  The
  // kernel's accumulators span one super-block (<= 2 x SBE multipliers), so
  // neither the warp count nor the subdomain size is limited by shared memory.
  // warps per apply CTA: bytes in flight bound the kernel (two 8 KB tile
  // loads per warp); the super-block edge is the largest the warps'
  // accumulators fit, balanced so the largest subdomain splits into equal
  // blocks (fewer, larger segments: less per-segment refill and combine)
  c->apply_nw = 8;
  if (const char* wenv = getenv("FETI_APPLY_WARPS")) c->apply_nw = std::max(1, std::min(APPLY_MAX_WARPS, atoi(wenv)));
  bool compact = false;
  {
    int maxT32 = 1;
    for (auto& s : c->subs) maxT32 = std::max(maxT32, s.T32);
    const int cap = std::min(apply_max_sb(c->apply_nw), 64);
    const int nbk = (maxT32 + cap - 1) / cap;
    c->apply_sb = (maxT32 + nbk - 1) / nbk;
    // every subdomain in one block with the compact layout when it fits
    // (one segment per subdomain slice: the fewest pipeline restarts)
    compact = maxT32 <= apply_max_compact(c->apply_nw);
    if (compact) c->apply_sb = maxT32;
    if (const char* senv = getenv("FETI_APPLY_SB")) {
      c->apply_sb = std::max(1, std::min(cap, atoi(senv)));
      compact = false;
    }
    // many small subdomains (every subdomain a few hundred tiles): two
    // 4-warp CTAs per SM, so one CTA streams while the other restarts its
    // pipeline at a subdomain boundary (same warps per SM)
    c->apply_cps = 1;
    const char* cenv = getenv("FETI_APPLY_CPS");
    if ((cenv ? atoi(cenv) == 2 : (compact && maxT32 <= 24 && !getenv("FETI_APPLY_WARPS")))) {
      c->apply_cps = 2;
      c->apply_nw = 4;
    }
  }
  const int SB = c->apply_sb, SBE = SB * AT;
  struct Blk { int sub, I, J; int64_t tiles; };
  std::vector<Blk> blks;
  int64_t total_tiles = 0;
  for (int si = 0; si < (int)c->subs.size(); ++si) {
    const SubHost& s = c->subs[si];
    if (s.m == 0) continue;
    const int nb = (s.T32 + SB - 1) / SB;
    for (int I = 0; I < nb; ++I)
      for (int J = I; J < nb; ++J) {
        const int64_t h = std::min(SB, s.T32 - I * SB), w = std::min(SB, s.T32 - J * SB);
        const int64_t nt = (I == J) ? h * (h + 1) / 2 : h * w;
        blks.push_back(Blk{si, I, J, nt});
        total_tiles += nt;
      }
  }
  const int64_t ncta =
      std::max<int64_t>(1, std::min<int64_t>((int64_t)c->num_sms * c->apply_cps, (total_tiles + 63) / 64));
  std::vector<ApplySeg> asegs;
  std::vector<int> seg_ptr;
  int64_t poff = 0;
  double apply_alg = 16.0 * (double)c->n_mult, apply_exec = 16.0 * (double)c->n_mult;
  {
    size_t bi = 0;
    int64_t bbase = 0;    // first global tile of block bi
    for (int64_t b = 0; b < ncta; ++b) {
      seg_ptr.push_back((int)asegs.size());
      const int64_t g0 = total_tiles * b / ncta, g1 = total_tiles * (b + 1) / ncta;
      while (bi < blks.size() && bbase + blks[bi].tiles <= g0) bbase += blks[bi++].tiles;
      for (size_t k = bi, kb = bbase; k < blks.size() && (int64_t)kb < g1; kb += blks[k++].tiles) {
        const int64_t lo = std::max<int64_t>(g0, kb), hi = std::min<int64_t>(g1, kb + blks[k].tiles);
        if (lo >= hi) continue;
        const Blk& B = blks[k];
        const SubHost& s = c->subs[B.sub];
        const int h = std::min(SB, s.T32 - B.I * SB), w = std::min(SB, s.T32 - B.J * SB);
        ApplySeg sg{B.sub, B.I, B.J, (int)(lo - kb), (int)(hi - kb), 0, poff, -1};
        poff += (int64_t)h * AT;
        if (B.I != B.J) {
          sg.out_c = poff;
          poff += (int64_t)w * AT;
        }
        asegs.push_back(sg);
      }
    }
    seg_ptr.push_back((int)asegs.size());
  }
  for (int si = 0; si < (int)c->subs.size(); ++si) {
    const SubHost& s = c->subs[si];
    apply_alg += 8.0 * s.m * (s.m + 1) / 2 + s.m * (8.0 + 16.0 + 4.0);
    apply_exec += 8.0 * ATILE * s.f_tiles() + s.T32 * AT * 12.0;
  }
  apply_exec += 16.0 * poff;
  if (compact) c->apply_sb = -SB;   // the kernel's compact-layout flag
  // partial positions of every (subdomain, local multiplier), in segment order
  std::vector<std::vector<std::vector<int64_t>>> lp(c->subs.size());
  for (int si = 0; si < (int)c->subs.size(); ++si) lp[si].assign(c->subs[si].m, {});
  for (const ApplySeg& sg : asegs) {
    const SubHost& s = c->subs[sg.sub];
    const int h = std::min(SB, s.T32 - sg.I * SB), w = std::min(SB, s.T32 - sg.J * SB);
    for (int a = 0; a < h * AT; ++a) {
      const int la = sg.I * SBE + a;
      if (la < s.m) lp[sg.sub][la].push_back(sg.out_r + a);
    }
    if (sg.I != sg.J)
      for (int a = 0; a < w * AT; ++a) {
        const int la = sg.J * SBE + a;
        if (la < s.m) lp[sg.sub][la].push_back(sg.out_c + a);
      }
  }
  // contributions per global multiplier, in registration (gather) order
  std::vector<int64_t> ridx;
  std::vector<std::vector<int4>> per_g((size_t)c->n_mult);
  for (int si = 0; si < (int)c->subs.size(); ++si) {
    const SubHost& s = c->subs[si];
    for (int a = 0; a < s.m; ++a) {
      const int b0 = (int)ridx.size();
      ridx.insert(ridx.end(), lp[si][a].begin(), lp[si][a].end());
      per_g[s.gids_sorted[a]].push_back(make_int4(a, b0, (int)ridx.size(), si));
    }
  }
  std::vector<std::vector<std::vector<int64_t>>>().swap(lp);
  std::vector<int> cptr((size_t)c->n_mult + 1, 0);
  std::vector<int4> cent;
  for (int64_t g = 0; g < c->n_mult; ++g) {
    cptr[g] = (int)cent.size();
    cent.insert(cent.end(), per_g[g].begin(), per_g[g].end());
  }
  cptr[c->n_mult] = (int)cent.size();


  if ((rc = upload(c, &c->d_w_unpack, wu))) return rc;
  if ((rc = upload(c, &c->d_w_diag, wd))) return rc;
  if ((rc = upload(c, &c->d_w_scale, ws))) return rc;
  if ((rc = upload(c, &c->d_w_chain, wc))) return rc;
  if ((rc = upload(c, &c->d_w_syrk, wy))) return rc;
  if ((rc = upload(c, &c->d_apply_segs, asegs))) return rc;
  if ((rc = upload(c, &c->d_apply_seg_ptr, seg_ptr))) return rc;
  if ((rc = upload(c, &c->d_ridx, ridx))) return rc;
  c->h_cptr = cptr;
  if ((rc = upload(c, &c->d_cptr, cptr))) return rc;
  if ((rc = upload(c, &c->d_cent, cent))) return rc;
  if ((rc = dev_alloc(c, (void**)&c->d_part, (size_t)std::max<int64_t>(poff, 1) * 8, true))) return rc;
  {
    std::vector<int64_t> ioff(c->subs.size());
    int64_t tot = 0;
    for (size_t si = 0; si < c->subs.size(); ++si) {
      ioff[si] = tot;
      tot += c->subs[si].m;
      c->impl_max_blocks = std::max(c->impl_max_blocks, c->subs[si].T - c->subs[si].smin);
    }
    if ((rc = upload(c, &c->d_impl_off, ioff))) return rc;
    if ((rc = dev_alloc(c, (void**)&c->d_impl_part, (size_t)std::max<int64_t>(tot, 1) * 8, true))) return rc;
    if (implicit_smem(c->impl_max_blocks) > 227 * 1024)
      c->impl_max_blocks = -1;   // implicit apply unavailable for this size
    else
      CUDA_TRY(configure_implicit(c->impl_max_blocks));
    if (c->implicit && c->sparse_factor && c->impl_max_blocks < 0)
      return fail(FETI_ERR_CAPACITY, "implicit strategy: subdomain too large for the cluster sweep's shared memory");
  }
  if ((rc = dev_alloc(c, (void**)&c->d_p, (size_t)std::max<int64_t>(c->n_mult, 1) * 8, true))) return rc;
  if ((rc = dev_alloc(c, (void**)&c->d_q, (size_t)std::max<int64_t>(c->n_mult, 1) * 8, true))) return rc;
  c->n_unpack = (int)wu.size();
  c->n_diag = (int)wd.size();
  c->n_scale = (int)ws.size();
  c->n_chain = (int)wc.size();
  c->n_syrk = (int)wy.size();
  c->n_apply = (int)ncta;

  feti_stats& st = c->stats;
  st.flops_trsm_alg = trsm_alg;
  st.flops_syrk_alg = syrk_alg;
  st.flops_trsm_exec = trsm_exec;
  st.flops_syrk_exec = syrk_exec;
  st.flops_scale_exec = scale_exec;
  st.apply_bytes_alg = apply_alg;
  st.apply_bytes_exec = apply_exec;
  st.n_subdomains = (int64_t)c->subs.size();
  st.n_multipliers = c->n_mult;
  st.launches_apply = 2;
  if (c->device_factor) {
    const size_t ns = c->subs.size();
    if ((rc = dev_alloc(c, (void**)&c->d_fsub, ns * sizeof(FactorSub), true))) return rc;
    if ((rc = dev_alloc(c, (void**)&c->d_dinv, ns * TILE * 8, false))) return rc;
    if ((rc = dev_alloc(c, (void**)&c->d_bad, ns * sizeof(int), false))) return rc;
    std::vector<int64_t> voff(ns + 1, 0);
    std::vector<int> slots(ns);
    for (size_t si = 0; si < ns; ++si) {
      voff[si + 1] = voff[si] + c->subs[si].n;
      slots[si] = (int)si;
    }
    if ((rc = upload(c, &c->d_vec_off, voff))) return rc;
    if ((rc = upload(c, &c->d_slots, slots))) return rc;
    if ((rc = dev_alloc(c, (void**)&c->d_sb, (size_t)std::max<int64_t>(voff[ns], 1) * 8, true))) return rc;
    if ((rc = dev_alloc(c, (void**)&c->d_sx, (size_t)std::max<int64_t>(voff[ns], 1) * 8, true))) return rc;
    CUDA_TRY(configure_factor(c->uniform_T));
  }
  if (c->sparse_factor && (rc = build_sparse_tasks(c))) return rc;
  CUDA_TRY(cudaDeviceSynchronize());
  c->finalized = true;
  return FETI_OK;
}

int feti_set_factor(feti_ctx* c, int64_t slot, const double* values, int64_t nnz, int where) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->finalized) return fail(FETI_ERR_LIFECYCLE, "preprocess before prepare");
  if (slot < 0 || slot >= (int64_t)c->subs.size()) return fail(FETI_ERR_ARG, "slot %lld out of range", (long long)slot);
  SubHost& s = c->subs[slot];
  if (nnz != s.nnz)
    return fail(FETI_ERR_ARG, "factor value buffer has the wrong length (%lld, expected %lld)", (long long)nnz,
                (long long)s.nnz);
  if (!values) return fail(FETI_ERR_ARG, "values is NULL");
  CUDA_TRY(cudaSetDevice(c->device));
  if (where == FETI_FACTOR_DEVICE) {
    s.d_raw = values + s.raw_off;
    s.factor_from_host = false;
    s.h_values = nullptr;
  } else {
    if (!s.d_raw_own) {
      int rc = dev_alloc(c, (void**)&s.d_raw_own, (size_t)std::max<int64_t>(s.upload_count(), 1) * 8, true);
      if (rc) return rc;
    }
    // the copy itself is issued by feti_assemble, in wave order, so that
    // each wave's kernels start as soon as its factors have landed
    s.h_values = values;
    if (s.d_raw != s.d_raw_own) c->subdev_dirty = true;
    s.d_raw = s.d_raw_own;
    s.factor_from_host = true;
  }
  s.factor_set = true;
  if (where == FETI_FACTOR_DEVICE) c->subdev_dirty = true;
  return FETI_OK;
}

// Launch the five assembly kernels for one set of work lists on `st`.
static int launch_assembly(feti_ctx* c, cudaStream_t st, const int4* wu, int nu, const int4* wd, int nd,
                           const int4* ws, int ns, const int4* wc, int nc, const int4* wy, int ny,
                           const std::vector<int>& sparse_slots, cudaEvent_t* marks, int* launches) {
  // the sparse factorization already left inv(L_kk) in the trailing diagonal tiles
  const bool inv_ready = c->sparse_factor;
  if (marks) CUDA_TRY(cudaEventRecord(marks[0], st));
  launch_unpack(c->d_subdev, wu, nu, st);
  *launches += nu > 0;
  for (int si : sparse_slots) {
    launch_scatter_sparse(c->d_subdev, si, (int)(c->subs[si].n - (int64_t)c->subs[si].smin * TB), st);
    ++*launches;
  }
  CUDA_TRY(cudaGetLastError());
  FETI_DEBUG_SYNC(st);
  if (marks) CUDA_TRY(cudaEventRecord(marks[1], st));
  if (!inv_ready) {
    launch_diag_inverse(c->d_subdev, wd, nd, st);
    *launches += nd > 0;
  }
  CUDA_TRY(cudaGetLastError());
  FETI_DEBUG_SYNC(st);
  if (marks) CUDA_TRY(cudaEventRecord(marks[2], st));
  launch_block_scale(c->d_subdev, ws, ns, st);
  *launches += ns > 0;
  CUDA_TRY(cudaGetLastError());
  FETI_DEBUG_SYNC(st);
  if (marks) CUDA_TRY(cudaEventRecord(marks[3], st));
  launch_trsm_chain(c->d_subdev, wc, nc, st);
  *launches += nc > 0;
  CUDA_TRY(cudaGetLastError());
  FETI_DEBUG_SYNC(st);
  if (marks) CUDA_TRY(cudaEventRecord(marks[4], st));
  if (c->path_trsm) {
    // second solve + row gather (dualop.py:472-479) in the SYRK's place
    launch_trsm_path(c->d_subdev, wd, nd, wc, nc, st);
    *launches += (nd > 0) + 2 * (nc > 0);
  }
  launch_syrk(c->d_subdev, wy, ny, st);
  *launches += ny > 0;
  CUDA_TRY(cudaGetLastError());
  FETI_DEBUG_SYNC(st);
  if (marks) CUDA_TRY(cudaEventRecord(marks[5], st));
  return FETI_OK;
}

// One factorization group's interface assembly + correction on its stream
// (sparse route): TRSM chain, then U2/W and the SYRK with the correction in
// its epilogue (explicit "syrk"), the U2 sweep (implicit), or the second
// solve + gather and the correction pass (path "trsm").
static int sparse_group_assembly(feti_ctx* c, int g, cudaStream_t gs, int* launches) {
  const auto& r = c->wv_range;
  std::vector<int> none;
  const bool fused = !c->implicit && !c->path_trsm;   // the SYRK follows sp_u2 below
  int rc;
  if ((rc = launch_assembly(c, gs, c->d_wv[0] + r[0][g].first, r[0][g].second, c->d_wv[1] + r[1][g].first,
                            r[1][g].second, c->d_wv[2] + r[2][g].first, r[2][g].second, c->d_wv[3] + r[3][g].first,
                            r[3][g].second, c->d_wv[4] + r[4][g].first, fused ? 0 : r[4][g].second, none, nullptr,
                            launches)))
    return rc;
  if (c->implicit) {
    // no F~: U2 (and U2f) by the backward sweep; the apply adds the correction
    launch_implicit_u2(c->d_subdev, c->d_spsub, c->sp_sub_rng[g].first, c->sp_sub_rng[g].second, c->sp_u2_cols,
                       c->impl_max_blocks, gs);
    *launches += c->sp_u2_cols > 0;
  } else if (!c->path_trsm) {
    // U2/W from X, then the SYRK with the correction in its epilogue
    // (launch_assembly above ran without the SYRK: ny = 0)
    launch_sp_u2(c->d_subdev, c->d_spsub, c->d_sp_panels + c->sp_corr_rng[g].first, c->sp_corr_rng[g].second,
                 c->sp_u2_cols, gs);
    launch_syrk(c->d_subdev, c->d_wv[4] + r[4][g].first, r[4][g].second, gs);
    *launches += (c->sp_corr_rng[g].second > 0) + (r[4][g].second > 0);
  } else {
    launch_sp_correct(c->d_subdev, c->d_spsub, c->d_sp_panels + c->sp_corr_rng[g].first, c->sp_corr_rng[g].second,
                      c->sp_sub_rng[g].first, c->sp_sub_rng[g].second, c->sp_max_T32, c->sp_u2_cols, gs);
    *launches += 2;
  }
  CUDA_TRY(cudaGetLastError());
  return FETI_OK;
}

int feti_assemble(feti_ctx* c) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->finalized) return fail(FETI_ERR_LIFECYCLE, "preprocess before prepare");
  for (size_t i = 0; i < c->subs.size(); ++i)
    if (!c->subs[i].factor_set) return fail(FETI_ERR_LIFECYCLE, "subdomain slot %zu has no factor values", i);
  if ((c->device_factor || c->sparse_factor) && !c->tiles_fresh)
    return fail(FETI_ERR_LIFECYCLE, "assemble needs a new feti_factorize (the tiles were already scaled)");
  c->tiles_fresh = false;
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  int launches = 0, rc;
  if ((rc = wait_applies(c))) return rc;
  bool pending = false;
  double fb = 0;
  for (auto& s : c->subs)
    if (s.factor_from_host && s.h_values) {
      pending = true;
      fb += 8.0 * s.upload_count();
    }
  feti_stats& S = c->stats;
  CUDA_TRY(cudaEventRecord(c->ev[0], st));
  if (c->subdev_dirty && (rc = sync_subdev(c))) return rc;
  if (c->sparse_factor) {
    // sparse route: each group's assembly + correction on the group's stream,
    // right behind its factorization (the persistent scheduler ran on the
    // context stream: the groups wait for it)
    const int G = c->sp_groups;
    const bool in_graph = c->sp_assembled_in_graph;
    c->sp_assembled_in_graph = false;
    if (in_graph) {
      // the factorization graph already ran every group's assembly behind its
      // column sequence
      launches = 0;
    } else {
      CUDA_TRY(cudaEventRecord(c->ev[2], st));
      for (int g = 0; g < G; ++g) {
        cudaStream_t gs = c->sp_streams[g];
        // the captured graph ran on the context stream
        if (c->sp_graph_used) CUDA_TRY(cudaStreamWaitEvent(gs, c->ev[2], 0));
        if ((rc = sparse_group_assembly(c, g, gs, &launches))) return rc;
        CUDA_TRY(cudaEventRecord(c->sp_join[g], gs));
        CUDA_TRY(cudaStreamWaitEvent(st, c->sp_join[g], 0));
      }
    }
    CUDA_TRY(cudaEventRecord(c->sp_ev[2], st));
    std::vector<int> bad(c->subs.size(), 1 << 30);
    if (!c->subs.empty())
      CUDA_TRY(cudaMemcpyAsync(bad.data(), c->d_bad, bad.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    float mf = 0, mp = 0;
    CUDA_TRY(cudaEventElapsedTime(&mp, c->sp_ev[0], c->sp_ev[2]));
    if (in_graph) {
      // the last group's factorization end
      for (int g = 0; g < G; ++g) {
        float t = 0;
        CUDA_TRY(cudaEventElapsedTime(&t, c->sp_ev[0], c->sp_fend[g]));
        mf = std::max(mf, t);
      }
    } else {
      CUDA_TRY(cudaEventElapsedTime(&mf, c->sp_ev[0], c->sp_ev[1]));
    }
    S.ms_factorize = mf;
    S.ms_preprocess = mp;
    S.ms_wait_upload = 0.0;
    S.ms_unpack = S.ms_diag_inverse = S.ms_block_scale = S.ms_trsm = S.ms_syrk = S.ms_correct = 0.0;
    S.ms_assemble = mp - mf;   // past the last group's factorization
    S.factor_bytes = 0.0;
    S.launches_assemble = launches;
    c->sp_pending_check = false;
    for (size_t si = 0; si < bad.size(); ++si)
      if (bad[si] < (1 << 30))
        return fail(FETI_ERR_NOT_SPD, "slot %d: non-positive pivot at permuted row %d: matrix is not SPD", (int)si,
                    bad[si]);
    c->assembled = true;
    return FETI_OK;
  }
  if (!pending) {
    // factors resident on the device: one batched launch per kernel over all
    // subdomains (largest chains first)
    std::vector<int> sparse;
    for (int si = 0; si < (int)c->subs.size(); ++si)
      if (!c->subs[si].dense) sparse.push_back(si);
    if ((rc = launch_assembly(c, st, c->d_w_unpack, c->n_unpack, c->d_w_diag, c->n_diag, c->d_w_scale, c->n_scale,
                              c->d_w_chain, c->n_chain, c->d_w_syrk, c->n_syrk, sparse, &c->ev[1], &launches)))
      return rc;
    CUDA_TRY(cudaEventRecord(c->ev[7], st));
    CUDA_TRY(cudaStreamSynchronize(st));
    float ms[5];
    for (int i = 0; i < 5; ++i) CUDA_TRY(cudaEventElapsedTime(&ms[i], c->ev[i + 1], c->ev[i + 2]));
    float msc = 0;
    CUDA_TRY(cudaEventElapsedTime(&msc, c->ev[6], c->ev[7]));
    S.ms_correct = msc;
    S.ms_wait_upload = 0.0;
    S.ms_unpack = ms[0];
    S.ms_diag_inverse = ms[1];
    S.ms_block_scale = ms[2];
    S.ms_trsm = ms[3];
    S.ms_syrk = ms[4];
    S.ms_assemble = ms[0] + ms[1] + ms[2] + ms[3] + ms[4] + msc;
    S.factor_bytes = 0.0;
  } else {
    // host factors: H2D in wave order on the copy stream; each wave's kernels
    // run on alternating streams as soon as its copies have landed, so the
    // PCIe transfer of wave w+1 overlaps the DMMA work of wave w
    CUDA_TRY(cudaEventRecord(c->ev[1], st));
    CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->ev[1], 0));
    for (size_t w = 0; w < c->waves.size(); ++w) {
      for (int si : c->waves[w]) {
        SubHost& s = c->subs[si];
        if (s.factor_from_host && s.h_values && s.upload_count() > 0)
          CUDA_TRY(cudaMemcpyAsync(s.d_raw_own, s.h_values + s.raw_off, (size_t)s.upload_count() * 8,
                                   cudaMemcpyHostToDevice, c->copy_stream));
      }
      CUDA_TRY(cudaEventRecord(c->wave_ev[w], c->copy_stream));
    }
    for (size_t w = 0; w < c->waves.size(); ++w) {
      cudaStream_t ws = c->wave_streams[w % feti_ctx::kWaveStreams];
      CUDA_TRY(cudaStreamWaitEvent(ws, c->wave_ev[w], 0));
      std::vector<int> sparse;
      for (int si : c->waves[w])
        if (!c->subs[si].dense) sparse.push_back(si);
      const auto& r = c->wv_range;
      if ((rc = launch_assembly(c, ws, c->d_wv[0] + r[0][w].first, r[0][w].second, c->d_wv[1] + r[1][w].first,
                                r[1][w].second, c->d_wv[2] + r[2][w].first, r[2][w].second,
                                c->d_wv[3] + r[3][w].first, r[3][w].second, c->d_wv[4] + r[4][w].first,
                                r[4][w].second, sparse, nullptr, &launches)))
        return rc;
    }
    for (int i = 0; i < feti_ctx::kWaveStreams; ++i) {
      CUDA_TRY(cudaEventRecord(c->wave_join[i], c->wave_streams[i]));
      CUDA_TRY(cudaStreamWaitEvent(st, c->wave_join[i], 0));
    }
    CUDA_TRY(cudaEventRecord(c->ev[2], st));
    CUDA_TRY(cudaStreamSynchronize(st));
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, c->ev[1], c->ev[2]));
    S.ms_wait_upload = ms;  // H2D + overlapped assembly, first copy to last kernel
    S.ms_unpack = S.ms_diag_inverse = S.ms_block_scale = S.ms_trsm = S.ms_syrk = 0.0;
    S.ms_assemble = ms;
    S.factor_bytes = fb;
    for (auto& s : c->subs) s.h_values = nullptr;
  }
  S.launches_assemble = launches;
  c->assembled = true;
  return FETI_OK;
}

int feti_local_operator(feti_ctx* c, int64_t slot, double* out) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->assembled) return fail(FETI_ERR_LIFECYCLE, "local operator before preprocess");
  if (c->implicit) return fail(FETI_ERR_LIFECYCLE, "the implicit strategy keeps no local operator");
  if (slot < 0 || slot >= (int64_t)c->subs.size()) return fail(FETI_ERR_ARG, "slot out of range");
  const SubHost& s = c->subs[slot];
  CUDA_TRY(cudaSetDevice(c->device));
  std::vector<double> tiles((size_t)s.f_tiles() * ATILE);
  if (!tiles.empty())
    CUDA_TRY(cudaMemcpy(tiles.data(), s.d_F, tiles.size() * 8, cudaMemcpyDeviceToHost));
  const int64_t m = s.m;
  std::vector<int64_t> pos(m);
  for (int64_t a = 0; a < m; ++a) pos[s.colperm[a]] = a;
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < m; ++j) {
      double v = 0.0;
      if (j >= i) {
        int64_t u = pos[i], w = pos[j];
        if (u > w) std::swap(u, w);
        v = tiles[(size_t)apply_tile_index(u / AT, w / AT, s.T32) * ATILE + (u % AT) * AT + (w % AT)];
      }
      out[i * m + j] = v;
    }
  return FETI_OK;
}

static int implicit_enqueue(feti_ctx* c, const double* d_p, double* d_q, cudaStream_t st, bool time_it);

// The descriptor table was uploaded by feti_assemble on the context stream;
// apply reads only finalize-time fields of it (F~ tiles, index maps).
static int apply_enqueue(feti_ctx* c, const double* d_p, double* d_q, cudaStream_t st, bool time_it) {
  if (time_it) CUDA_TRY(cudaEventRecord(c->ev[0], st));
  launch_apply(c->apply_nw, c->apply_sb, c->d_subdev, c->d_apply_segs, c->d_apply_seg_ptr, c->n_apply, c->d_part, d_p, st);
  launch_reduce((int)c->n_mult, c->d_cptr, c->d_cent, c->d_ridx, c->d_part, d_q, st);
  CUDA_TRY(cudaGetLastError());
  if (time_it) CUDA_TRY(cudaEventRecord(c->ev[1], st));
  return mark_apply(c, st);
}

int feti_apply(feti_ctx* c, const double* p, double* q) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->assembled) return fail(FETI_ERR_LIFECYCLE, "apply before preprocess for the current values");
  if (!p || !q) return fail(FETI_ERR_ARG, "NULL vector");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  CUDA_TRY(cudaMemcpyAsync(c->d_p, p, (size_t)c->n_mult * 8, cudaMemcpyHostToDevice, st));
  int rc = c->implicit ? implicit_enqueue(c, c->d_p, c->d_q, st, true) : apply_enqueue(c, c->d_p, c->d_q, st, true);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(q, c->d_q, (size_t)c->n_mult * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  float ms = 0;
  CUDA_TRY(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
  c->stats.ms_apply = ms;
  return FETI_OK;
}

int feti_set_preconditioner(feti_ctx* c, int64_t slot, const double* P) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->finalized) return fail(FETI_ERR_LIFECYCLE, "set_preconditioner before prepare");
  if (slot < 0 || slot >= (int64_t)c->subs.size()) return fail(FETI_ERR_ARG, "slot out of range");
  if (!P) return fail(FETI_ERR_ARG, "P is NULL");
  CUDA_TRY(cudaSetDevice(c->device));
  SubHost& s = c->subs[slot];
  int rc;
  if (!s.d_Fp) {
    if ((rc = dev_alloc(c, (void**)&s.d_Fp, (size_t)std::max<int64_t>(s.f_tiles(), 1) * ATILE * 8, true))) return rc;
    ++c->n_precond_set;
  }
  // pack into the apply layout: upper triangle of 32x32 tiles in sorted
  // column order, diagonal tiles full, padding zero
  std::vector<double> t((size_t)s.f_tiles() * ATILE, 0.0);
  const int64_t m = s.m;
  for (int ti = 0; ti < s.T32; ++ti)
    for (int tj = ti; tj < s.T32; ++tj) {
      double* dst = t.data() + (size_t)apply_tile_index(ti, tj, s.T32) * ATILE;
      for (int u = 0; u < AT; ++u) {
        const int64_t a = (int64_t)ti * AT + u;
        if (a >= m) break;
        const double* row = P + s.colperm[a] * m;
        for (int v = 0; v < AT; ++v) {
          const int64_t b = (int64_t)tj * AT + v;
          if (b >= m) break;
          dst[u * AT + v] = row[s.colperm[b]];
        }
      }
    }
  CUDA_TRY(cudaMemcpy(s.d_Fp, t.data(), t.size() * 8, cudaMemcpyHostToDevice));
  if (c->n_precond_set == (int)c->subs.size()) {
    // descriptor table for the preconditioner apply (F -> preconditioner tiles)
    std::vector<SubDev> h;
    fill_subdev(c, h);
    for (size_t i = 0; i < h.size(); ++i) h[i].F = c->subs[i].d_Fp;
    if (!c->d_subdev_p && (rc = dev_alloc(c, (void**)&c->d_subdev_p, h.size() * sizeof(SubDev), true))) return rc;
    CUDA_TRY(cudaMemcpy(c->d_subdev_p, h.data(), h.size() * sizeof(SubDev), cudaMemcpyHostToDevice));
  }
  return FETI_OK;
}

int feti_precond_apply_device(feti_ctx* c, const double* d_w, double* d_out, void* stream) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->d_subdev_p || c->n_precond_set != (int)c->subs.size())
    return fail(FETI_ERR_LIFECYCLE, "preconditioner apply before feti_set_preconditioner for every slot");
  if (!d_w || !d_out) return fail(FETI_ERR_ARG, "NULL vector");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  launch_apply(c->apply_nw, c->apply_sb, c->d_subdev_p, c->d_apply_segs, c->d_apply_seg_ptr, c->n_apply, c->d_part, d_w, st);
  launch_reduce((int)c->n_mult, c->d_cptr, c->d_cent, c->d_ridx, c->d_part, d_out, st);
  CUDA_TRY(cudaGetLastError());
  return mark_apply(c, st);
}

int feti_precond_apply(feti_ctx* c, const double* w, double* out) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!w || !out) return fail(FETI_ERR_ARG, "NULL vector");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  CUDA_TRY(cudaMemcpyAsync(c->d_p, w, (size_t)c->n_mult * 8, cudaMemcpyHostToDevice, st));
  int rc = feti_precond_apply_device(c, c->d_p, c->d_q, st);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(out, c->d_q, (size_t)c->n_mult * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return FETI_OK;
}

int feti_exchange_setup(feti_ctx* c, int rank, int world, char* handle_out) {
  if (!c || !handle_out) return fail(FETI_ERR_ARG, "NULL argument");
  if (!c->finalized) return fail(FETI_ERR_LIFECYCLE, "exchange setup before prepare");
  if (world < 1 || rank < 0 || rank >= world) return fail(FETI_ERR_ARG, "bad rank %d of %d", rank, world);
  if (c->x_slab) return fail(FETI_ERR_LIFECYCLE, "exchange already set up");
  CUDA_TRY(cudaSetDevice(c->device));
  c->x_rank = rank;
  c->x_world = world;
  const size_t bytes = ((size_t)2 * world * std::max<int64_t>(c->n_mult, 1) + world) * 8;
  int rc;
  if ((rc = dev_alloc(c, (void**)&c->x_slab, bytes, true))) return rc;
  CUDA_TRY(cudaMemset(c->x_slab, 0, bytes));   // zero slabs, flags = epoch 0
  std::vector<int> touched;
  for (int64_t g = 0; g < c->n_mult; ++g)
    if (c->h_cptr[g + 1] > c->h_cptr[g]) touched.push_back((int)g);
  c->x_n_touched = (int)touched.size();
  if ((rc = upload(c, &c->d_x_touched, touched))) return rc;
  if ((rc = dev_alloc(c, (void**)&c->d_x_done, 64, true))) return rc;
  CUDA_TRY(cudaMemset(c->d_x_done, 0, 64));
  c->d_x_error = reinterpret_cast<int*>(reinterpret_cast<char*>(c->d_x_done) + 32);
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, c->x_slab));
  static_assert(sizeof(cudaIpcMemHandle_t) == FETI_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof(h));
  CUDA_TRY(cudaDeviceSynchronize());
  return FETI_OK;
}

int feti_exchange_connect(feti_ctx* c, const char* handles) {
  if (!c || !handles) return fail(FETI_ERR_ARG, "NULL argument");
  if (!c->x_slab) return fail(FETI_ERR_LIFECYCLE, "exchange connect before setup");
  CUDA_TRY(cudaSetDevice(c->device));
  std::vector<double*> peers(c->x_world, nullptr);
  for (int p = 0; p < c->x_world; ++p) {
    if (p == c->x_rank) {
      peers[p] = c->x_slab;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + (size_t)p * FETI_IPC_HANDLE_BYTES, sizeof(h));
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(FETI_ERR_CUDA, "rank %d: opening the slab of rank %d failed: %s", c->x_rank, p,
                  cudaGetErrorString(e));
    }
    peers[p] = static_cast<double*>(ptr);
    c->x_open.push_back(peers[p]);
  }
  int rc;
  if ((rc = upload(c, &c->d_x_peers, peers))) return rc;
  c->x_ready = true;
  return FETI_OK;
}

int feti_apply_exchange_device(feti_ctx* c, const double* d_p, double* d_q, void* stream) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->assembled) return fail(FETI_ERR_LIFECYCLE, "apply before preprocess for the current values");
  if (!c->x_ready) return fail(FETI_ERR_LIFECYCLE, "exchange not connected");
  if (c->implicit) return fail(FETI_ERR_ARG, "the fused exchange serves the explicit strategy");
  if (!d_p || !d_q) return fail(FETI_ERR_ARG, "NULL vector");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  // slab parity (epoch % 2) reuse is safe only if this rank's previous sum
  // finished first (feti_exchange.cu header): order it explicitly, whatever
  // stream the caller used last time
  CUDA_TRY(cudaStreamWaitEvent(st, c->x_sum_done, 0));
  launch_apply(c->apply_nw, c->apply_sb, c->d_subdev, c->d_apply_segs, c->d_apply_seg_ptr, c->n_apply, c->d_part, d_p, st);
  XchgArgs a{c->d_x_peers, c->d_x_touched, c->d_cptr, c->d_cent, c->d_ridx, c->d_part, c->d_x_done,
             c->d_x_error, c->x_epoch + 1, c->x_n_touched, (int)c->n_mult, c->x_rank, c->x_world};
  launch_exchange(a, d_q, st);
  CUDA_TRY(cudaGetLastError());
  ++c->x_epoch;   // only once the launches were accepted: ranks stay in step
  CUDA_TRY(cudaEventRecord(c->x_sum_done, st));
  return mark_apply(c, st);
}

int feti_exchange_status(feti_ctx* c) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->d_x_error) return FETI_OK;
  int err = 0;
  CUDA_TRY(cudaMemcpy(&err, c->d_x_error, sizeof(int), cudaMemcpyDeviceToHost));
  if (err) return fail(FETI_ERR_CUDA, "rank %d: a peer never published its contribution (exchange timed out)",
                       c->x_rank);
  return FETI_OK;
}

int feti_apply_device(feti_ctx* c, const double* d_p, double* d_q, void* stream) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->assembled) return fail(FETI_ERR_LIFECYCLE, "apply before preprocess for the current values");
  if (!d_p || !d_q) return fail(FETI_ERR_ARG, "NULL vector");
  CUDA_TRY(cudaSetDevice(c->device));
  // the handle is used verbatim: NULL is the legacy default stream, as in CUDA
  if (c->implicit) return implicit_enqueue(c, d_p, d_q, (cudaStream_t)stream, false);
  return apply_enqueue(c, d_p, d_q, (cudaStream_t)stream, false);
}

int feti_enable_device_factorization(feti_ctx* c) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (c->finalized) return fail(FETI_ERR_LIFECYCLE, "device factorization must be chosen before finalize");
  c->device_factor = true;
  return FETI_OK;
}

int feti_enable_sparse_factorization(feti_ctx* c) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (c->finalized) return fail(FETI_ERR_LIFECYCLE, "sparse factorization must be chosen before finalize");
  if (c->device_factor) return fail(FETI_ERR_ARG, "dense device factorization is already enabled");
  c->sparse_factor = true;
  return FETI_OK;
}

int feti_set_sparse_pattern(feti_ctx* c, int64_t slot, int64_t n, const int64_t* indptr, const int64_t* indices,
                            const int64_t* perm, int64_t r, const int64_t* fix) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (c->finalized) return fail(FETI_ERR_LIFECYCLE, "the sparse pattern must be set before finalize");
  if (!c->sparse_factor) return fail(FETI_ERR_LIFECYCLE, "sparse factorization is not enabled");
  if (slot < 0 || slot >= (int64_t)c->subs.size()) return fail(FETI_ERR_ARG, "slot out of range");
  SubHost& s = c->subs[slot];
  // n DOFs; the slot was registered with s.n >= n positions (tile-aligned
  // orderings pad segments to 128 rows; perm holds -1 at padding positions)
  if (n <= 0 || n > s.n)
    return fail(FETI_ERR_ARG, "pattern size %lld does not fit the subdomain's %lld positions", (long long)n,
                (long long)s.n);
  if (!indptr || !indices || !perm || r < 0 || r > 8 || (r > 0 && !fix))
    return fail(FETI_ERR_ARG, "bad sparse pattern arguments (kernel dimension must be <= 8)");
  if (indptr[0] != 0) return fail(FETI_ERR_ARG, "pattern pointer must start at 0");
  std::vector<int64_t> pv(perm, perm + s.n), ip(n, -1);
  for (int64_t i = 0; i < s.n; ++i) {
    if (pv[i] == -1) continue;
    if (pv[i] < 0 || pv[i] >= n || ip[pv[i]] >= 0) return fail(FETI_ERR_ARG, "ordering is not a permutation");
    ip[pv[i]] = i;
  }
  for (int64_t a = 0; a < n; ++a)
    if (ip[a] < 0) return fail(FETI_ERR_ARG, "ordering misses DOF %lld", (long long)a);
  const int64_t nnz = indptr[n];
  for (int64_t a = 0; a < n; ++a) {
    if (indptr[a + 1] < indptr[a]) return fail(FETI_ERR_ARG, "pattern pointer is not monotone");
    bool diag = false;
    for (int64_t p = indptr[a]; p < indptr[a + 1]; ++p) {
      if (indices[p] < 0 || indices[p] >= n) return fail(FETI_ERR_ARG, "pattern column out of range");
      diag |= indices[p] == a;
    }
    if (!diag) return fail(FETI_ERR_ARG, "stiffness row %lld has no diagonal entry", (long long)a);
  }
  for (int64_t q = 0; q < r; ++q)
    if (fix[q] < 0 || fix[q] >= n) return fail(FETI_ERR_ARG, "fixing DOF out of range");
  s.sp_perm = std::move(pv);
  s.sp_iperm = std::move(ip);
  s.sp_kptr.assign(indptr, indptr + n + 1);
  s.sp_kind.assign(indices, indices + nnz);
  s.sp_fix.assign(fix, fix + r);
  s.sp_r = (int)r;
  s.sp_n = n;
  s.sp_pattern = true;
  return FETI_OK;
}

int feti_set_stiffness(feti_ctx* c, int64_t slot, int64_t n, const int64_t* indptr, const int64_t* indices,
                       const double* data, int64_t nnz, const double* Q, int64_t r, double rho, const int64_t* perm) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->finalized || !(c->device_factor || c->sparse_factor))
    return fail(FETI_ERR_LIFECYCLE, "set_stiffness needs a finalized context with device factorization");
  if (slot < 0 || slot >= (int64_t)c->subs.size()) return fail(FETI_ERR_ARG, "slot out of range");
  SubHost& s = c->subs[slot];
  const int64_t ndof = c->sparse_factor ? s.sp_n : s.n;
  if (n != ndof) return fail(FETI_ERR_ARG, "stiffness size %lld does not match the subdomain (%lld)", (long long)n,
                             (long long)ndof);
  if (!indptr || !indices || !data || (r > 0 && !Q) || !perm || r < 0 || r > 64 || nnz != indptr[n])
    return fail(FETI_ERR_ARG, "bad stiffness arguments");
  if (c->sparse_factor) {
    if ((int)r != s.sp_r) return fail(FETI_ERR_ARG, "kernel dimension differs from the sparse pattern's");
    if (nnz != s.sp_kptr[n] || !std::equal(perm, perm + s.n, s.sp_perm.begin()) ||
        !std::equal(indptr, indptr + n + 1, s.sp_kptr.begin()))
      return fail(FETI_ERR_ARG, "stiffness pattern or ordering differs from the sparse pattern");
  }
  CUDA_TRY(cudaSetDevice(c->device));
  int rc;
  if (!s.stiff_set) {
    std::vector<int64_t> pv, ip;
    if (c->sparse_factor) {   // the pattern call validated the (padded) ordering
      pv = s.sp_perm;
      ip = s.sp_iperm;
    } else {
      pv.assign(perm, perm + n);
      ip.assign(n, -1);
      for (int64_t i = 0; i < n; ++i) {
        if (pv[i] < 0 || pv[i] >= n || ip[pv[i]] >= 0) return fail(FETI_ERR_ARG, "ordering is not a permutation");
        ip[pv[i]] = i;
      }
    }
    std::vector<int64_t> kp(indptr, indptr + n + 1), ki(indices, indices + nnz);
    if ((rc = upload(c, &s.d_perm, pv))) return rc;
    if ((rc = upload(c, &s.d_iperm, ip))) return rc;
    if ((rc = upload(c, &s.d_kptr, kp))) return rc;
    if ((rc = upload(c, &s.d_kind, ki))) return rc;
    if ((rc = dev_alloc(c, (void**)&s.d_kdata, (size_t)std::max<int64_t>(nnz, 1) * 8, true))) return rc;
    if ((rc = dev_alloc(c, (void**)&s.d_Q, (size_t)std::max<int64_t>(n * r, 1) * 8, true))) return rc;
    s.k_nnz = nnz;
    s.kr = (int)r;
    s.stiff_set = true;
  } else if (nnz != s.k_nnz || (int)r != s.kr) {
    return fail(FETI_ERR_ARG, "stiffness pattern changed after the first call");
  }
  if (c->sparse_factor) {
    if (!s.d_kdiag) {
      std::vector<int64_t> kd(n, -1);
      for (int64_t i = 0; i < n; ++i)
        for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p)
          if (indices[p] == i) kd[i] = p;
      if ((rc = upload(c, &s.d_kdiag, kd))) return rc;
      if ((rc = dev_alloc(c, (void**)&s.d_rho, sizeof(double), true))) return rc;
    }
    return stiffness_values_async(c, s, data, Q);
  }
  CUDA_TRY(cudaMemcpy(s.d_kdata, data, (size_t)nnz * 8, cudaMemcpyHostToDevice));
  if (r > 0) CUDA_TRY(cudaMemcpy(s.d_Q, Q, (size_t)(n * r) * 8, cudaMemcpyHostToDevice));
  s.rho = rho;
  return FETI_OK;
}

int feti_set_stiffness_values(feti_ctx* c, int64_t nslots, const int64_t* slots, const double* const* data,
                              const int64_t* nnz, const double* const* Q) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->finalized || !c->sparse_factor)
    return fail(FETI_ERR_LIFECYCLE, "set_stiffness_values needs a finalized context with sparse factorization");
  if (nslots < 0 || (nslots > 0 && (!slots || !data || !nnz))) return fail(FETI_ERR_ARG, "bad batch arguments");
  CUDA_TRY(cudaSetDevice(c->device));
  for (int64_t i = 0; i < nslots; ++i) {
    if (slots[i] < 0 || slots[i] >= (int64_t)c->subs.size()) return fail(FETI_ERR_ARG, "slot out of range");
    SubHost& s = c->subs[slots[i]];
    if (!s.stiff_set)
      return fail(FETI_ERR_LIFECYCLE, "slot %lld: the first hand-over goes through feti_set_stiffness",
                  (long long)slots[i]);
    if (nnz[i] != s.k_nnz || !data[i])
      return fail(FETI_ERR_ARG, "slot %lld: %lld values for a pattern of %lld", (long long)slots[i],
                  (long long)nnz[i], (long long)s.k_nnz);
    int rc = stiffness_values_async(c, s, data[i], Q ? Q[i] : nullptr);
    if (rc) return rc;
  }
  return FETI_OK;
}

int feti_enable_dual_rhs(feti_ctx* c) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (c->finalized) return fail(FETI_ERR_LIFECYCLE, "the dual right-hand side must be enabled before finalize");
  if (!c->sparse_factor) return fail(FETI_ERR_ARG, "the device dual right-hand side needs the sparse-factor route");
  c->dual_rhs = true;
  return FETI_OK;
}

int feti_set_forces(feti_ctx* c, int64_t nslots, const int64_t* slots, const double* const* fproj,
                    const double* const* qtf) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->finalized || !c->dual_rhs) return fail(FETI_ERR_LIFECYCLE, "set_forces needs feti_enable_dual_rhs");
  if (nslots < 0 || (nslots > 0 && (!slots || !fproj))) return fail(FETI_ERR_ARG, "bad force arguments");
  CUDA_TRY(cudaSetDevice(c->device));
  if (!c->k_pending) {
    CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->k_free, 0));   // the last init read the old values
    c->k_pending = true;
  }
  for (int64_t i = 0; i < nslots; ++i) {
    if (slots[i] < 0 || slots[i] >= (int64_t)c->subs.size() || !fproj[i]) return fail(FETI_ERR_ARG, "bad slot");
    SubHost& s = c->subs[slots[i]];
    CUDA_TRY(cudaMemcpyAsync(s.d_fproj, fproj[i], (size_t)s.sp_n * 8, cudaMemcpyHostToDevice, c->copy_stream));
    c->k_early = true;
    if (s.sp_r > 0) {
      if (!qtf || !qtf[i]) return fail(FETI_ERR_ARG, "slot %lld needs Q^T f", (long long)slots[i]);
      s.h_qtf.assign(qtf[i], qtf[i] + s.sp_r);
      CUDA_TRY(cudaMemcpyAsync(s.d_qtf, s.h_qtf.data(), (size_t)s.sp_r * 8, cudaMemcpyHostToDevice, c->copy_stream));
    }
    mark_group_ready(c, (int)slots[i]);
  }
  CUDA_TRY(cudaEventRecord(c->k_ready, c->copy_stream));
  return FETI_OK;
}

int feti_dual_rhs(feti_ctx* c, const double* cvec, double* d) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->dual_rhs) return fail(FETI_ERR_LIFECYCLE, "feti_dual_rhs needs feti_enable_dual_rhs");
  if (!c->assembled) return fail(FETI_ERR_LIFECYCLE, "dual right-hand side before preprocess");
  if (!d) return fail(FETI_ERR_ARG, "d is NULL");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  int rc;
  if ((rc = wait_applies(c))) return rc;
  if (cvec) CUDA_TRY(cudaMemcpyAsync(c->d_p, cvec, (size_t)c->n_mult * 8, cudaMemcpyHostToDevice, st));
  launch_sp_dual_rhs(c->d_spsub, (int)c->n_mult, c->d_cptr, c->d_cent, cvec ? c->d_p : nullptr, c->d_q, st);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(d, c->d_q, (size_t)c->n_mult * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return FETI_OK;
}

int feti_factorize(feti_ctx* c) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->finalized || !(c->device_factor || c->sparse_factor))
    return fail(FETI_ERR_LIFECYCLE, "factorize needs a finalized context with device factorization");
  for (size_t i = 0; i < c->subs.size(); ++i)
    if (!c->subs[i].stiff_set) return fail(FETI_ERR_LIFECYCLE, "subdomain slot %zu has no stiffness", i);
  CUDA_TRY(cudaSetDevice(c->device));
  if (int rc0 = wait_applies(c)) return rc0;
  c->assembled = false;   // apply / solve need the assembly of the new factor
  if (c->sparse_factor) return factorize_sparse(c);
  cudaStream_t st = c->stream;
  const int ns = (int)c->subs.size();
  std::vector<FactorSub> fs(ns);
  for (int si = 0; si < ns; ++si) {
    SubHost& s = c->subs[si];
    fs[si] = FactorSub{s.d_Q, s.d_perm, s.d_iperm, s.d_kptr, s.d_kind, s.d_kdata, s.rho, s.kr, 0};
    s.src = SRC_TILES;
    c->subdev_dirty = true;
  }
  CUDA_TRY(cudaMemcpyAsync(c->d_fsub, fs.data(), ns * sizeof(FactorSub), cudaMemcpyHostToDevice, st));
  int rc;
  if ((rc = sync_subdev(c))) return rc;
  std::vector<int> big(ns, 1 << 30);
  CUDA_TRY(cudaMemcpyAsync(c->d_bad, big.data(), ns * sizeof(int), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaEventRecord(c->ev[0], st));
  const int T = c->uniform_T;
  int max_n = 0;
  for (auto& s : c->subs) max_n = std::max(max_n, (int)s.n);
  launch_kreg_build(c->d_subdev, c->d_fsub, ns, T, max_n, st);
  CUDA_TRY(cudaGetLastError());
  FETI_DEBUG_SYNC(st);
  for (int k = 0; k < T;) {
    k = launch_factor_step(c->d_subdev, c->d_dinv, c->d_bad, ns, k, T, st);
    CUDA_TRY(cudaGetLastError());
    FETI_DEBUG_SYNC(st);
  }
  CUDA_TRY(cudaEventRecord(c->ev[1], st));
  CUDA_TRY(cudaMemcpyAsync(big.data(), c->d_bad, ns * sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  float ms = 0;
  CUDA_TRY(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
  c->stats.ms_factorize = ms;
  for (int si = 0; si < ns; ++si)
    if (big[si] < (1 << 30))
      return fail(FETI_ERR_NOT_SPD, "slot %d: non-positive pivot at permuted row %d: matrix is not SPD", si,
                  big[si]);
  for (auto& s : c->subs) s.factor_set = true;
  c->tiles_fresh = true;
  return FETI_OK;
}

// replace a per-call device buffer by a larger one (frees the old one)
static int grow(feti_ctx* c, void** p, size_t* cap, size_t bytes) {
  if (bytes <= *cap) return FETI_OK;
  if (*p) {
    c->allocs.erase(std::find(c->allocs.begin(), c->allocs.end(), *p));
    c->bytes_temporary -= (int64_t)*cap;
    CUDA_TRY(cudaFree(*p));
    *p = nullptr;
    *cap = 0;
  }
  int rc = dev_alloc(c, p, bytes, false);
  if (rc) return rc;
  *cap = bytes;
  return FETI_OK;
}

// sparse route: one CTA per right-hand side through the block-sparse factor
static int solve_many_sparse(feti_ctx* c, int64_t nslots, const int64_t* slots, const double* b, double* x) {
  cudaStream_t st = c->stream;
  std::vector<SpSolveItem> items((size_t)nslots);
  int64_t nb = 0, nscr = 0;
  for (int64_t q = 0; q < nslots; ++q) {
    if (slots[q] < 0 || slots[q] >= (int64_t)c->subs.size()) return fail(FETI_ERR_ARG, "slot out of range");
    const SubHost& s = c->subs[slots[q]];
    items[q] = SpSolveItem{(int)slots[q], 0, nb, nscr};
    nb += s.sp_n;
    nscr += 3 * (int64_t)s.sp.T * TB;
  }
  int rc;
  const size_t bytes = (size_t)(2 * nb + nscr) * 8;
  if ((rc = grow(c, (void**)&c->d_sps, &c->sps_cap, bytes))) return rc;
  if ((rc = grow(c, (void**)&c->d_sps_items, &c->sps_items_cap, items.size() * sizeof(SpSolveItem)))) return rc;
  double* db = c->d_sps;
  double* dx = db + nb;
  CUDA_TRY(cudaMemcpyAsync(c->d_sps_items, items.data(), items.size() * sizeof(SpSolveItem), cudaMemcpyHostToDevice,
                           st));
  CUDA_TRY(cudaMemcpyAsync(db, b, (size_t)nb * 8, cudaMemcpyHostToDevice, st));
  launch_sp_solve(c->d_subdev, c->d_spsub, c->d_sps_items, (int)nslots, db, dx, dx + nb, st);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(x, dx, (size_t)nb * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return FETI_OK;
}

int feti_solve_many(feti_ctx* c, int64_t nslots, const int64_t* slots, const double* b, double* x) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (c->sparse_factor && c->assembled) {
    if (nslots <= 0 || !slots || !b || !x) return fail(FETI_ERR_ARG, "bad solve arguments");
    CUDA_TRY(cudaSetDevice(c->device));
    return solve_many_sparse(c, nslots, slots, b, x);
  }
  if (!c->device_factor || !c->assembled)
    return fail(FETI_ERR_LIFECYCLE, "solve needs an assembled context with dense device factorization");
  if (nslots <= 0 || nslots > (int64_t)c->subs.size() || !slots || !b || !x) return fail(FETI_ERR_ARG, "bad solve arguments");
  if (solve_smem(c->uniform_T) > 227 * 1024) return fail(FETI_ERR_CAPACITY, "subdomain too large for the solve sweep");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  std::vector<int64_t> off(nslots + 1, 0);
  std::vector<int> sl(nslots);
  for (int64_t q = 0; q < nslots; ++q) {
    if (slots[q] < 0 || slots[q] >= (int64_t)c->subs.size()) return fail(FETI_ERR_ARG, "slot out of range");
    sl[q] = (int)slots[q];
    off[q + 1] = off[q] + c->subs[sl[q]].n;
  }
  // scratch: per-call offsets/slots at the front of the lib's buffers
  CUDA_TRY(cudaMemcpyAsync(c->d_slots, sl.data(), nslots * sizeof(int), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(c->d_vec_off, off.data(), (nslots + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(c->d_sb, b, (size_t)off[nslots] * 8, cudaMemcpyHostToDevice, st));
  launch_solve(c->d_subdev, c->d_fsub, c->d_slots, (int)nslots, c->uniform_T, c->d_vec_off, c->d_sb, c->d_sx, st);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(x, c->d_sx, (size_t)off[nslots] * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return FETI_OK;
}

static int implicit_enqueue(feti_ctx* c, const double* d_p, double* d_q, cudaStream_t st, bool time_it) {
  if (c->impl_max_blocks < 0)
    return fail(FETI_ERR_CAPACITY, "implicit apply: subdomain too large for the single-CTA sweep");
  if (time_it) CUDA_TRY(cudaEventRecord(c->ev[0], st));
  launch_implicit_apply(c->d_subdev, c->sparse_factor ? c->d_spsub : nullptr, (int)c->subs.size(), c->impl_max_blocks, c->d_impl_off, d_p, c->d_impl_part,
                        (int)c->n_mult, c->d_cptr, c->d_cent, d_q, st);
  CUDA_TRY(cudaGetLastError());
  if (time_it) CUDA_TRY(cudaEventRecord(c->ev[1], st));
  return mark_apply(c, st);
}

int feti_apply_implicit(feti_ctx* c, const double* p, double* q) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->assembled) return fail(FETI_ERR_LIFECYCLE, "apply before preprocess for the current values");
  if (!p || !q) return fail(FETI_ERR_ARG, "NULL vector");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  CUDA_TRY(cudaMemcpyAsync(c->d_p, p, (size_t)c->n_mult * 8, cudaMemcpyHostToDevice, st));
  int rc = implicit_enqueue(c, c->d_p, c->d_q, st, true);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpyAsync(q, c->d_q, (size_t)c->n_mult * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  float ms = 0;
  CUDA_TRY(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
  c->stats.ms_apply = ms;
  return FETI_OK;
}

int feti_apply_implicit_device(feti_ctx* c, const double* d_p, double* d_q, void* stream) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->assembled) return fail(FETI_ERR_LIFECYCLE, "apply before preprocess for the current values");
  if (!d_p || !d_q) return fail(FETI_ERR_ARG, "NULL vector");
  CUDA_TRY(cudaSetDevice(c->device));
  return implicit_enqueue(c, d_p, d_q, (cudaStream_t)stream, false);
}

int feti_coarse_setup(feti_ctx* c, const int64_t* kdim, const double* G, const double* coarse_inv, int64_t nk) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->finalized) return fail(FETI_ERR_LIFECYCLE, "coarse setup before prepare");
  if (c->d_coarse) return fail(FETI_ERR_LIFECYCLE, "coarse space already set up");
  if (!kdim || !G || !coarse_inv || nk < 0 || nk > (1 << 20)) return fail(FETI_ERR_ARG, "bad coarse arguments");
  CUDA_TRY(cudaSetDevice(c->device));
  int64_t tot = 0, gsz = 0;
  for (size_t si = 0; si < c->subs.size(); ++si) {
    if (kdim[si] < 0) return fail(FETI_ERR_ARG, "negative kernel dimension");
    tot += kdim[si];
    gsz += c->subs[si].m * kdim[si];
  }
  if (tot != nk) return fail(FETI_ERR_ARG, "kernel dimensions sum to %lld, expected %lld", (long long)tot, (long long)nk);
  // permute each block to the sorted local order of the apply's index maps
  std::vector<double> gs((size_t)std::max<int64_t>(gsz, 1));
  std::vector<CoarseSub> hs(c->subs.size());
  std::vector<int2> cols;
  int64_t goff = 0, koff = 0;
  double* d_g = nullptr;
  int rc;
  if ((rc = dev_alloc(c, (void**)&d_g, gs.size() * 8, true))) return rc;
  for (size_t si = 0; si < c->subs.size(); ++si) {
    const SubHost& s = c->subs[si];
    const int r = (int)kdim[si];
    for (int64_t a = 0; a < s.m; ++a)
      for (int k = 0; k < r; ++k) gs[goff + a * r + k] = G[goff + s.colperm[a] * r + k];
    hs[si].G = d_g + goff;
    hs[si].gids = s.d_g;
    hs[si].m = (int)s.m;
    hs[si].r = r;
    hs[si].koff = (int)koff;
    for (int k = 0; k < r; ++k) cols.push_back(make_int2((int)si, k));
    goff += s.m * r;
    koff += r;
  }
  CUDA_TRY(cudaMemcpy(d_g, gs.data(), gs.size() * 8, cudaMemcpyHostToDevice));
  if ((rc = upload(c, &c->d_coarse, hs))) return rc;
  if ((rc = upload(c, &c->d_kcols, cols))) return rc;
  std::vector<double> ci(coarse_inv, coarse_inv + nk * nk);
  if ((rc = upload(c, &c->d_cinv, ci))) return rc;
  {
    // G by kernel column, entries of a column contiguous (sorted local order),
    // cut into pieces of <= kPiece entries that never straddle columns
    std::vector<double> gv;
    std::vector<int> gi;
    std::vector<int4> pcs;
    int64_t go = 0;
    for (size_t si = 0; si < c->subs.size(); ++si) {
      const SubHost& sh = c->subs[si];
      const int r = (int)kdim[si];
      for (int k = 0; k < r; ++k) {
        const int col = hs[si].koff + k;
        const int e0 = (int)gv.size();
        for (int64_t a = 0; a < sh.m; ++a) {
          gv.push_back(gs[go + a * r + k]);
          gi.push_back(sh.gids_sorted[a]);
        }
        for (int e = e0; e < (int)gv.size(); e += kPiece)
          pcs.push_back(make_int4(col, e, std::min<int>(e + kPiece, (int)gv.size()), 0));
      }
      go += sh.m * r;
    }
    if ((rc = upload(c, &c->d_gval, gv))) return rc;
    if ((rc = upload(c, &c->d_gidx, gi))) return rc;
    if ((rc = upload(c, &c->d_pieces, pcs))) return rc;
    c->npieces = (int)pcs.size();
    if ((rc = dev_alloc(c, (void**)&c->d_ppart, (size_t)std::max(c->npieces, 1) * 8, true))) return rc;
  }
  if ((rc = dev_alloc(c, (void**)&c->d_kv, (size_t)std::max<int64_t>(nk, 1) * 8, true))) return rc;
  if ((rc = dev_alloc(c, (void**)&c->d_kz, (size_t)std::max<int64_t>(nk, 1) * 8, true))) return rc;
  c->nk = (int)nk;
  return FETI_OK;
}

int feti_project_device(feti_ctx* c, const double* d_x, double* d_out, void* stream) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->d_coarse) return fail(FETI_ERR_LIFECYCLE, "projector before coarse setup");
  if (!d_x || !d_out) return fail(FETI_ERR_ARG, "NULL vector");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  launch_gtx(c->d_coarse, c->d_kcols, c->nk, d_x, c->d_kv, st);
  launch_coarse(c->nk, c->d_cinv, c->d_kv, c->d_kz, st);
  launch_project((int)c->n_mult, c->d_cptr, c->d_cent, c->d_coarse, c->d_kz, d_x, 1.0, d_out, st);
  CUDA_TRY(cudaGetLastError());
  return FETI_OK;
}

int feti_coarse_apply_device(feti_ctx* c, const double* d_v, double* d_out, void* stream) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->d_coarse) return fail(FETI_ERR_LIFECYCLE, "coarse apply before coarse setup");
  if (!d_v || !d_out) return fail(FETI_ERR_ARG, "NULL vector");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  launch_coarse(c->nk, c->d_cinv, d_v, c->d_kz, st);
  launch_project((int)c->n_mult, c->d_cptr, c->d_cent, c->d_coarse, c->d_kz, nullptr, -1.0, d_out, st);
  CUDA_TRY(cudaGetLastError());
  return FETI_OK;
}

int feti_pcpg_solve(feti_ctx* c, const double* d, const double* e, double tol, int64_t maxit, int precond,
                    double* lam, int64_t* iterations, double* rel_residual) {
  if (!c) return fail(FETI_ERR_ARG, "ctx is NULL");
  if (!c->assembled) return fail(FETI_ERR_LIFECYCLE, "PCPG before preprocess");
  if (c->implicit) return fail(FETI_ERR_ARG, "the device PCPG runs on the explicit operator");
  if (!c->d_coarse) return fail(FETI_ERR_LIFECYCLE, "PCPG before feti_coarse_setup");
  if (precond != 0 && precond != 1) return fail(FETI_ERR_ARG, "precond must be 0 (none) or 1 (lumped)");
  if (precond == 1 && (!c->d_subdev_p || c->n_precond_set != (int)c->subs.size()))
    return fail(FETI_ERR_LIFECYCLE, "lumped PCPG before feti_set_preconditioner for every slot");
  if (!d || (c->nk > 0 && !e) || !lam || !(tol >= 0.0)) return fail(FETI_ERR_ARG, "bad PCPG arguments");
  CUDA_TRY(cudaSetDevice(c->device));
  const int n = (int)c->n_mult, nk = c->nk;
  int rc;
  if (!c->pc_vec) {
    if ((rc = dev_alloc(c, (void**)&c->pc_vec, (size_t)8 * std::max(n, 1) * 8, true))) return rc;
    if ((rc = dev_alloc(c, (void**)&c->pc_k, (size_t)4 * std::max(nk, 1) * 8, true))) return rc;
    if ((rc = dev_alloc(c, (void**)&c->pc_bpart, pcpg_bpart_doubles(n, nk) * 8, true))) return rc;
    if ((rc = dev_alloc(c, (void**)&c->pc_sc, sizeof(PcpgScal), true))) return rc;
    CUDA_TRY(cudaMemset(c->pc_sc, 0, sizeof(PcpgScal)));
    CUDA_TRY(cudaHostAlloc((void**)&c->pc_sc_host, sizeof(PcpgScal), cudaHostAllocDefault));
  }
  double* v = c->pc_vec;
  const size_t N = (size_t)std::max(n, 1);
  PcpgDev P{};
  P.n_mult = n;
  P.nk = nk;
  P.ncols = nk;
  P.cptr = c->d_cptr;
  P.cent = c->d_cent;
  P.ridx = c->d_ridx;
  P.part = c->d_part;
  P.cs = c->d_coarse;
  P.kcols = c->d_kcols;
  P.cinv = c->d_cinv;
  double* dd = v + 7 * N;
  P.d = dd;
  P.lam = v;
  P.r = v + N;
  P.p = v + 2 * N;
  P.q = v + 3 * N;
  P.y = v + 4 * N;
  P.w = v + 5 * N;
  P.z = v + 6 * N;
  const size_t K = (size_t)std::max(nk, 1);
  P.kv = c->pc_k;
  P.kz = c->pc_k + K;
  P.kv2 = c->pc_k + 2 * K;
  P.kz2 = c->pc_k + 3 * K;
  P.bpart = c->pc_bpart;
  P.sc = c->pc_sc;
  P.gval = c->d_gval;
  P.gidx = c->d_gidx;
  P.pieces = c->d_pieces;
  P.npieces = c->npieces;
  P.ppart = c->d_ppart;
  cudaStream_t st = c->stream;
  if ((rc = wait_applies(c))) return rc;
  CUDA_TRY(cudaMemcpyAsync(dd, d, (size_t)n * 8, cudaMemcpyHostToDevice, st));
  if (nk > 0) CUDA_TRY(cudaMemcpyAsync(P.kv, e, (size_t)nk * 8, cudaMemcpyHostToDevice, st));
  // lam0 = G (G^T G)^-1 e (feasible_start, solver.py:121-123)
  launch_coarse(nk, c->d_cinv, P.kv, P.kz, st);
  launch_project(n, c->d_cptr, c->d_cent, c->d_coarse, P.kz, nullptr, -1.0, P.lam, st);
  // r = d - F lam
  launch_apply(c->apply_nw, c->apply_sb, c->d_subdev, c->d_apply_segs, c->d_apply_seg_ptr, c->n_apply, c->d_part, P.lam, st);
  launch_reduce(n, c->d_cptr, c->d_cent, c->d_ridx, c->d_part, P.q, st);
  launch_pcpg_sub(n, dd, P.q, P.r, st);
  // w = P r, z = M w, y = P z
  launch_gtx(c->d_coarse, c->d_kcols, nk, P.r, P.kv, st);
  launch_coarse(nk, c->d_cinv, P.kv, P.kz, st);
  launch_project(n, c->d_cptr, c->d_cent, c->d_coarse, P.kz, P.r, 1.0, P.w, st);
  const double* zsrc = P.w;
  if (precond == 1) {
    launch_apply(c->apply_nw, c->apply_sb, c->d_subdev_p, c->d_apply_segs, c->d_apply_seg_ptr, c->n_apply, c->d_part, P.w, st);
    launch_reduce(n, c->d_cptr, c->d_cent, c->d_ridx, c->d_part, P.z, st);
    zsrc = P.z;
  }
  launch_gtx(c->d_coarse, c->d_kcols, nk, zsrc, P.kv, st);
  launch_coarse(nk, c->d_cinv, P.kv, P.kz, st);
  launch_project(n, c->d_cptr, c->d_cent, c->d_coarse, P.kz, zsrc, 1.0, P.y, st);
  launch_pcpg_init_dots(P, st);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(c->pc_sc_host, c->pc_sc, sizeof(PcpgScal), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  PcpgScal h = *c->pc_sc_host;
  const int64_t cap = maxit > 0 ? maxit : (int64_t)n;
  c->stats.pcpg_iterations = 0;
  c->stats.ms_pcpg = 0.0;
  if (h.w0 <= 1e-14 * std::max(1.0, h.dnorm)) {   // roundoff guard (solver.py:233-241)
    CUDA_TRY(cudaMemcpy(lam, P.lam, (size_t)n * 8, cudaMemcpyDeviceToHost));
    if (iterations) *iterations = 0;
    if (rel_residual) *rel_residual = 0.0;
    return FETI_OK;
  }
  h.tolw0 = tol * h.w0;
  h.maxit = cap;
  *c->pc_sc_host = h;
  CUDA_TRY(cudaMemcpyAsync(c->pc_sc, c->pc_sc_host, sizeof(PcpgScal), cudaMemcpyHostToDevice, st));
  // the iteration body, kPcpgGraphIters iterations per graph (no-ops once done)
  cudaGraphExec_t& ge = c->pc_graph[precond];
  // FETI_PCPG_COOP=0: the five-launch iteration (B, D, F, G separately)
  const int coop = (getenv("FETI_PCPG_COOP") && atoi(getenv("FETI_PCPG_COOP")) == 0)
                       ? 0 : std::min(pcpg_coop_grid(c->num_sms), 1024);
  // FETI_PCPG_FUSED=0: the apply and the vector work as two launches
  const size_t asmem = apply_smem(c->apply_nw, c->apply_sb);
  const int fused = (coop > 0 && c->apply_nw == 8 && c->apply_cps == 1 &&
                     !(getenv("FETI_PCPG_FUSED") && atoi(getenv("FETI_PCPG_FUSED")) == 0))
                        ? pcpg_fused_grid(c->n_apply, asmem) : 0;
  const ApplyArgs aargs{c->d_subdev, c->d_apply_segs, c->d_apply_seg_ptr, c->d_part, c->apply_sb, 0};
  if (!ge) {
    CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    const int* done = &c->pc_sc->done;
    const double* beta = &c->pc_sc->beta;
    for (int it = 0; it < feti_ctx::kPcpgGraphIters; ++it) {
      if (precond == 0 && fused > 0) {
        CUDA_TRY(launch_pcpg_iter_fused(P, aargs, fused, asmem, st));
        continue;
      }
      launch_apply(c->apply_nw, c->apply_sb, c->d_subdev, c->d_apply_segs, c->d_apply_seg_ptr, c->n_apply, c->d_part, P.p, st,
                   P.y, beta, done);
      if (precond == 0 && coop > 0) {
        // the vector work of the iteration in one cooperative launch
        CUDA_TRY(launch_pcpg_iter_coop(P, coop, st));
        continue;
      }
      launch_pcpg_reduce_pq(P, st);
      launch_pcpg_gtx_r(P, st);
      if (precond == 0) {
        launch_pcpg_gtx_w(P, st);
        launch_pcpg_update(P, 0, st);
      } else {
        launch_pcpg_update(P, 1, st);
        launch_apply(c->apply_nw, c->apply_sb, c->d_subdev_p, c->d_apply_segs, c->d_apply_seg_ptr, c->n_apply, c->d_part, P.w,
                     st, nullptr, nullptr, done);
        launch_reduce(n, c->d_cptr, c->d_cent, c->d_ridx, c->d_part, P.z, st);
        launch_pcpg_gtx_x(P, P.z, st);
        launch_pcpg_update(P, 2, st);
      }
    }
    cudaGraph_t graph = nullptr;
    CUDA_TRY(cudaStreamEndCapture(st, &graph));
    CUDA_TRY(cudaGraphInstantiate(&ge, graph, 0));
    CUDA_TRY(cudaGraphDestroy(graph));
  }
  CUDA_TRY(cudaEventRecord(c->ev[0], st));
  for (;;) {
    CUDA_TRY(cudaGraphLaunch(ge, st));
    CUDA_TRY(cudaMemcpyAsync(c->pc_sc_host, c->pc_sc, sizeof(PcpgScal), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (c->pc_sc_host->done) break;
  }
  CUDA_TRY(cudaEventRecord(c->ev[1], st));
  CUDA_TRY(cudaMemcpyAsync(lam, P.lam, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  float ms = 0;
  CUDA_TRY(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
  h = *c->pc_sc_host;
  c->stats.ms_pcpg = ms;
  c->stats.pcpg_iterations = h.k;
  if (iterations) *iterations = h.k;
  if (rel_residual) *rel_residual = h.w0 > 0 ? h.wn / h.w0 : 0.0;
  if (h.status == PCPG_BREAKDOWN)
    return fail(FETI_ERR_BREAKDOWN, "p^T F p = %.3e at iteration %lld", h.pq, (long long)h.k);
  if (h.status == PCPG_MAXIT)
    return fail(FETI_ERR_NOT_CONVERGED, "PCPG did not reach tol %.1e in %lld iterations (relative residual %.3e)",
                tol, (long long)h.k, h.w0 > 0 ? h.wn / h.w0 : 0.0);
  return FETI_OK;
}

int feti_get_stats(feti_ctx* c, feti_stats* out) {
  if (!c || !out) return fail(FETI_ERR_ARG, "NULL argument");
  c->stats.bytes_persistent = c->bytes_persistent;
  c->stats.bytes_temporary = c->bytes_temporary;
  *out = c->stats;
  return FETI_OK;
}

int feti_debug_kernel_attributes(char* buf, int len) {
  if (!buf || len <= 0) return fail(FETI_ERR_ARG, "bad buffer");
  buf[0] = 0;
  feti::kernel_attributes(buf, len);
  return FETI_OK;
}

int feti_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(FETI_ERR_ARG, "out is NULL");
  CUDA_TRY(cudaHostAlloc(out, bytes ? bytes : 16, cudaHostAllocPortable));
  return FETI_OK;
}

int feti_host_free(void* ptr) {
  if (ptr) CUDA_TRY(cudaFreeHost(ptr));
  return FETI_OK;
}

}  // extern "C"
