// Shared device helpers for the B200 explicit FETI dual operator.
//
// FP64 on sm_100a has no tcgen05 kind (ptxas rejects .kind::f64), so the dense
// contractions run on the FP64 tensor pipe through warp-level
// mma.sync.m8n8k4.f64 (SASS: DMMA.8x8x4).  Operand tiles are staged into
// shared memory with the Blackwell bulk-copy engine (cp.async.bulk, SASS
// UBLKCP) completing on mbarriers, consumed by warp-specialised DMMA warps.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace feti {

// ---- tiling constants ------------------------------------------------------
constexpr int TB = 128;            // block rows of L / columns per RHS panel
constexpr int TILE = TB * TB;      // doubles per 128x128 tile (128 KB)
constexpr int KS = 32;             // k-slice depth staged per pipeline stage
constexpr int SLICE = KS * TB;     // doubles per slice (32 KB)
constexpr int AT = 32;             // apply-side tile edge (32x32 = 8 KB)
constexpr int ATILE = AT * AT;
constexpr int BIG_ROW = 1 << 30;   // sentinel first-row of padding columns
// One apply work segment: tiles [t0, t1) (row-major) of the super-block
// (I, J), I <= J, of subdomain `sub`'s packed upper triangle of 32x32 tiles.
// Partial sums: rows of block I at part[out_r ...], columns of block J at
// part[out_c ...] (off-diagonal blocks only).
struct ApplySeg {
  int sub, I, J, t0, t1, pad_;
  int64_t out_r, out_c;
};

// Every 128-wide tile (L blocks, X panels, inverse diagonal blocks) is stored
// as [major][minor] with the minor index XOR-swizzled by the major index:
//     pos(major, minor) = major*128 + (minor ^ ((major & 3) << 2))
// so that the DMMA fragment reads (4 k-values x 8 rows per 16 lanes) hit 16
// distinct bank pairs, and a 32-major slice is one contiguous 32 KB chunk a
// single bulk copy lands conflict-free in shared memory.
__host__ __device__ __forceinline__ int swz(int major, int minor) {
  return major * TB + (minor ^ ((major & 3) << 2));
}

__host__ __device__ __forceinline__ int64_t tri_index(int64_t K, int64_t Lc) {
  return K * (K + 1) / 2 + Lc;   // lower block-triangle tile (K >= Lc)
}

// C -= acc for a warp's MI x 4 DMMA fragments (8 rows x 8 columns each) of a
// 128x128 swizzled tile in global memory.  A plain `*cp -= acc` per element
// serialises 8 MI load-use-store round trips to L2 (the stores may alias the
// next loads); here fragment row mi+1 is loaded before row mi is stored, so
// one round trip per fragment row overlaps the previous row's stores.
template <int MI>
__device__ __forceinline__ void tile_sub_acc(double* __restrict__ Ct, const double (&acc)[MI][4][2], int wm, int wn,
                                             int gq, int t) {
  double cur[8], nxt[8];
  auto load_row = [&](int mi, double (&v)[8]) {
    const int m = wm * 64 + mi * 8 + gq;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) v[ni * 2 + e] = __ldcg(Ct + swz(wn * 32 + ni * 8 + 2 * t + e, m));
  };
  load_row(0, cur);
#pragma unroll
  for (int mi = 0; mi < MI; ++mi) {
    if (mi + 1 < MI) load_row(mi + 1, nxt);
    const int m = wm * 64 + mi * 8 + gq;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) Ct[swz(wn * 32 + ni * 8 + 2 * t + e, m)] = cur[ni * 2 + e] - acc[mi][ni][e];
    if (mi + 1 < MI)
#pragma unroll
      for (int k = 0; k < 8; ++k) cur[k] = nxt[k];
  }
}

// upper triangle of apply tiles, row-major over tile rows
__host__ __device__ __forceinline__ int64_t apply_tile_index(int64_t ti, int64_t tj, int64_t T32) {
  return ti * T32 - ti * (ti - 1) / 2 + (tj - ti);
}

// Per-subdomain device descriptor (all pointers device).
struct SubDev {
  const double* raw;        // factor values, reference CSR-of-U order
  const int64_t* up;        // pattern (nullptr => dense packed col-major lower)
  const int64_t* ui;
  double* tiles;            // T(T+1)/2 tiles, col-major swizzled
  double* X;                // P panels x (T*128 rows) x 128, row-major swizzled
  double* F;                // apply tiles (upper triangle of 32x32 tiles)
  double* U;                // path "trsm": u = L_ll^T Y panels (X layout), or nullptr
  double* Y;                // path "trsm": Y = L^-T X panels (X layout)
  double* Lt;               // path "trsm": transposed trailing tiles (slot of (l, k) holds Lhat_lk^T, inv(L_kk)^T)
  const double* U1;         // sparse route, fused correction in the SYRK epilogue (kr > 0):
  const double* U2W;        //   F[a][b] += U1[a] . W[b] - U2[a] . U1[b]  (feti_sparse.h SpSub)
  const int* r_sorted;      // P*128 first rows, sorted ascending, BIG_ROW pads
  const double* s_sorted;   // P*128 signs (0 for pads)
  const int* gids_sorted;   // T32*32 global multiplier ids (-1 pads)
  const int* panel_minrow;  // P
  int64_t nnz;
  int64_t raw_off;          // raw points at value index raw_off (suffix upload)
  int n, m, T, P, T32;
  int smin;                 // first block row any X column reaches (pruning)
  int tbase;                // first block row/column stored in `tiles`
  int src;                  // factor source: SRC_RAW_DENSE / SRC_RAW_SPARSE / SRC_TILES
  int kr;                   // kernel dimension of the fused correction (0: none)
};

enum { SRC_RAW_DENSE = 0, SRC_RAW_SPARSE = 1, SRC_TILES = 2 };

// Only block rows/columns >= smin are ever touched by the assembly: X = L^-1
// P B~^T is zero above the smallest first row of the subdomain, so the X
// panels and the factor upload start there and, for host factors, so do the
// stored tiles (tbase = smin).  A factor computed on the device keeps every
// tile (tbase = 0): the factorization and full solves need them.
__host__ __device__ __forceinline__ int64_t tile_offset(int tbase, int K, int Lc) {
  return tri_index(K - tbase, Lc - tbase) * TILE;
}
__device__ __forceinline__ double* tile_ptr(const SubDev& S, int K, int Lc) {
  return S.tiles + tile_offset(S.tbase, K, Lc);
}
// X panel c, global row `row` (>= smin*128), row-major swizzled, 128 wide
__device__ __forceinline__ double* xrow_ptr(const SubDev& S, int c, int row) {
  return S.X + (size_t)c * (S.T - S.smin) * TILE + (size_t)(row - S.smin * TB) * TB;
}
// the same layout in another panel buffer (U, Y of the TRSM path)
__device__ __forceinline__ double* panel_row_ptr(const SubDev& S, double* base, int c, int row) {
  return base + (size_t)c * (S.T - S.smin) * TILE + (size_t)(row - S.smin * TB) * TB;
}

// ---- PTX wrappers ------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 1-D bulk copy global -> shared (TMA engine), completes on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Bulk prefetch of a global range into L2 (TMA engine, no completion).
__device__ __forceinline__ void bulk_prefetch_l2(const void* gsrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(gsrc), "r"(bytes) : "memory");
}

// 8-byte asynchronous global->shared copy (LDGSTS) for gathers whose source
// alignment rules out bulk copies (the reference's packed factor columns).
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Arrive on `bar` once all of this thread's prior cp.async copies landed.
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// Order this thread's generic-proxy shared-memory accesses before later
// async-proxy (bulk copy) writes to the same buffer (ring-slot release).
__device__ __forceinline__ void fence_proxy_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// Make this thread's generic-proxy global writes visible to later async-proxy
// (bulk copy) reads.
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}

}  // namespace feti
