// Device kernels of the explicit FETI local dual operator (sm_100a).
//
// Assembly of F~_i = X^T X with X = L^-1 P B~^T (
// reference dualop.py:427-501, sparse.py:469-563, _kernels.py:168-214,299-305):
//
//   1. unpack   raw factor (CSR-of-U == packed col-major L)  -> 128x128 tiles
//   2. diaginv  inv(L_kk) of every diagonal block             -> tile (k,k)
//   3. scale    Lhat_kl = inv(L_kk) L_kl  (block-row scaling, l<k)  [DMMA]
//   4. trsm     per (subdomain, 128-column panel) chain:            [DMMA]
//                 X_k = inv(L_kk) Z_k - sum_{l=s..k-1} Lhat_kl X_l
//               Z = P B~^T is never materialised: each column is one +-1 at
//               its first row r_j, so inv(L_kk) Z_k is a signed column gather
//               of tile (k,k); panels start at their first nonzero block row.
//   5. syrk     F_IJ = sum_rows X_I^T X_J over rows >= max(first rows) [DMMA]
//               written as packed upper-triangle 32x32 tiles for the apply.
//
// Apply q = sum_i B~_i^T F~_i B~_i p (dualop.py:348-388, _kernels.py:274-287):
//   6. apply    gather p~ into smem, stream every stored tile once, row sums via
//               a butterfly transpose-reduce, column sums in registers;
//               per-warp smem accumulators combined in fixed order
//   7. reduce   q[g] = sum over (subdomain, local) contributions in the
//               reference's fixed gather order (dualop.py:375-379).
#include <cstdio>
#include <cstdlib>

#include "feti_common.cuh"
#include "feti_apply.cuh"
#include "feti_dense128.cuh"
#include "feti_kernels.h"

namespace feti {

// ---------------------------------------------------------------------------
// 1. unpack
// ---------------------------------------------------------------------------
// work: (sub, K, Lc, -).  Dense pattern: column j of L = raw[colstart(j) ..]
// with rows j..n-1 (reference: rows of U, diagonal first, sparse.py:9-15).
// raw == nullptr (sparse pattern) => zero fill, then the scatter kernel.
__global__ void __launch_bounds__(256) unpack_dense_kernel(const SubDev* __restrict__ subs,
                                                           const int4* __restrict__ work) {
  const int4 w = work[blockIdx.x];
  const SubDev& S = subs[w.x];
  const int K = w.y, Lc = w.z;
  const int64_t n = S.n;
  double* tile = tile_ptr(S, K, Lc);
  const bool dense = (S.src == SRC_RAW_DENSE);
  for (int idx = threadIdx.x; idx < TILE; idx += blockDim.x) {
    const int jl = idx >> 7;
    const int il = (idx & 127) ^ ((jl & 3) << 2);
    const int64_t i = (int64_t)K * TB + il, j = (int64_t)Lc * TB + jl;
    double v = 0.0;
    if (i < n && j < n) {
      if (dense && i >= j) v = __ldcs(S.raw + ((j * n - j * (j - 1) / 2) + (i - j) - S.raw_off));
    } else if (i == j) {
      v = 1.0;  // identity padding keeps the diagonal blocks invertible
    }
    tile[idx] = v;
  }
}

// Sparse pattern: one CTA per factor column j >= smin*128 (row j of U)
__global__ void __launch_bounds__(256) scatter_sparse_kernel(const SubDev* __restrict__ subs, int sub) {
  const SubDev& S = subs[sub];
  const int64_t j = (int64_t)S.smin * TB + blockIdx.x;
  const int64_t b = S.up[j], e = S.up[j + 1];
  const int Lc = (int)(j / TB), jl = (int)(j % TB);
  for (int64_t p = b + threadIdx.x; p < e; p += blockDim.x) {
    const int64_t i = S.ui[p];
    const int K = (int)(i / TB), il = (int)(i % TB);
    tile_ptr(S, K, Lc)[swz(jl, il)] = S.raw[p - S.raw_off];
  }
}

// ---------------------------------------------------------------------------
// 2. inverse of each diagonal block, blocked 4 x 4 over 32-wide sub-blocks
// ---------------------------------------------------------------------------
// Phase 1: warp w inverts the 32x32 diagonal sub-block D_w; lane c carries
// column c of inv(D_w) in registers through a lock-step forward substitution
// (the L row is a shared-memory broadcast).  Phase 2: the off-diagonal
// sub-blocks by distance d = 1, 2, 3:  Y_IJ = -inv(D_I) sum_{K=J}^{I-1} L_IK Y_KJ.
// L and Y live as packed lower triangles in shared memory.
__global__ void __launch_bounds__(256) diag_inverse_kernel(const SubDev* __restrict__ subs,
                                                           const int4* __restrict__ work) {
  // L_kk into a row-major 128 x PO_LD array, then the tensor-pipe inverse of
  // the device factorization (po_inverse): four 32x32 diagonal-block
  // substitutions + DMMA off-diagonal blocks (round 1 used scalar FMA loops
  // for those: 54 us per block)
  extern __shared__ double dsm[];
  double* sA = dsm;                   // TB x PO_LD: L lower, inv(L)^T strict upper
  double* sYd = dsm + TB * PO_LD;     // 1 / L(i, i), then the inverse's diagonal
  double* sT = sYd + TB;              // 3 x 1024 scratch
  const int4 w = work[blockIdx.x];
  const SubDev& S = subs[w.x];
  const int k = w.y;
  double* tile = tile_ptr(S, k, k);
  const int tid = threadIdx.x;
  if (S.src == SRC_RAW_DENSE) {
    // dense pattern: the diagonal block straight from the packed factor
    const int64_t n = S.n;
    for (int idx = tid; idx < TILE; idx += 256) {
      const int jl = idx >> 7, il = idx & 127;
      if (il < jl) continue;
      const int64_t i = (int64_t)k * TB + il, j = (int64_t)k * TB + jl;
      double v;
      if (i < n)
        v = S.raw[(j * n - j * (j - 1) / 2) + (i - j) - S.raw_off];
      else
        v = (i == j) ? 1.0 : 0.0;    // identity padding
      sA[il * PO_LD + jl] = v;
    }
  } else {
    for (int idx = tid; idx < TILE; idx += 256) {
      const int jl = idx >> 7;
      const int il = (idx & 127) ^ ((jl & 3) << 2);
      if (il >= jl) sA[il * PO_LD + jl] = tile[idx];
    }
  }
  __syncthreads();
  if (tid < TB) sYd[tid] = 1.0 / sA[tid * PO_LD + tid];
  __syncthreads();
  po_inverse(sA, sYd, sT);
  for (int idx = tid; idx < TILE; idx += 256) {
    const int jl = idx >> 7;
    const int il = (idx & 127) ^ ((jl & 3) << 2);
    tile[idx] = il > jl ? sA[jl * PO_LD + il] : (il == jl ? sYd[il] : 0.0);
  }
}

// ---------------------------------------------------------------------------
// 3. block-row scaling  Lhat_kl = inv(L_kk) * L_kl  for smin <= l < k
// ---------------------------------------------------------------------------
// One CTA per block row (sub, k): inv(L_kk) stays resident in shared memory
// (128 KB, bulk copy) while the row's L_kl are streamed through a 3-stage ring
// of 32-column quarters.  Dense pattern: quarters are gathered straight from
// the reference's packed factor with 8-byte cp.async (no unpacked copy of L
// is ever written); sparse pattern: bulk copies of the scattered tiles.
// The producer warp fills the ring, 8 DMMA warps compute 128x32 per quarter
// (inv(L_kk) is lower triangular: k-steps above each warp's rows are skipped).
constexpr int BS_STAGES = 3;
constexpr int QCOLS = 32;
constexpr int QSIZE = QCOLS * TB;   // 4096 doubles (32 KB)
constexpr int BS_THREADS = 256;

// Issue the copies of quarter qi of row k into `dst` (all 256 threads).
__device__ __forceinline__ void bs_load_quarter(const SubDev& S, int k, int qi, double* dst, bool dense) {
  const int l = S.tbase + qi / (TB / QCOLS), q = qi % (TB / QCOLS);
  if (dense) {
    // column jg of L: rows k*128 + kk at raw[colstart(jg) + (i - jg)]; thread
    // (jq, kk-quarter): 4 columns x 32 consecutive rows per warp -> coalesced
    const int64_t n = S.n;
    const int64_t i0 = (int64_t)k * TB;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int c = 0; c < QCOLS / 8; ++c) {
      const int jq = warp * (QCOLS / 8) + c;
      const int64_t jg = (int64_t)l * TB + q * QCOLS + jq;
      const double* col = S.raw + (jg * n - jg * (jg - 1) / 2 - jg - S.raw_off);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int kk = lane + 32 * t;
        if (i0 + kk < n) cp_async8(dst + swz(jq, kk), col + i0 + kk);
      }
    }
  } else {
    const double* src = tile_ptr(S, k, l) + q * QSIZE;
    for (int idx = threadIdx.x * 2; idx < QSIZE; idx += BS_THREADS * 2) cp_async16(dst + idx, src + idx);
  }
}

// k-steps [kb0, kb1) for the row groups M0..3 of this warp (all active).
// Even and odd k-steps accumulate into separate registers so that each warp
// keeps twice as many independent DMMA chains in flight (the tail phases have
// only 1-2 active row groups).
template <int M0>
__device__ __forceinline__ void bs_step(int kb, double (&acc)[4][2][2], const int (&rg)[4],
                                        const double* __restrict__ sA, const double* __restrict__ b_s, int wn,
                                        int g, int t, int rows_valid) {
  const int kk = kb * 4 + t;
  double bf[2], af[4];
#pragma unroll
  for (int ni = 0; ni < 2; ++ni) {
    const double v = b_s[swz(wn * 16 + ni * 8 + g, kk)];
    bf[ni] = kk < rows_valid ? v : 0.0;
  }
#pragma unroll
  for (int mi = M0; mi < 4; ++mi) af[mi] = sA[swz(kk, rg[mi] * 8 + g)];
#pragma unroll
  for (int mi = M0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
}

template <int M0>
__device__ __forceinline__ void bs_steps(int kb0, int kb1, double (&acc)[4][2][2], double (&acc2)[4][2][2],
                                         const int (&rg)[4], const double* __restrict__ sA,
                                         const double* __restrict__ b_s, int wn, int g, int t, int rows_valid) {
  int kb = kb0;
  for (; kb + 1 < kb1; kb += 2) {
    bs_step<M0>(kb, acc, rg, sA, b_s, wn, g, t, rows_valid);
    bs_step<M0>(kb + 1, acc2, rg, sA, b_s, wn, g, t, rows_valid);
  }
  if (kb < kb1) bs_step<M0>(kb, acc, rg, sA, b_s, wn, g, t, rows_valid);
}

__global__ void __launch_bounds__(BS_THREADS, 1) block_scale_kernel(const SubDev* __restrict__ subs,
                                                                    const int4* __restrict__ work) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sA = reinterpret_cast<double*>(smem_raw);      // TILE
  double* sB = sA + TILE;                                 // BS_STAGES * QSIZE
  uint64_t* barA = reinterpret_cast<uint64_t*>(sB + BS_STAGES * QSIZE);
  const int4 w = work[blockIdx.x];
  const SubDev S = subs[w.x];   // by value: no reloads after the epilogue's global stores
  const int k = w.y;
  const int nq = (k - S.tbase) * (TB / QCOLS);
  const bool dense = (S.src == SRC_RAW_DENSE);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(barA, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(barA, TILE * 8);
    const double* inv = tile_ptr(S, k, k);
    for (int s = 0; s < 4; ++s) bulk_g2s(sA + s * SLICE, inv + s * SLICE, SLICE * 8, barA);
  }
  // classic multistage cp.async ring for the L_kl quarters (every thread
  // issues 16 of the 8-byte copies of a quarter; the sources are the
  // reference's packed columns, whose alignment rules out bulk copies)
#pragma unroll
  for (int st = 0; st < BS_STAGES - 1; ++st) {
    if (st < nq) bs_load_quarter(S, k, st, sB + st * QSIZE, dense);
    cp_async_commit();
  }
  // inv(L_kk) is lower triangular: 8-row group r needs k-steps kb <= 2r+1.
  // Each warp takes 4 row groups whose triangular costs sum to the same 68
  // DMMA k-steps ({w, 15-w, 7-w, 8+w}), so no warp idles at the quarter end.
  const int wm = warp >> 1, wn = warp & 1;     // 4 row groups x 16 columns of 128 x 32
  const int g = lane >> 2, t = lane & 3;
  const int rg[4] = {wm, 7 - wm, 8 + wm, 15 - wm};
  const int rows_valid = S.n - k * TB;         // padding rows of the last block row
  mbar_wait(barA, 0);
  for (int qi = 0; qi < nq; ++qi) {
    cp_async_wait_group<BS_STAGES - 2>();
    __syncthreads();                           // quarter qi landed; stage (qi-1) free
    const int nx = qi + BS_STAGES - 1;
    if (nx < nq) bs_load_quarter(S, k, nx, sB + (nx % BS_STAGES) * QSIZE, dense);
    cp_async_commit();
    const double* b_s = sB + (qi % BS_STAGES) * QSIZE;
    double acc[4][2][2], acc2[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = acc2[a][b][0] = acc2[a][b][1] = 0.0;
    // rg ascending (w < 7-w < 8+w < 15-w): the active row groups shrink at
    // k-step 2w+2, 16-2w, 18+2w; each phase runs a fixed, unrolled set
    bs_steps<0>(0, 2 * wm + 2, acc, acc2, rg, sA, b_s, wn, g, t, rows_valid);
    bs_steps<1>(2 * wm + 2, 16 - 2 * wm, acc, acc2, rg, sA, b_s, wn, g, t, rows_valid);
    bs_steps<2>(16 - 2 * wm, 18 + 2 * wm, acc, acc2, rg, sA, b_s, wn, g, t, rows_valid);
    bs_steps<3>(18 + 2 * wm, 32 - 2 * wm, acc, acc2, rg, sA, b_s, wn, g, t, rows_valid);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        acc[a][b][0] += acc2[a][b][0];
        acc[a][b][1] += acc2[a][b][1];
      }
    const int l = S.tbase + qi / (TB / QCOLS), q = qi % (TB / QCOLS);
    double* Lkl = tile_ptr(S, k, l);
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int i = rg[mi] * 8 + g;
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) {
        const int j = q * QCOLS + wn * 16 + ni * 8 + 2 * t;
        Lkl[swz(j, i)] = acc[mi][ni][0];
        Lkl[swz(j + 1, i)] = acc[mi][ni][1];
      }
    }
  }
  cp_async_wait_group<0>();
}

// ---------------------------------------------------------------------------
// shared consumer micro-kernel: 128x128 CTA tile, 8 warps of 64x32,
// one 32-deep slice of A ([k][m] swizzled) and B ([k][n] swizzled).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mma_slice_128x128(const double* __restrict__ a_s,
                                                  const double* __restrict__ b_s, double (&acc)[8][4][2],
                                                  int wm, int wn, int g, int t) {
#pragma unroll
  for (int kb = 0; kb < KS / 4; ++kb) {
    const int kr = kb * 4 + t;
    double bf[4];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) bf[ni] = b_s[swz(kr, wn * 32 + ni * 8 + g)];
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) {
      const double af = a_s[swz(kr, wm * 64 + mi * 8 + g)];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af, bf[ni]);
    }
  }
}

constexpr int PIPE_STAGES = 3;
constexpr int PIPE_THREADS = 288;   // 8 DMMA warps + 1 bulk-copy producer warp

// ---------------------------------------------------------------------------
// 4. pruned forward solve, one (subdomain, panel) chain per CTA
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(PIPE_THREADS, 1) trsm_chain_kernel(const SubDev* __restrict__ subs,
                                                                     const int4* __restrict__ work) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sA = reinterpret_cast<double*>(smem_raw);
  double* sB = sA + PIPE_STAGES * SLICE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + PIPE_STAGES * SLICE);
  uint64_t* empty = full + PIPE_STAGES;
  uint64_t* xready = empty + PIPE_STAGES;

  const int4 w = work[blockIdx.x];
  const SubDev& S = subs[w.x];
  const int c = w.y;
  const int T = S.T;
  const int s0 = S.panel_minrow[c] / TB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < PIPE_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 8);
    }
    mbar_init(xready, 8);
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == 8) {  // ---- producer: bulk copies of Lhat_kl and X_l slices
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int k = s0 + 1; k < T; ++k) {
        for (int l = s0; l < k; ++l) {
          if (l == k - 1) mbar_wait(xready, (uint32_t)((k - 1 - s0) & 1));
          const double* At = tile_ptr(S, k, l);
          const double* Bt = xrow_ptr(S, c, l * TB);
          for (int s = 0; s < TB / KS; ++s) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full[stage], 2 * SLICE * 8);
            bulk_g2s(sA + stage * SLICE, At + s * SLICE, SLICE * 8, &full[stage]);
            bulk_g2s(sB + stage * SLICE, Bt + s * SLICE, SLICE * 8, &full[stage]);
            if (++stage == PIPE_STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
    return;
  }

  // ---- consumers
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t = lane & 3;
  int rj[4][2];
  double sj[4][2];
#pragma unroll
  for (int ni = 0; ni < 4; ++ni)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = c * TB + wn * 32 + ni * 8 + 2 * t + e;
      rj[ni][e] = S.r_sorted[j];
      sj[ni][e] = S.s_sorted[j];
    }
  int stage = 0;
  uint32_t phase = 0;
  for (int k = s0; k < T; ++k) {
    double acc[8][4][2];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    const int nsl = (k - s0) * (TB / KS);
    for (int sl = 0; sl < nsl; ++sl) {
      mbar_wait(&full[stage], phase);
      mma_slice_128x128(sA + stage * SLICE, sB + stage * SLICE, acc, wm, wn, g, t);
      fence_proxy_async_shared();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == PIPE_STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }
    // epilogue: X_k = inv(L_kk) Z_k - acc
    const double* inv = tile_ptr(S, k, k);
    double* Xk = xrow_ptr(S, c, k * TB);
    const int kb0 = k * TB;
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) {
      const int i = wm * 64 + mi * 8 + g;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        double v[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int rr = rj[ni][e] - kb0;
          double pv = 0.0;
          if (rr >= 0 && rr < TB && i >= rr) pv = sj[ni][e] * inv[swz(rr, i)];
          v[e] = pv - acc[mi][ni][e];
        }
        const int j0 = wn * 32 + ni * 8 + 2 * t;
        *reinterpret_cast<double2*>(Xk + swz(i, j0)) = make_double2(v[0], v[1]);
      }
    }
    fence_proxy_async_global();
    __syncwarp();
    if (lane == 0) mbar_arrive(xready);
  }
}

// ---------------------------------------------------------------------------
// 4b. path "trsm" (assemble_explicit_local with config.path == "trsm",
// dualop.py:472-479): the second triangular solve Y = L^-T X and the row
// gather F = B~ Y (spmm_rows) instead of the SYRK.
//   transpose_trail_kernel  Lt(l, k) = Lhat_lk^T, Lt(k, k) = inv(L_kk)^T (smin <= k <= l)
//   backward_chain_kernel   per (subdomain, panel), k = T-1 .. smin:
//                             u_k = X_k - sum_{l>k} Lhat_lk^T u_l   (u_l = L_ll^T Y_l)
//                             Y_k = inv(L_kk)^T u_k
//   trsm_gather_kernel      F[a][b] = s_a Y[r_a][b] (upper), diagonal tiles mirrored
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) transpose_trail_kernel(const SubDev* __restrict__ subs,
                                                              const int4* __restrict__ work) {
  __shared__ double blk[32][33];
  const int4 w = work[blockIdx.x];
  const SubDev& S = subs[w.x];
  const int l = w.y;
  if (l < S.smin) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int k = S.smin; k <= l; ++k) {
    const double* src = tile_ptr(S, l, k);
    double* dst = S.Lt + tile_offset(S.smin, l, k);
    // 32x32 blocks: dst[swz(a, b)] = src[swz(b, a)]
    for (int bb = 0; bb < 16; ++bb) {
      const int a0 = (bb >> 2) * 32, b0 = (bb & 3) * 32;
      for (int y = ty; y < 32; y += 8) blk[y][tx] = src[swz(b0 + y, a0 + tx)];
      __syncthreads();
      for (int y = ty; y < 32; y += 8) dst[swz(a0 + y, b0 + tx)] = blk[tx][y];
      __syncthreads();
    }
  }
}

// consumer side of the bulk-copy ring: acc = sum of nsl (A, B) slices
__device__ __forceinline__ void pipe_consume(int nsl, double (&acc)[8][4][2], const double* sA, const double* sB,
                                             uint64_t* full, uint64_t* empty, int& stage, uint32_t& phase, int wm,
                                             int wn, int g, int t, int lane) {
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int sl = 0; sl < nsl; ++sl) {
    mbar_wait(&full[stage], phase);
    mma_slice_128x128(sA + stage * SLICE, sB + stage * SLICE, acc, wm, wn, g, t);
    fence_proxy_async_shared();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == PIPE_STAGES) {
      stage = 0;
      phase ^= 1;
    }
  }
}

__global__ void __launch_bounds__(PIPE_THREADS, 1) backward_chain_kernel(const SubDev* __restrict__ subs,
                                                                         const int4* __restrict__ work) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sA = reinterpret_cast<double*>(smem_raw);
  double* sB = sA + PIPE_STAGES * SLICE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + PIPE_STAGES * SLICE);
  uint64_t* empty = full + PIPE_STAGES;
  uint64_t* uready = empty + PIPE_STAGES;

  const int4 w = work[blockIdx.x];
  const SubDev& S = subs[w.x];
  const int c = w.y;
  const int T = S.T, s0 = S.smin;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < PIPE_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 8);
    }
    mbar_init(uready, 8);
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == 8) {  // ---- producer: (Lhat_lk^T, u_l) slices, then (inv(L_kk)^T, u_k)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      auto issue = [&](const double* At, const double* Bt) {
        for (int sl = 0; sl < TB / KS; ++sl) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], 2 * SLICE * 8);
          bulk_g2s(sA + stage * SLICE, At + sl * SLICE, SLICE * 8, &full[stage]);
          bulk_g2s(sB + stage * SLICE, Bt + sl * SLICE, SLICE * 8, &full[stage]);
          if (++stage == PIPE_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      };
      for (int k = T - 1; k >= s0; --k) {
        for (int l = T - 1; l > k; --l)
          issue(S.Lt + tile_offset(s0, l, k), panel_row_ptr(S, S.U, c, l * TB));
        mbar_wait(uready, (uint32_t)((T - 1 - k) & 1));   // u_k written by the consumers
        issue(S.Lt + tile_offset(s0, k, k), panel_row_ptr(S, S.U, c, k * TB));
      }
    }
    return;
  }

  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t = lane & 3;
  int stage = 0;
  uint32_t phase = 0;
  double acc[8][4][2];
  for (int k = T - 1; k >= s0; --k) {
    pipe_consume((T - 1 - k) * (TB / KS), acc, sA, sB, full, empty, stage, phase, wm, wn, g, t, lane);
    // u_k = X_k - acc (X_k is zero above the panel's first block row and
    // was never written there by the forward chain)
    const double* Xk = xrow_ptr(S, c, k * TB);
    double* Uk = panel_row_ptr(S, S.U, c, k * TB);
    const bool xnz = k >= S.panel_minrow[c] / TB;
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) {
      const int i = wm * 64 + mi * 8 + g;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int j0 = wn * 32 + ni * 8 + 2 * t;
        const double2 x = xnz ? *reinterpret_cast<const double2*>(Xk + swz(i, j0)) : make_double2(0.0, 0.0);
        *reinterpret_cast<double2*>(Uk + swz(i, j0)) = make_double2(x.x - acc[mi][ni][0], x.y - acc[mi][ni][1]);
      }
    }
    fence_proxy_async_global();
    __syncwarp();
    if (lane == 0) mbar_arrive(uready);
    // Y_k = inv(L_kk)^T u_k
    pipe_consume(TB / KS, acc, sA, sB, full, empty, stage, phase, wm, wn, g, t, lane);
    double* Yk = panel_row_ptr(S, S.Y, c, k * TB);
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) {
      const int i = wm * 64 + mi * 8 + g;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int j0 = wn * 32 + ni * 8 + 2 * t;
        *reinterpret_cast<double2*>(Yk + swz(i, j0)) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
      }
    }
  }
}

// one CTA per (subdomain, panel c): the 4 tile columns of F that panel c's
// 128 columns make up, rows a <= b
__global__ void __launch_bounds__(256) trsm_gather_kernel(const SubDev* __restrict__ subs,
                                                          const int4* __restrict__ work) {
  const int4 w = work[blockIdx.x];
  const SubDev& S = subs[w.x];
  const int c = w.y, T32 = S.T32;
  auto yval = [&](int a, int b) -> double {   // s_a Y[r_a][b] (0 for padding rows/columns)
    if (a >= S.m || b >= S.m) return 0.0;
    const int ra = S.r_sorted[a];
    const double* yr = panel_row_ptr(S, S.Y, b / TB, ra);
    return S.s_sorted[a] * yr[(b % TB) ^ ((ra & 3) << 2)];
  };
  for (int tj = c * (TB / AT); tj < min((c + 1) * (TB / AT), T32); ++tj)
    for (int ti = 0; ti <= tj; ++ti) {
      double* F = S.F + apply_tile_index(ti, tj, T32) * ATILE;
      for (int e = threadIdx.x; e < ATILE; e += 256) {
        const int al = e / AT, bl = e % AT;
        const int a = ti * AT + al, b = tj * AT + bl;
        F[e] = (ti == tj && al > bl) ? yval(b, a) : yval(a, b);
      }
    }
}

// ---------------------------------------------------------------------------
// 5. SYRK  F_IJ = X_I^T X_J  (I <= J), pruned to rows >= max first row
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(PIPE_THREADS, 1) syrk_kernel(const SubDev* __restrict__ subs,
                                                               const int4* __restrict__ work) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sA = reinterpret_cast<double*>(smem_raw);
  double* sB = sA + PIPE_STAGES * SLICE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + PIPE_STAGES * SLICE);
  uint64_t* empty = full + PIPE_STAGES;

  const int4 w = work[blockIdx.x];
  const SubDev& S = subs[w.x];
  const int I = w.y, J = w.z;
  const int rstart = max(S.panel_minrow[I], S.panel_minrow[J]) & ~(KS - 1);
  const int rend = (S.n + KS - 1) & ~(KS - 1);
  const int nsl = (rend - rstart) / KS;
  const double* XI = xrow_ptr(S, I, rstart);
  const double* XJ = xrow_ptr(S, J, rstart);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < PIPE_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 8);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == 8) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int sl = 0; sl < nsl; ++sl) {
        const size_t off = (size_t)sl * KS * TB;
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], 2 * SLICE * 8);
        bulk_g2s(sA + stage * SLICE, XI + off, SLICE * 8, &full[stage]);
        bulk_g2s(sB + stage * SLICE, XJ + off, SLICE * 8, &full[stage]);
        if (++stage == PIPE_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }

  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t = lane & 3;
  // diagonal blocks: warps strictly below the diagonal produce nothing stored
  const bool idle = (I == J) && (wn * 32 + 31 < wm * 64);
  double acc[8][4][2];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  int stage = 0;
  uint32_t phase = 0;
  for (int sl = 0; sl < nsl; ++sl) {
    mbar_wait(&full[stage], phase);
    if (!idle) mma_slice_128x128(sA + stage * SLICE, sB + stage * SLICE, acc, wm, wn, g, t);
    fence_proxy_async_shared();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == PIPE_STAGES) {
      stage = 0;
      phase ^= 1;
    }
  }
  const int T32 = S.T32;
  if (S.kr > 0) {
    // sparse route: + U1[a] . W[b] - U2[a] . U1[b]  (W = C U1 - U2; U2W rows hold [U2 | W])
    const int r = S.kr;
    for (int q = 0; q < r; ++q) {
      double u1b[4][2], wb[4][2];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int b = J * TB + wn * 32 + ni * 8 + 2 * t + e;
          u1b[ni][e] = S.U1[(size_t)b * r + q];
          wb[ni][e] = S.U2W[(size_t)b * 2 * r + r + q];
        }
#pragma unroll
      for (int mi = 0; mi < 8; ++mi) {
        const int a = I * TB + wm * 64 + mi * 8 + g;
        const double u1a = S.U1[(size_t)a * r + q], u2a = S.U2W[(size_t)a * 2 * r + q];
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) acc[mi][ni][e] += u1a * wb[ni][e] - u2a * u1b[ni][e];
      }
    }
  }
#pragma unroll
  for (int mi = 0; mi < 8; ++mi) {
    const int a = I * TB + wm * 64 + mi * 8 + g;
    const int ti = a >> 5;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int b = J * TB + wn * 32 + ni * 8 + 2 * t;
      const int tj = b >> 5;
      if (ti <= tj && tj < T32) {
        double* dst = S.F + apply_tile_index(ti, tj, T32) * ATILE + (a & 31) * AT + (b & 31);
        *reinterpret_cast<double2*>(dst) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// 6. apply: batched packed SYMV fused with the B~ gather/scatter
// ---------------------------------------------------------------------------
template <int NW>
__global__ void __launch_bounds__(NW * 32) apply_kernel(const SubDev* __restrict__ subs,
                                                        const ApplySeg* __restrict__ segs,
                                                        const int* __restrict__ seg_ptr,
                                                        double* __restrict__ part,
                                                        const double* __restrict__ p,
                                                        const double* __restrict__ py,
                                                        const double* __restrict__ pbeta,
                                                        const int* __restrict__ done, int sb) {
  apply_body<NW>(subs, segs, seg_ptr, part, p, py, pbeta, done, sb);
}

// ---------------------------------------------------------------------------
// 7. ordered reduction into the global dual vector
// ---------------------------------------------------------------------------
// per global multiplier: its (subdomain, local) contributions in the
// reference's gather order (dualop.py:375-379); contribution e sums the
// partials ridx[cent[e].y .. cent[e].z) of the super-block segments that
// touched it, in segment order
__global__ void __launch_bounds__(256) reduce_kernel(int n_mult, const int* __restrict__ cptr,
                                                     const int4* __restrict__ cent,
                                                     const int64_t* __restrict__ ridx,
                                                     const double* __restrict__ part, double* __restrict__ q) {
  const int gidx = blockIdx.x * blockDim.x + threadIdx.x;
  if (gidx >= n_mult) return;
  double acc = 0.0;
  for (int e = cptr[gidx]; e < cptr[gidx + 1]; ++e) {
    const int4 c = cent[e];
    double v = 0.0;
    for (int k = c.y; k < c.z; ++k) v += part[ridx[k]];
    acc += v;
  }
  q[gidx] = acc;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static size_t pipe_smem() { return 2 * PIPE_STAGES * SLICE * sizeof(double) + 8 * (2 * PIPE_STAGES + 1); }
static size_t scale_smem() { return (TILE + BS_STAGES * QSIZE) * sizeof(double) + 16; }

cudaError_t configure_kernels() {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(trsm_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pipe_smem())))
    return e;
  if ((e = cudaFuncSetAttribute(backward_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)pipe_smem())))
    return e;
  if ((e = cudaFuncSetAttribute(syrk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pipe_smem())))
    return e;
  if ((e = cudaFuncSetAttribute(block_scale_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)scale_smem())))
    return e;
  if ((e = cudaFuncSetAttribute(diag_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                POTRF_SMEM_DOUBLES * 8)))
    return e;
  const void* applies[APPLY_MAX_WARPS] = {
      (const void*)apply_kernel<1>,  (const void*)apply_kernel<2>,  (const void*)apply_kernel<3>,
      (const void*)apply_kernel<4>,  (const void*)apply_kernel<5>,  (const void*)apply_kernel<6>,
      (const void*)apply_kernel<7>,  (const void*)apply_kernel<8>};
  for (int w = 1; w <= APPLY_MAX_WARPS; ++w)
    if ((e = cudaFuncSetAttribute(applies[w - 1], cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)))
      return e;
  return cudaSuccess;
}

void launch_unpack(const SubDev* subs, const int4* work, int nwork, cudaStream_t st) {
  if (nwork > 0) unpack_dense_kernel<<<nwork, 256, 0, st>>>(subs, work);
}
void launch_scatter_sparse(const SubDev* subs, int sub, int n, cudaStream_t st) {
  if (n > 0) scatter_sparse_kernel<<<n, 256, 0, st>>>(subs, sub);
}
void launch_diag_inverse(const SubDev* subs, const int4* work, int nwork, cudaStream_t st) {
  if (nwork > 0) diag_inverse_kernel<<<nwork, 256, POTRF_SMEM_DOUBLES * 8, st>>>(subs, work);
}
void launch_block_scale(const SubDev* subs, const int4* work, int nwork, cudaStream_t st) {
  if (nwork > 0) block_scale_kernel<<<nwork, BS_THREADS, scale_smem(), st>>>(subs, work);
}
void launch_trsm_chain(const SubDev* subs, const int4* work, int nwork, cudaStream_t st) {
  if (nwork > 0) trsm_chain_kernel<<<nwork, PIPE_THREADS, pipe_smem(), st>>>(subs, work);
}
void launch_trsm_path(const SubDev* subs, const int4* wd, int nd, const int4* wc, int nc, cudaStream_t st) {
  if (nd > 0) transpose_trail_kernel<<<nd, 256, 0, st>>>(subs, wd);
  if (nc > 0) {
    backward_chain_kernel<<<nc, PIPE_THREADS, pipe_smem(), st>>>(subs, wc);
    trsm_gather_kernel<<<nc, 256, 0, st>>>(subs, wc);
  }
}

void launch_syrk(const SubDev* subs, const int4* work, int nwork, cudaStream_t st) {
  if (nwork > 0) syrk_kernel<<<nwork, PIPE_THREADS, pipe_smem(), st>>>(subs, work);
}
size_t apply_smem(int nw, int sb) {
  return sb < 0 ? (size_t)(1 + nw) * (-sb) * AT * sizeof(double) : (size_t)(2 + 2 * nw) * sb * AT * sizeof(double);
}

int apply_max_sb(int nw) { return (int)((227 * 1024) / ((size_t)(2 + 2 * nw) * AT * sizeof(double))); }
int apply_max_compact(int nw) { return (int)((227 * 1024) / ((size_t)(1 + nw) * AT * sizeof(double))); }

void launch_apply(int nw, int sb, const SubDev* subs, const ApplySeg* segs, const int* seg_ptr, int nctas,
                  double* part, const double* p, cudaStream_t st, const double* py, const double* pbeta,
                  const int* done) {
  if (nctas <= 0) return;
#define FETI_APPLY_CASE(W) \
  case W:                  \
    apply_kernel<W><<<nctas, W * 32, apply_smem(W, sb), st>>>(subs, segs, seg_ptr, part, p, py, pbeta, done, sb); \
    break;
  switch (nw) {
    FETI_APPLY_CASE(8)
    FETI_APPLY_CASE(7)
    FETI_APPLY_CASE(6)
    FETI_APPLY_CASE(5)
    FETI_APPLY_CASE(4)
    FETI_APPLY_CASE(3)
    FETI_APPLY_CASE(2)
    default: FETI_APPLY_CASE(1)
  }
#undef FETI_APPLY_CASE
}
void launch_reduce(int n_mult, const int* cptr, const int4* cent, const int64_t* ridx, const double* part,
                   double* q, cudaStream_t st) {
  if (n_mult > 0) reduce_kernel<<<(n_mult + 255) / 256, 256, 0, st>>>(n_mult, cptr, cent, ridx, part, q);
}

}  // namespace feti

namespace feti {
// diagnostics: per-kernel register/thread limits (used by tests and debugging)
int kernel_attributes(char* buf, int len) {
  struct K { const char* name; const void* fn; } ks[] = {
      {"unpack_dense", (const void*)unpack_dense_kernel},   {"scatter_sparse", (const void*)scatter_sparse_kernel},
      {"diag_inverse", (const void*)diag_inverse_kernel},   {"block_scale", (const void*)block_scale_kernel},
      {"trsm_chain", (const void*)trsm_chain_kernel},       {"syrk", (const void*)syrk_kernel},
      {"apply8", (const void*)apply_kernel<8>},             {"reduce", (const void*)reduce_kernel}};
  int off = 0;
  for (auto& k : ks) {
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, k.fn);
    off += snprintf(buf + off, len - off, "%s: err=%d regs=%d maxthr=%d smem_static=%zu maxdyn=%d\n", k.name, (int)e,
                    a.numRegs, a.maxThreadsPerBlock, a.sharedSizeBytes, a.maxDynamicSharedSizeBytes);
    if (off >= len) break;
  }
  return off;
}
}  // namespace feti
