// 128x128 dense lower-triangular helpers shared by the assembly's diagonal
// inverse and the device factorizations (256 threads, shared memory).
#pragma once
#include "feti_common.cuh"

namespace feti {

// In-place Cholesky of the 128x128 tile (col-major swizzled, lower part read)
// and its inverse: tile <- L (upper part zeroed), D <- inv(L) (same layout).
// A non-positive pivot is reported as atomicMin(bad, rowbase + j) and
// replaced by 1 so the sweep completes.  Must be called by all 256 threads.
//
// Shared memory: one 128 x 132 row-major array (stride = 4 mod 16 doubles:
// the DMMA fragment loads, rows g8 x columns t4, are bank-conflict free; the
// odd stride 129 made them 4-way and measured 70.0 vs 61.4 us per tile,
// scripts/gpu_potrf.sh, profiles/r01d_potrf_stride.md.  The row-per-lane
// walks -- tile load scatter, diagonal-block row load/store, panel
// substitution, inverse store, writeback -- stay up to 4-way conflicted with
// this stride: 32 rows map to 4 bank groups) holding L in its lower triangle and
// Y = inv(L) transposed in its strict upper triangle (Y(i, j), i > j, at
// [j][i]), the diagonal of Y apart, plus a 3 x 32 x 32 scratch.  Blocked
// over four 32-wide block columns: one warp factors and inverts the 32x32
// diagonal block in registers (shuffle broadcasts), all warps apply it to
// the panel below and update the trailing matrix; the off-diagonal blocks of
// Y follow by distance, Y_IJ = -Y_II sum_{K=J}^{I-1} L_IK Y_KJ.
#ifndef FETI_PO_LD
#define FETI_PO_LD (TB + 4)
#endif
constexpr int PO_LD = FETI_PO_LD;

// Barrier over the 256 threads (warps 0-7) that run potrf_invert_128: a named
// barrier, so a persistent CTA with extra warps can call it.
__device__ __forceinline__ void po_sync() { asm volatile("bar.sync 1, 256;\n" ::: "memory"); }
constexpr int POTRF_SMEM_DOUBLES = TB * PO_LD + TB + 3 * 1024;

// Y = inv(L) for the 128x128 lower-triangular L in sA (row-major, stride
// PO_LD, lower triangle) with sYd[i] = 1 / L(i, i): Y's strict lower triangle
// ends up transposed in sA's strict upper triangle (Y(i, j), i > j, at
// [j][i]) and its diagonal in sYd.  The four 32x32 diagonal blocks by one
// warp each (lane = column, forward substitution), the off-diagonal blocks by
// distance on the tensor pipe: T = sum_{K=J}^{I-1} L_IK Y_KJ, Y_IJ = -Y_II T.
// sT: 3 x 1024 scratch.  Called by all 256 threads; ends synchronised.
__device__ __forceinline__ void po_inverse(double* __restrict__ sA, double* __restrict__ sYd,
                                           double* __restrict__ sT) {
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g8 = lane >> 2, t4 = lane & 3;      // DMMA fragment coordinates
  // inverses of the four 32x32 diagonal blocks, one warp each, lane = column
  if (warp < 4) {
    const int o = warp * 32;
    double y[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const double* Lr = sA + (o + r) * PO_LD + o;
      double a0 = (r == lane) ? 1.0 : 0.0, a1 = 0.0;
#pragma unroll
      for (int j = 0; j < r; ++j) {
        if (j & 1)
          a1 = fma(-Lr[j], y[j], a1);
        else
          a0 = fma(-Lr[j], y[j], a0);
      }
      y[r] = (a0 + a1) * sYd[o + r];
    }
#pragma unroll
    for (int r = 0; r < 32; ++r)
      if (r > lane) sA[(o + lane) * PO_LD + o + r] = y[r];
  }
  po_sync();
  // off-diagonal blocks of Y by distance d on the tensor pipe:
  // T = sum_{K=J}^{I-1} L_IK Y_KJ, then Y_IJ = -Y_II T
  auto ylo = [&](int r, int c) -> double { return r > c ? sA[c * PO_LD + r] : (r == c ? sYd[r] : 0.0); };
  for (int d = 1; d < 4; ++d) {
    const int nb = 4 - d;
    for (int tl = warp; tl < nb * 16; tl += 8) {
      const int bI = tl >> 4, tm = (tl >> 2) & 3, tn = tl & 3;
      const int J = bI, I = bI + d;
      const double* Lr = sA + (I * 32 + tm * 8 + g8) * PO_LD;
      const int cn = J * 32 + tn * 8 + g8;
      double c0v = 0.0, c1v = 0.0;
      for (int k0 = J * 32 + tn * 8; k0 < I * 32; k0 += 4) {
        const int k = k0 + t4;
        dmma(c0v, c1v, Lr[k], ylo(k, cn));
      }
      double* Tb = sT + bI * 1024 + (tm * 8 + g8) * 32 + tn * 8 + 2 * t4;
      Tb[0] = c0v;
      Tb[1] = c1v;
    }
    po_sync();
    for (int tl = warp; tl < nb * 16; tl += 8) {
      const int bI = tl >> 4, tm = (tl >> 2) & 3, tn = tl & 3;
      const int J = bI, I = bI + d;
      const int rm = I * 32 + tm * 8 + g8;
      double c0v = 0.0, c1v = 0.0;
      for (int k0 = 0; k0 < tm * 8 + 8; k0 += 4) {
        const int k = k0 + t4;
        dmma(c0v, c1v, ylo(rm, I * 32 + k), sT[bI * 1024 + k * 32 + tn * 8 + g8]);
      }
      const int m = I * 32 + tm * 8 + g8, n = J * 32 + tn * 8 + 2 * t4;
      sA[n * PO_LD + m] = -c0v;
      sA[(n + 1) * PO_LD + m] = -c1v;
    }
    po_sync();
  }
}

__device__ __forceinline__ void potrf_invert_128(double* __restrict__ tile, double* __restrict__ D,
                                                 int* __restrict__ bad, int rowbase, double* __restrict__ smem) {
  double* sA = smem;                    // [i][j] at i * PO_LD + j
  double* sYd = smem + TB * PO_LD;      // diagonal of Y
  double* sT = sYd + TB;                // 3 x 1024 scratch
  double* colbuf = sT;                  // 32: one column of a diagonal block (scratch is free then)
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g8 = lane >> 2, t4 = lane & 3;      // DMMA fragment coordinates
  // 16 loads in flight per thread (the tile is usually cold in HBM)
  for (int base = 0; base < TILE / 256; base += 16) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = __ldcg(tile + (base + u) * 256 + tid);
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int idx = (base + u) * 256 + tid;
      const int jl = idx >> 7;
      const int il = (idx & 127) ^ ((jl & 3) << 2);
      if (il >= jl) sA[il * PO_LD + jl] = v[u];
    }
  }
  po_sync();
  // Y(r, c) for r >= c (lower triangle of inv(L))
  auto yat = [&](int r, int c) -> double { return r == c ? sYd[r] : sA[c * PO_LD + r]; };
  // trailing update A_ij -= L_ib L_jb^T of source block ob over the lower 8x8
  // tiles of rows/cols >= ob + 32 (DMMA), tiles pidx in [p0, p1) (row-major
  // over tile rows), spread over `nw` warps starting at warp `w0`
  auto trail = [&](int ob, int p0, int p1, int w0, int nw) {
    const int nb = (TB - ob - 32) / 8;
    p1 = min(p1, nb * (nb + 1) / 2);
    for (int pidx = p0 + (warp - w0); pidx < p1; pidx += nw) {
      int I = (int)((sqrt(8.0 * pidx + 1.0) - 1.0) * 0.5);
      while ((I + 1) * (I + 2) / 2 <= pidx) ++I;
      while (I * (I + 1) / 2 > pidx) --I;
      const int J = pidx - I * (I + 1) / 2;
      const int i0 = ob + 32 + 8 * I, j0 = ob + 32 + 8 * J;
      const double* Ar = sA + (i0 + g8) * PO_LD + ob;
      const double* Br = sA + (j0 + g8) * PO_LD + ob;
      double c0v = 0.0, c1v = 0.0;
#pragma unroll
      for (int k0 = 0; k0 < 32; k0 += 4) dmma(c0v, c1v, Ar[k0 + t4], Br[k0 + t4]);
      const int row = i0 + g8, col = j0 + 2 * t4;
      if (I > J || row >= col) sA[row * PO_LD + col] -= c0v;
      if (I > J || row >= col + 1) sA[row * PO_LD + col + 1] -= c1v;
    }
  };
  // Look-ahead: block bb's trailing update is split into the next diagonal
  // block ([o+32, o+64)^2: its first 10 tiles, applied right after the
  // panel) and the rest, which warps 1-7 apply while warp 0 factors that
  // next diagonal block.
  constexpr int kNextDiagTiles = 10;   // 4 x 5 / 2 tiles of 8x8
  for (int bb = 0; bb < 4; ++bb) {
    const int o = bb * 32;
#ifndef PO_SKIP_DIAG
    if (warp == 0) {
      // diagonal block by warp 0 in registers; lane = row,
      // row[j] = A(o+lane, o+j), j <= lane
      double row[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) row[j] = (j <= lane) ? sA[(o + lane) * PO_LD + o + j] : 0.0;
      double rdiag = 1.0;                      // 1 / L(o+lane, o+lane)
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        double d = __shfl_sync(0xffffffffu, row[k], k);
        if (!(d > 0.0)) {
          if (tid == 0) atomicMin(bad, rowbase + o + k);    // first non-positive pivot (permuted row)
          d = 1.0;
        }
        // one rsqrt + multiply instead of sqrt + divide on the serial chain
        // (both are multi-instruction FP64 sequences): 1/L_kk and L_kk
        const double rp = rsqrt(d);
        const double pv = d * rp;
        if (lane == k) rdiag = rp;
        const double lik = (lane == k) ? pv : (lane > k ? row[k] * rp : 0.0);
        row[k] = lik;
        colbuf[lane] = lik;                    // column k, read back as broadcasts
        __syncwarp();
#pragma unroll
        for (int j = k + 1; j < 32; ++j) row[j] = fma(-lik, colbuf[j], row[j]);
        __syncwarp();
      }
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j <= lane) sA[(o + lane) * PO_LD + o + j] = row[j];
      if (tid < 32) sYd[o + lane] = rdiag;     // 1 / L_kk (the inverse's diagonal, used by the panel)
    }
#endif
#ifndef PO_SKIP_TRAIL
    if (warp != 0 && bb > 0) trail(o - 32, kNextDiagTiles, 1 << 20, 1, 7);
#endif
    po_sync();
    const int R = TB - o - 32;                 // rows below the block
    if (R == 0) break;
#ifndef PO_SKIP_PANEL
    // panel L_ib = A_ib L_bb^-T by forward substitution, one row per thread
    // (x_c = (a_c - sum_{l<c} x_l L_cl) / L_cc): no inverse on the critical path
    if (tid < R) {
      double* Ar = sA + (o + 32 + tid) * PO_LD + o;
      double x[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const double* Lc = sA + (o + c) * PO_LD + o;
        double a0 = Ar[c], a1 = 0.0;
#pragma unroll
        for (int l = 0; l < c; ++l) {
          if (l & 1)
            a1 = fma(-x[l], Lc[l], a1);
          else
            a0 = fma(-x[l], Lc[l], a0);
        }
        x[c] = (a0 + a1) * sYd[o + c];
      }
#pragma unroll
      for (int c = 0; c < 32; ++c) Ar[c] = x[c];
    }
    po_sync();
#endif
#ifndef PO_SKIP_TRAIL
    trail(o, 0, kNextDiagTiles, 0, 8);
    po_sync();
#endif
  }
#ifndef PO_SKIP_INV
  po_inverse(sA, sYd, sT);
#endif
  for (int idx = tid; idx < TILE; idx += 256) {
    const int jl = idx >> 7;
    const int il = (idx & 127) ^ ((jl & 3) << 2);
    double lv = 0.0, yv = 0.0;
    if (il >= jl) {
      lv = sA[il * PO_LD + jl];
      yv = yat(il, jl);
    }
    tile[idx] = lv;
    D[idx] = yv;
  }
}

}  // namespace feti
