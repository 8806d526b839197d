// 128x128 dense lower-triangular helpers shared by the assembly's diagonal
// inverse and the device factorization (256 threads, shared memory).
#pragma once
#include "feti_common.cuh"

namespace feti {

__device__ __forceinline__ int plo(int i, int j) { return i * (i + 1) / 2 + j; }

// sY (packed lower) = inv(sL) for a 128x128 lower-triangular sL (packed
// lower), blocked 4 x 4 over 32-wide sub-blocks.  Phase 1: warp w inverts
// the diagonal sub-block D_w, lane c carrying column c in registers through a
// lock-step forward substitution (the L row is a shared-memory broadcast).
// Phase 2: off-diagonal sub-blocks by distance d = 1, 2, 3:
//   Y_IJ = -inv(D_I) sum_{K=J}^{I-1} L_IK Y_KJ .
// sT: 3 x 1024 scratch.  Must be called by all 256 threads; ends synchronised.
__device__ __forceinline__ void invert_lower_128(const double* __restrict__ sL, double* __restrict__ sY,
                                                 double* __restrict__ sT) {
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (warp < 4) {
    const int o = warp * 32;
    double y[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const double* Lr = sL + plo(o + r, o);
      double acc = (r == lane) ? 1.0 : 0.0;
#pragma unroll
      for (int j = 0; j < r; ++j) acc = fma(-Lr[j], y[j], acc);
      y[r] = acc / Lr[r];
    }
#pragma unroll
    for (int r = 0; r < 32; ++r)
      if (r >= lane) sY[plo(o + r, o + lane)] = y[r];
  }
  __syncthreads();
  // thread -> (row r, 4 consecutive columns c..c+3) of a 32x32 sub-block
  const int rr = tid >> 3, cc = (tid & 7) * 4;
  for (int d = 1; d < 4; ++d) {
    const int nb = 4 - d;
    for (int bI = 0; bI < nb; ++bI) {          // T_b = sum_{K=J}^{I-1} L_IK Y_KJ
      const int J = bI, I = bI + d;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      const double* Lr = sL + plo(I * 32 + rr, 0);
      for (int kk = J * 32; kk < I * 32; ++kk) {
        const double lv = Lr[kk];
        const double* Yk = sY + plo(kk, 0);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int col = J * 32 + cc + e;
          if (kk >= col) acc[e] = fma(lv, Yk[col], acc[e]);
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) sT[bI * 1024 + rr * 32 + cc + e] = acc[e];
    }
    __syncthreads();
    for (int bI = 0; bI < nb; ++bI) {          // Y_IJ = -inv(D_I) T_b
      const int J = bI, I = bI + d;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      const double* Yr = sY + plo(I * 32 + rr, I * 32);
      for (int kk = 0; kk <= rr; ++kk) {
        const double yv = Yr[kk];
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[e] = fma(yv, sT[bI * 1024 + kk * 32 + cc + e], acc[e]);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) sY[plo(I * 32 + rr, J * 32 + cc + e)] = -acc[e];
    }
    __syncthreads();
  }
}


// In-place Cholesky of the 128x128 tile (col-major swizzled, lower part read)
// and its inverse: tile <- L (upper part zeroed), D <- inv(L) (same layout).
// A non-positive pivot is reported as atomicMin(bad, rowbase + j) and
// replaced by 1 so the sweep completes.  smem: (2 * 8256 + 3 * 1024) doubles.
// Must be called by all 256 threads of the CTA.
__device__ __forceinline__ void potrf_invert_128(double* __restrict__ tile, double* __restrict__ D,
                                                 int* __restrict__ bad, int rowbase, double* __restrict__ smem) {
  double* sL = smem;              // 8256 packed lower
  double* sY = smem + 8256;       // 8256 packed lower
  double* sT = smem + 2 * 8256;   // 3072 scratch
  const int tid = threadIdx.x;
  for (int idx = tid; idx < TILE; idx += 256) {
    const int jl = idx >> 7;
    const int il = (idx & 127) ^ ((jl & 3) << 2);
    if (il >= jl) sL[plo(il, jl)] = tile[idx];
  }
  __syncthreads();
  // blocked right-looking factorization over four 32-wide block columns
  const int lane = tid & 31;
  for (int bb = 0; bb < 4; ++bb) {
    const int o = bb * 32;
    if (tid < 32) {
      // (1) diagonal block, one warp, lane = row
      double lik = 0.0;
      for (int k = 0; k < 32; ++k) {
        __syncwarp();
        double d = sL[plo(o + k, o + k)];
        if (!(d > 0.0)) {
          if (lane == 0) atomicMin(bad, rowbase + o + k);   // first non-positive pivot (permuted row)
          d = 1.0;
        }
        const double pv = sqrt(d);
        __syncwarp();
        if (lane == k) sL[plo(o + k, o + k)] = pv;
        if (lane > k) {
          lik = sL[plo(o + lane, o + k)] / pv;
          sL[plo(o + lane, o + k)] = lik;
        }
        __syncwarp();
        if (lane > k)
          for (int l = k + 1; l <= lane; ++l) sL[plo(o + lane, o + l)] -= lik * sL[plo(o + l, o + k)];
      }
      __syncwarp();
      // (2) inverse of the diagonal block into sY, lane = column
      double y[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const double* Lr = sL + plo(o + r, o);
        double acc = (r == lane) ? 1.0 : 0.0;
#pragma unroll
        for (int j = 0; j < r; ++j) acc = fma(-Lr[j], y[j], acc);
        y[r] = acc / Lr[r];
      }
#pragma unroll
      for (int r = 0; r < 32; ++r)
        if (r >= lane) sY[plo(o + r, o + lane)] = y[r];
    }
    __syncthreads();
    const int R = TB - o - 32;                 // rows below the block
    if (R == 0) break;
    // (3) panel L_ib = A_ib inv(L_bb)^T: item = (row, 4 columns), <= 3 per thread
    double pout[3][4];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int it = tid + u * 256;
      if (it < R * 8) {
        const int i = o + 32 + it / 8, c0 = (it % 8) * 4;
        const double* Ar = sL + plo(i, o);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int c = c0 + e;
          const double* Yc = sY + plo(o + c, o);
          double acc = 0.0;
          for (int l = 0; l <= c; ++l) acc = fma(Ar[l], Yc[l], acc);
          pout[u][e] = acc;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int it = tid + u * 256;
      if (it < R * 8) {
        const int i = o + 32 + it / 8, c0 = (it % 8) * 4;
#pragma unroll
        for (int e = 0; e < 4; ++e) sL[plo(i, o + c0 + e)] = pout[u][e];
      }
    }
    __syncthreads();
    // (4) trailing update A_ij -= sum_c L_ic L_jc over 4x4 register blocks
    const int NB = R / 4;
    const int npairs = NB * (NB + 1) / 2;
    for (int pidx = tid; pidx < npairs; pidx += 256) {
      int I = (int)((sqrt(8.0 * pidx + 1.0) - 1.0) * 0.5);
      while ((I + 1) * (I + 2) / 2 <= pidx) ++I;
      while (I * (I + 1) / 2 > pidx) --I;
      const int J = pidx - I * (I + 1) / 2;
      const int i0 = o + 32 + 4 * I, j0 = o + 32 + 4 * J;
      double acc[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
      for (int c = 0; c < 32; ++c) {
        double av[4], bv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          av[u] = sL[plo(i0 + u, o + c)];
          bv[u] = sL[plo(j0 + u, o + c)];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v)
          if (i0 + u >= j0 + v) sL[plo(i0 + u, j0 + v)] -= acc[u][v];
    }
    __syncthreads();
  }
  for (int idx = tid; idx < TILE; idx += 256) {
    const int jl = idx >> 7;
    const int il = (idx & 127) ^ ((jl & 3) << 2);
    tile[idx] = (il >= jl) ? sL[plo(il, jl)] : 0.0;
  }
  invert_lower_128(sL, sY, sT);
  for (int idx = tid; idx < TILE; idx += 256) {
    const int jl = idx >> 7;
    const int il = (idx & 127) ^ ((jl & 3) << 2);
    D[idx] = (il >= jl) ? sY[plo(il, jl)] : 0.0;
  }
}

}  // namespace feti
