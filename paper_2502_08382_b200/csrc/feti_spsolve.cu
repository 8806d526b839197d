// Device solve_local for the sparse-factor route: x = K_reg^-1 b through the
// block-sparse factor of K_s = K + rho E E^T (CholFactor.solve,
// sparse.py:324-337, with the reference's K_reg = K + rho Q Q^T recovered as
//   K_reg^-1 = Pi K_s^-1 Pi + rho^-1 Q Q^T,  Pi = I - Q Q^T
// (Q orthonormal, the derivation of sp_dual_rhs_kernel).
//
// One CTA per right-hand side; the vectors live in a global scratch (they
// outgrow shared memory at config 5).  After the assembly the pool holds
// three kinds of tiles, each swept in its own form:
//   block rows k < smin          L_kl and the factor's L_kk
//   k >= smin, column l < smin   L_kl
//   k >= smin, column l >= smin  Lhat_kl = inv(L_kk) L_kl, inv(L_kk) on the diagonal
// forward  (L z = v):  k < smin:  z_k = L_kk^-1 (v_k - sum_l L_kl z_l)   (substitution in smem)
//                      k >= smin: z_k = inv(L_kk) (v_k - sum_{l<smin} L_kl z_l) - sum_{l>=smin} Lhat_kl z_l
// backward (L^T y = z), with u_l = L_ll^T y_l kept for l >= smin:
//                      k >= smin: u_k = z_k - sum_{l>k} Lhat_lk^T u_l,  y_k = inv(L_kk)^T u_k
//                      k < smin:  y_k = L_kk^-T (z_k - sum_{l>k} L_lk^T y_l)
// The tile products are split over 4 row-thread groups and summed in a fixed
// order (bit-reproducible).
#include "feti_common.cuh"
#include "feti_sparse.h"

namespace feti {

constexpr int SS_THREADS = 512;
constexpr int SS_GROUPS = SS_THREADS / TB;
constexpr int SS_LD = TB + 1;   // padded row-major diagonal tile in shared memory

// deterministic CTA sum of nv (<= 8) per-thread values; result in out[0..nv)
__device__ __forceinline__ void ss_block_sum(const double* v, int nv, double* red, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (q >= nv) break;
    double s = v[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[warp * 8 + q] = s;
  }
  __syncthreads();
  if (threadIdx.x < nv) {
    double s = 0.0;
    for (int w = 0; w < SS_THREADS / 32; ++w) s += red[w * 8 + threadIdx.x];
    out[threadIdx.x] = s;
  }
  __syncthreads();
}

// load the diagonal tile (col-major swizzled in HBM) as padded row-major
__device__ __forceinline__ void ss_load_diag(const double* __restrict__ t, double* Ls) {
  for (int e = threadIdx.x; e < TILE; e += SS_THREADS) {
    const int j = e >> 7, i = e & (TB - 1);
    Ls[i * SS_LD + j] = __ldcs(t + swz(j, i));
  }
}

__global__ void __launch_bounds__(SS_THREADS, 1)
    sp_solve_kernel(const SubDev* __restrict__ subs, const SpSub* __restrict__ ss, const SpSolveItem* __restrict__ items,
                    const double* __restrict__ b, double* __restrict__ x, double* __restrict__ scratch) {
  extern __shared__ double ssm[];
  double* Ls = ssm;                           // 128 x 129
  double* red = Ls + TB * SS_LD;              // SS_GROUPS x 2 x 128 partials
  double* vec = red + SS_GROUPS * 2 * TB;     // 128: the block row's right-hand side
  double* wred = vec + TB;                    // 16 warps x 8
  double* coef = wred + (SS_THREADS / 32) * 8;   // c = Q^T b (8), d = Q^T x' (8)
  const SpSolveItem it = items[blockIdx.x];
  const SubDev& S = subs[it.sub];
  const SpSub& Q = ss[it.sub];
  const int tid = threadIdx.x, i = tid & (TB - 1), g = tid >> 7;
  const int T = Q.T, smin = S.smin, r = Q.r, n = Q.n;
  const int npos = T * TB;
  const double* bb = b + it.off;
  double* xx = x + it.off;
  double* z = scratch + it.scr;               // v, then z (in place)
  double* y = z + npos;
  double* u = y + npos;
  const double* pool = Q.pool;
  auto tile = [&](int K, int L) -> const double* {
    const int s = Q.tmap[(size_t)K * Q.Tq + L];
    return s < 0 ? nullptr : pool + (size_t)s * TILE;
  };

  // ---- c = Q^T b; v = P (b - Q c)
  double loc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) loc[q] = 0.0;
  for (int d = tid; d < n; d += SS_THREADS) {
    const double bd = bb[d];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < r) loc[q] = fma(Q.Q[(size_t)d * r + q], bd, loc[q]);
  }
  if (r > 0) ss_block_sum(loc, r, wred, coef);
  for (int p = tid; p < npos; p += SS_THREADS) {
    const int64_t d = p < Q.npos ? Q.perm[p] : -1;
    double v = 0.0;
    if (d >= 0) {
      v = bb[d];
      for (int q = 0; q < r; ++q) v = fma(-Q.Q[(size_t)d * r + q], coef[q], v);
    }
    z[p] = v;
  }
  __syncthreads();

  // ---- forward sweep
  for (int k = 0; k < T; ++k) {
    double accU = 0.0, accH = 0.0;
    for (int l = g; l < k; l += SS_GROUPS) {
      const double* t = tile(k, l);
      if (!t) continue;
      const double* zl = z + (size_t)l * TB;
      double s = 0.0, s2 = 0.0;
#pragma unroll 8
      for (int j = 0; j < TB; j += 2) {
        s = fma(__ldcs(t + swz(j, i)), zl[j], s);
        s2 = fma(__ldcs(t + swz(j + 1, i)), zl[j + 1], s2);
      }
      if (k >= smin && l >= smin) accH += s + s2;
      else accU += s + s2;
    }
    const double* td = tile(k, k);
    if (k < smin) ss_load_diag(td, Ls);
    red[(g * 2) * TB + i] = accU;
    red[(g * 2 + 1) * TB + i] = accH;
    __syncthreads();
    double* zk = z + (size_t)k * TB;
    double H = 0.0;
    if (g == 0) {
      double U = 0.0;
#pragma unroll
      for (int g2 = 0; g2 < SS_GROUPS; ++g2) {
        U += red[(g2 * 2) * TB + i];
        H += red[(g2 * 2 + 1) * TB + i];
      }
      vec[i] = zk[i] - U;
    }
    __syncthreads();
    if (k >= smin) {
      // z_k = inv(L_kk) U - H: the 128 columns split over the groups
      double s = 0.0;
#pragma unroll 8
      for (int j = g * (TB / SS_GROUPS); j < (g + 1) * (TB / SS_GROUPS); ++j) s = fma(__ldcs(td + swz(j, i)), vec[j], s);
      red[g * TB + i] = s;
      __syncthreads();
      if (g == 0) {
        double t = 0.0;
#pragma unroll
        for (int g2 = 0; g2 < SS_GROUPS; ++g2) t += red[g2 * TB + i];
        zk[i] = t - H;
      }
    } else if (tid < 32) {
      // L_kk z_k = U by column substitution in one warp (lane owns rows lane + 32 q)
      double tq[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) tq[q] = vec[tid + 32 * q];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        for (int jj = 0; jj < 32; ++jj) {
          const int j = 32 * q + jj;
          double zj = 0.0;
          if (tid == jj) zj = tq[q] / Ls[j * SS_LD + j];
          zj = __shfl_sync(0xffffffffu, zj, jj);
          if (tid == jj) tq[q] = zj;
          if (tid > jj) tq[q] = fma(-Ls[(32 * q + tid) * SS_LD + j], zj, tq[q]);
#pragma unroll
          for (int q2 = q + 1; q2 < 4; ++q2) tq[q2] = fma(-Ls[(32 * q2 + tid) * SS_LD + j], zj, tq[q2]);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) zk[tid + 32 * q] = tq[q];
    }
    __syncthreads();
  }

  // ---- backward sweep
  for (int k = T - 1; k >= 0; --k) {
    double acc = 0.0;
    for (int l = k + 1 + g; l < T; l += SS_GROUPS) {
      const double* t = tile(l, k);
      if (!t) continue;
      const double* col = t + (size_t)i * TB;             // column i of the tile
      const double* w = (k >= smin ? u : y) + (size_t)l * TB;
      double s = 0.0, s2 = 0.0;
      const int sw = (i & 3) << 2;
#pragma unroll 8
      for (int rr = 0; rr < TB; rr += 2) {
        s = fma(__ldcs(col + (rr ^ sw)), w[rr], s);
        s2 = fma(__ldcs(col + ((rr + 1) ^ sw)), w[rr + 1], s2);
      }
      acc += s + s2;
    }
    const double* td = tile(k, k);
    if (k < smin) ss_load_diag(td, Ls);
    red[g * TB + i] = acc;
    __syncthreads();
    if (g == 0) {
      double a = 0.0;
#pragma unroll
      for (int g2 = 0; g2 < SS_GROUPS; ++g2) a += red[g2 * TB + i];
      vec[i] = z[(size_t)k * TB + i] - a;
      if (k >= smin) u[(size_t)k * TB + i] = vec[i];
    }
    __syncthreads();
    double* yk = y + (size_t)k * TB;
    if (k >= smin) {
      // y_k = inv(L_kk)^T u_k
      const double* col = td + (size_t)i * TB;
      const int sw = (i & 3) << 2;
      double s = 0.0;
#pragma unroll 8
      for (int rr = g * (TB / SS_GROUPS); rr < (g + 1) * (TB / SS_GROUPS); ++rr) s = fma(__ldcs(col + (rr ^ sw)), vec[rr], s);
      red[g * TB + i] = s;
      __syncthreads();
      if (g == 0) {
        double t = 0.0;
#pragma unroll
        for (int g2 = 0; g2 < SS_GROUPS; ++g2) t += red[g2 * TB + i];
        yk[i] = t;
      }
    } else if (tid < 32) {
      // L_kk^T y_k = w by backward column substitution (row j of L_kk)
      double tq[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) tq[q] = vec[tid + 32 * q];
#pragma unroll
      for (int q = 3; q >= 0; --q) {
        for (int jj = 31; jj >= 0; --jj) {
          const int j = 32 * q + jj;
          double yj = 0.0;
          if (tid == jj) yj = tq[q] / Ls[j * SS_LD + j];
          yj = __shfl_sync(0xffffffffu, yj, jj);
          if (tid == jj) tq[q] = yj;
          if (tid < jj) tq[q] = fma(-Ls[j * SS_LD + 32 * q + tid], yj, tq[q]);
#pragma unroll
          for (int q2 = 0; q2 < q; ++q2) tq[q2] = fma(-Ls[j * SS_LD + 32 * q2 + tid], yj, tq[q2]);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) yk[tid + 32 * q] = tq[q];
    }
    __syncthreads();
  }

  // ---- x' = P^T y; x = x' - Q (Q^T x') + Q c / rho
  if (r == 0) {
    for (int d = tid; d < n; d += SS_THREADS) xx[d] = y[Q.iperm[d]];
    return;
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) loc[q] = 0.0;
  for (int d = tid; d < n; d += SS_THREADS) {
    const double xd = y[Q.iperm[d]];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < r) loc[q] = fma(Q.Q[(size_t)d * r + q], xd, loc[q]);
  }
  ss_block_sum(loc, r, wred, coef + 8);
  const double irho = 1.0 / *Q.rho;
  for (int d = tid; d < n; d += SS_THREADS) {
    double v = y[Q.iperm[d]];
    for (int q = 0; q < r; ++q) v = fma(Q.Q[(size_t)d * r + q], coef[q] * irho - coef[8 + q], v);
    xx[d] = v;
  }
}

size_t sp_solve_smem() {
  return ((size_t)TB * SS_LD + SS_GROUPS * 2 * TB + TB + (SS_THREADS / 32) * 8 + 16) * sizeof(double);
}

cudaError_t configure_sp_solve() {
  return cudaFuncSetAttribute(sp_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp_solve_smem());
}

void launch_sp_solve(const SubDev* subs, const SpSub* ss, const SpSolveItem* items, int nitems, const double* b,
                     double* x, double* scratch, cudaStream_t st) {
  if (nitems > 0) sp_solve_kernel<<<nitems, SS_THREADS, sp_solve_smem(), st>>>(subs, ss, items, b, x, scratch);
}

}  // namespace feti
