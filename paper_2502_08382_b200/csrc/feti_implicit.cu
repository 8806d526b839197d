// Implicit GPU apply: q = sum_i B~_i^T (L^-T (L^-1 (B~_i p))).
//
// The reference's implicit strategy (apply_implicit_local, dualop.py:504-521)
// runs two sparse triangular solves per subdomain per iteration.  Here the
// solves reuse what the explicit assembly already left in HBM: the block-row
// scaled factor Lhat_kl = inv(L_kk) L_kl and inv(L_kk) in the diagonal tiles.
//   forward   x_k = inv(L_kk) b_k - sum_{l<k} Lhat_kl x_l
//   backward  u_k = x_k - sum_{l>k} Lhat_lk^T u_l ,  y_k = inv(L_kk)^T u_k
// (L^T y = x with u_l = L_ll^T y_l.)  b = P B~^T p is nonzero only from the
// smallest first row on, and q needs y only at the constrained rows, so both
// sweeps run over block rows [smin, T) only -- the tiles the assembly keeps.
// A 2-CTA cluster per subdomain streams its trailing tiles twice (HBM-bound).
//
// Sparse-factor route (K_s = K + rho E E^T factored on the device, see
// feti_sparse.cu): the same sweeps give F_s p; the rank-2r correction
//   F~ p = F_s p + U1 (W^T p) - U2 (U1^T p),  W = U1 C - U2 (C = y^T y + I/rho)
// is added to each subdomain's partial from two r-vectors of dots (W^T p =
// C U1^T p - U2^T p).  U2 = B~ K_s^-1 Q is solved once per assembly by the
// backward sweep alone, started from y = L^-1 P Q (the appended block row),
// one column per launch row (MODE_U2; the device dual rhs's f' column too).
#include <cooperative_groups.h>

#include "feti_common.cuh"
#include "feti_implicit.h"
#include "feti_sparse.h"

namespace feti {

constexpr int IM_THREADS = 512;
constexpr int IM_GROUPS = IM_THREADS / TB;   // row-thread groups splitting the tile loops
constexpr int IM_CLUSTER = 2;                // CTAs per subdomain (DSMEM exchange)

// One cluster of IM_CLUSTER CTAs per subdomain: the tiles of every block row
// are dealt round-robin over the CTA-groups (rank, group); each step's
// partial sums are exchanged through distributed shared memory so that every
// CTA holds the full x/u/y vectors.
enum { MODE_APPLY = 0, MODE_U2 = 1 };
constexpr int IM_MAXR = 8;

template <int MODE>
__global__ void __cluster_dims__(IM_CLUSTER, 1, 1) __launch_bounds__(IM_THREADS, 1)
    implicit_apply_kernel(const SubDev* __restrict__ subs, const SpSub* __restrict__ ss, int sub0,
                          const int64_t* __restrict__ out_off, const double* __restrict__ p,
                          double* __restrict__ out) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ double ism[];
  const int rank = (int)cluster.block_rank();
  const int sub = sub0 + blockIdx.x / IM_CLUSTER;
  const SubDev S = subs[sub];
  const int nb = S.T - S.smin;             // block rows touched
  double* xs = ism;                        // nb*128: b, then x, then u
  double* ys = ism + nb * TB;              // nb*128: y
  double* red = ys + nb * TB;              // IM_GROUPS * 128 partials of this CTA
  double* red_peer = cluster.map_shared_rank(red, rank ^ 1);
  const int tid = threadIdx.x;
  const int i = tid & (TB - 1), grp = tid >> 7;
  const int lane_id = rank * IM_GROUPS + grp, nlanes = IM_CLUSTER * IM_GROUPS;
  const int r0 = S.smin * TB;
  // MODE_U2: launch row q solves column q of y (Q columns, then the f' row)
  const int qcol = blockIdx.y;
  int nr = 0;
  if (MODE == MODE_U2) nr = ss[sub].frow >= 0 ? ss[sub].frow + 1 : ss[sub].r;
  const bool active = S.m > 0 && nb > 0 && (MODE == MODE_APPLY || qcol < nr);   // uniform over the cluster
  if (active && MODE == MODE_U2) {
    // x = y[:, q] over block rows [smin, T): row q of the (P Q)^T block-row tiles
    const SpSub& Q = ss[sub];
    for (int a = tid; a < nb * TB; a += IM_THREADS) {
      const int kb = S.smin + a / TB, il = a % TB;
      const int slot = Q.tmap[(size_t)Q.T * Q.Tq + kb];
      xs[a] = slot >= 0 ? Q.pool[(size_t)slot * TILE + swz(il, qcol)] : 0.0;
    }
  }
  if (active && MODE == MODE_APPLY) {
    for (int a = tid; a < nb * TB; a += IM_THREADS) xs[a] = 0.0;
    __syncthreads();
    // b = P B~^T p: columns are sorted by first row, runs of equal rows summed
    // in column order by the run's first thread (deterministic)
    for (int a = tid; a < S.m; a += IM_THREADS) {
      const int r = S.r_sorted[a];
      if (a > 0 && S.r_sorted[a - 1] == r) continue;
      double s = 0.0;
      for (int b = a; b < S.m && S.r_sorted[b] == r; ++b) s += S.s_sorted[b] * __ldg(p + S.gids_sorted[b]);
      xs[r - r0] = s;
    }
  }
  __syncthreads();
  auto combine = [&](double v) -> double {
    // sum of all (rank, group) partials of row/column i in a fixed order
    red[grp * TB + i] = v;
    cluster.sync();
    double t = 0.0;
    for (int rk = 0; rk < IM_CLUSTER; ++rk) {
      const double* src = (rk == rank) ? red : red_peer;
#pragma unroll
      for (int g2 = 0; g2 < IM_GROUPS; ++g2) t += src[g2 * TB + i];
    }
    cluster.sync();
    return t;
  };
  if (active) {
    // ---- forward sweep: x_k = inv(L_kk) b_k - sum_{l<k} Lhat_kl x_l
    for (int k = S.smin; k < S.T && MODE == MODE_APPLY; ++k) {
      double* bk = xs + (k - S.smin) * TB;
      double acc = 0.0;
      // work items: the k - smin off-diagonal tiles plus the diagonal (inverse) tile
      for (int w = lane_id; w <= k - S.smin; w += nlanes) {
        const int l = S.smin + w;
        if (l < k) {
          const double* t = tile_ptr(S, k, l);
          const double* xl = xs + (l - S.smin) * TB;
          double a2 = 0.0;
#pragma unroll 16
          for (int j = 0; j < TB; j += 2) {
            acc = fma(-__ldcs(t + swz(j, i)), xl[j], acc);
            a2 = fma(-__ldcs(t + swz(j + 1, i)), xl[j + 1], a2);
          }
          acc += a2;
        } else {
          const double* inv = tile_ptr(S, k, k);
#pragma unroll 8
          for (int j = 0; j < TB; ++j) acc = fma(__ldcs(inv + swz(j, i)), bk[j], acc);
        }
      }
      const double xk = combine(acc);
      if (grp == 0) bk[i] = xk;
      __syncthreads();
    }
    // ---- backward sweep: u_k = x_k - sum_{l>k} Lhat_lk^T u_l ; y_k = inv(L_kk)^T u_k
    for (int k = S.T - 1; k >= S.smin; --k) {
      double acc = 0.0;
      for (int w = lane_id; w < S.T - 1 - k; w += nlanes) {
        const int l = k + 1 + w;
        const double* col = tile_ptr(S, l, k) + i * TB;     // column i of Lhat_lk
        const double* ul = xs + (l - S.smin) * TB;
        double a2 = 0.0;
#pragma unroll 16
        for (int r = 0; r < TB; r += 2) {
          acc = fma(__ldcs(col + (r ^ ((i & 3) << 2))), ul[r], acc);
          a2 = fma(__ldcs(col + ((r + 1) ^ ((i & 3) << 2))), ul[r + 1], a2);
        }
        acc += a2;
      }
      double* uk = xs + (k - S.smin) * TB;
      const double uk_i = uk[i] - combine(acc);
      __syncthreads();
      if (grp == 0) uk[i] = uk_i;
      __syncthreads();
      const double* col = tile_ptr(S, k, k) + i * TB;       // column i of inv(L_kk)
      double y = 0.0;
      const int rb = lane_id * (TB / nlanes);
#pragma unroll 4
      for (int r = rb; r < rb + TB / nlanes; ++r) y = fma(__ldcs(col + (r ^ ((i & 3) << 2))), uk[r], y);
      const double yk = combine(y);
      if (grp == 0) ys[(k - S.smin) * TB + i] = yk;
    }
    __syncthreads();
    if (MODE == MODE_U2) {
      // U2[a][q] = B~_a (K_s^-1 Q)[:, q] (or U2f[a] for the f' column)
      const SpSub& Q = ss[sub];
      if (rank == 0)
        for (int a = tid; a < S.m; a += IM_THREADS) {
          const double v = S.s_sorted[a] * ys[S.r_sorted[a] - r0];
          if (qcol < Q.r) Q.U2W[(size_t)a * 2 * Q.r + qcol] = v;
          else Q.U2f[a] = v;
        }
      return;
    }
    // q_loc[a] = B~_a y[r_a] (sorted local order), written by cluster rank 0
    if (rank == 0) {
      double* o = out + out_off[sub];
      const int r = ss ? ss[sub].r : 0;
      if (r == 0) {
        for (int a = tid; a < S.m; a += IM_THREADS) o[a] = S.s_sorted[a] * ys[S.r_sorted[a] - r0];
      } else {
        // sparse route: + U1 (C al - be) - U2 al with al = U1^T p, be = U2^T p
        // (fixed-order reductions: per-thread strided sums, warp tree, warps in order)
        const SpSub& Q = ss[sub];
        double d[2 * IM_MAXR];
#pragma unroll
        for (int q = 0; q < 2 * IM_MAXR; ++q) d[q] = 0.0;
        for (int a = tid; a < S.m; a += IM_THREADS) {
          const double pa = __ldg(p + S.gids_sorted[a]);
#pragma unroll
          for (int q = 0; q < IM_MAXR; ++q)
            if (q < r) {
              d[q] = fma(Q.U1[(size_t)a * r + q], pa, d[q]);
              d[IM_MAXR + q] = fma(Q.U2W[(size_t)a * 2 * r + q], pa, d[IM_MAXR + q]);
            }
        }
        const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
        for (int q = 0; q < 2 * IM_MAXR; ++q) {
          double v = d[q];
#pragma unroll
          for (int o2 = 16; o2 > 0; o2 >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o2);
          if (lane == 0) red[warp * 2 * IM_MAXR + q] = v;
        }
        __syncthreads();
        double* g = red + (IM_THREADS / 32) * 2 * IM_MAXR;   // al[0..r), ga[0..r)
        if (tid < 2 * IM_MAXR) {
          double v = 0.0;
          for (int w = 0; w < IM_THREADS / 32; ++w) v += red[w * 2 * IM_MAXR + tid];
          g[tid] = v;
        }
        __syncthreads();
        if (tid < r) {
          // ga = C al - be,  C[q][q2] = -tile(T,T)[q][q2] + [q == q2] / rho
          const double* cq = Q.pool + (size_t)Q.tmap[(size_t)Q.T * Q.Tq + Q.T] * TILE;
          double v = -g[IM_MAXR + tid];
          for (int q2 = 0; q2 < r; ++q2)
            v = fma(-cq[swz(q2, tid)] + (tid == q2 ? 1.0 / *Q.rho : 0.0), g[q2], v);
          g[2 * IM_MAXR + tid] = v;
        }
        __syncthreads();
        for (int a = tid; a < S.m; a += IM_THREADS) {
          double v = S.s_sorted[a] * ys[S.r_sorted[a] - r0];
          for (int q = 0; q < r; ++q) {
            v = fma(Q.U1[(size_t)a * r + q], g[2 * IM_MAXR + q], v);
            v = fma(-Q.U2W[(size_t)a * 2 * r + q], g[q], v);
          }
          o[a] = v;
        }
      }
    }
  }
}

// q[g] = sum over (slot, local) contributions in the reference's gather order
__global__ void __launch_bounds__(256) implicit_reduce_kernel(int n_mult, const int* __restrict__ cptr,
                                                              const int4* __restrict__ cent,
                                                              const int64_t* __restrict__ out_off,
                                                              const double* __restrict__ part,
                                                              double* __restrict__ q) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_mult) return;
  double acc = 0.0;
  for (int e = cptr[g]; e < cptr[g + 1]; ++e) {
    const int4 c = cent[e];
    acc += part[out_off[c.w] + c.x];
  }
  q[g] = acc;
}

size_t implicit_smem(int max_blocks) { return ((size_t)2 * max_blocks * TB + IM_GROUPS * TB) * sizeof(double); }
static_assert((IM_THREADS / 32 + 2) * 2 * IM_MAXR <= IM_GROUPS * TB, "correction scratch fits the partials buffer");

cudaError_t configure_implicit(int max_blocks) {
  cudaError_t e = cudaFuncSetAttribute(implicit_apply_kernel<MODE_APPLY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)implicit_smem(max_blocks));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(implicit_apply_kernel<MODE_U2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)implicit_smem(max_blocks));
}

void launch_implicit_apply(const SubDev* subs, const SpSub* ss, int nsub, int max_blocks, const int64_t* out_off,
                           const double* p, double* part, int n_mult, const int* cptr, const int4* cent, double* q,
                           cudaStream_t st) {
  if (nsub > 0)
    implicit_apply_kernel<MODE_APPLY>
        <<<nsub * IM_CLUSTER, IM_THREADS, implicit_smem(max_blocks), st>>>(subs, ss, 0, out_off, p, part);
  if (n_mult > 0) implicit_reduce_kernel<<<(n_mult + 255) / 256, 256, 0, st>>>(n_mult, cptr, cent, out_off, part, q);
}

void launch_implicit_u2(const SubDev* subs, const SpSub* ss, int sub0, int nsub, int max_cols, int max_blocks,
                        cudaStream_t st) {
  if (nsub > 0 && max_cols > 0)
    implicit_apply_kernel<MODE_U2><<<dim3(nsub * IM_CLUSTER, max_cols), IM_THREADS, implicit_smem(max_blocks), st>>>(
        subs, ss, sub0, nullptr, nullptr, nullptr);
}

}  // namespace feti
