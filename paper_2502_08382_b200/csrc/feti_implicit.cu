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
// One CTA per subdomain streams its trailing tiles twice (HBM-bound).
#include "feti_common.cuh"
#include "feti_implicit.h"

namespace feti {

constexpr int IM_THREADS = 256;

__global__ void __launch_bounds__(IM_THREADS, 1) implicit_apply_kernel(const SubDev* __restrict__ subs,
                                                                       const int64_t* __restrict__ out_off,
                                                                       const double* __restrict__ p,
                                                                       double* __restrict__ out) {
  extern __shared__ double ism[];
  const SubDev S = subs[blockIdx.x];
  const int nb = S.T - S.smin;            // block rows touched
  if (S.m == 0 || nb <= 0) return;
  double* xs = ism;                        // nb*128: b, then x, then u
  double* ys = ism + nb * TB;              // nb*128: y
  double* red = ys + nb * TB;              // 2 * 256 partials
  const int tid = threadIdx.x;
  const int i = tid & (TB - 1), h = tid >> 7;
  const int r0 = S.smin * TB;
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
  __syncthreads();
  // ---- forward sweep
  for (int k = S.smin; k < S.T; ++k) {
    const double* bk = xs + (k - S.smin) * TB;
    double accL = 0.0, accI = 0.0;
    for (int l = S.smin + h; l < k; l += 2) {             // halves split the l tiles
      const double* t = tile_ptr(S, k, l);
      const double* xl = xs + (l - S.smin) * TB;
#pragma unroll 8
      for (int j = 0; j < TB; ++j) accL = fma(__ldcs(t + swz(j, i)), xl[j], accL);
    }
    {
      const double* inv = tile_ptr(S, k, k);
#pragma unroll 8
      for (int j = h * 64; j < h * 64 + 64; ++j) accI = fma(__ldcs(inv + swz(j, i)), bk[j], accI);
    }
    red[tid] = accI - accL;
    __syncthreads();
    if (tid < TB) xs[(k - S.smin) * TB + i] = red[i] + red[TB + i];
    __syncthreads();
  }
  // ---- backward sweep (thread j = i owns column j of the block)
  for (int k = S.T - 1; k >= S.smin; --k) {
    double acc = 0.0;
    for (int l = k + 1 + h; l < S.T; l += 2) {
      const double* t = tile_ptr(S, l, k);
      const double* ul = xs + (l - S.smin) * TB;
      const double* col = t + i * TB;                      // column i of Lhat_lk
#pragma unroll 8
      for (int r = 0; r < TB; ++r) acc = fma(__ldcs(col + (r ^ ((i & 3) << 2))), ul[r], acc);
    }
    red[tid] = acc;
    __syncthreads();
    double* uk = xs + (k - S.smin) * TB;
    if (tid < TB) uk[i] -= red[i] + red[TB + i];
    __syncthreads();
    // y_k = inv(L_kk)^T u_k : column j of inv(L_kk) dotted with u_k, halves over rows
    const double* inv = tile_ptr(S, k, k);
    const double* col = inv + i * TB;
    double y = 0.0;
#pragma unroll 8
    for (int r = h * 64; r < h * 64 + 64; ++r) y = fma(__ldcs(col + (r ^ ((i & 3) << 2))), uk[r], y);
    red[tid] = y;
    __syncthreads();
    if (tid < TB) ys[(k - S.smin) * TB + i] = red[i] + red[TB + i];
    __syncthreads();
  }
  // q_loc[a] = B~_a y[r_a]   (sorted local order)
  double* o = out + out_off[blockIdx.x];
  for (int a = tid; a < S.m; a += IM_THREADS) o[a] = S.s_sorted[a] * ys[S.r_sorted[a] - r0];
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

size_t implicit_smem(int max_blocks) { return ((size_t)2 * max_blocks * TB + 2 * IM_THREADS) * sizeof(double); }

cudaError_t configure_implicit(int max_blocks) {
  return cudaFuncSetAttribute(implicit_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)implicit_smem(max_blocks));
}

void launch_implicit_apply(const SubDev* subs, int nsub, int max_blocks, const int64_t* out_off, const double* p,
                           double* part, int n_mult, const int* cptr, const int4* cent, double* q, cudaStream_t st) {
  if (nsub > 0)
    implicit_apply_kernel<<<nsub, IM_THREADS, implicit_smem(max_blocks), st>>>(subs, out_off, p, part);
  if (n_mult > 0) implicit_reduce_kernel<<<(n_mult + 255) / 256, 256, 0, st>>>(n_mult, cptr, cent, out_off, part, q);
}

}  // namespace feti
