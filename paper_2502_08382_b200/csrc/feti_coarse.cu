// Coarse-space kernels for a GPU-resident PCPG.
//
// The reference's projector P x = x - G (G^T G)^-1 G^T x (solver.py:117-119)
// uses a dense G of n_mult x (sum of kernel dims).  G = B R is block sparse:
// column block s is nonzero only on subdomain s's multipliers, with
// G_s[a][c] = B~_s[a] * R_s[dof_a][c].  The kernels keep G as one dense m_s x r_s
// block per subdomain (sorted local order, matching the apply's index maps):
//   gtx      v = G^T x            one warp per kernel column, fixed-order tree
//   coarse   z = C v              C = (G^T G)^-1 precomputed on the host
//   project  out = x - G z        one thread per multiplier, contributions in
//                                 the reference's gather order
#include "feti_coarse.h"

namespace feti {

// one 256-thread block per kernel column; fixed strided partials, a shuffle
// tree per warp and the 8 warp sums in warp order: deterministic
__global__ void __launch_bounds__(256) gtx_kernel(const CoarseSub* __restrict__ cs, const int2* __restrict__ cols,
                                                  int ncols, const double* __restrict__ x, double* __restrict__ v) {
  __shared__ double red[8];
  const int2 sc = cols[blockIdx.x];
  const CoarseSub& S = cs[sc.x];
  double acc = 0.0;
  for (int a = threadIdx.x; a < S.m; a += 256) acc = fma(S.G[(int64_t)a * S.r + sc.y], __ldg(x + S.gids[a]), acc);
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += red[i];
    v[S.koff + sc.y] = t;
  }
}

__global__ void __launch_bounds__(256) coarse_kernel(int nk, const double* __restrict__ C,
                                                     const double* __restrict__ v, double* __restrict__ z) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= nk) return;
  double acc = 0.0;
  for (int c = lane; c < nk; c += 32) acc = fma(C[(int64_t)row * nk + c], v[c], acc);
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) z[row] = acc;
}

// out[g] = (x ? x[g] : 0) - sign * sum_{(s,a) in contrib(g)} sum_c G_s[a][c] z[koff_s + c]
__global__ void __launch_bounds__(256) project_kernel(int n_mult, const int* __restrict__ cptr,
                                                      const int4* __restrict__ cent, const CoarseSub* __restrict__ cs,
                                                      const double* __restrict__ z, const double* __restrict__ x,
                                                      double sign, double* __restrict__ out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_mult) return;
  double acc = 0.0;
  for (int e = cptr[g]; e < cptr[g + 1]; ++e) {
    const int4 c = cent[e];
    const CoarseSub& S = cs[c.w];
    const double* Ga = S.G + (int64_t)c.x * S.r;
    double v = 0.0;
    for (int k = 0; k < S.r; ++k) v = fma(Ga[k], z[S.koff + k], v);
    acc += v;
  }
  out[g] = (x ? x[g] : 0.0) - sign * acc;
}

void launch_gtx(const CoarseSub* cs, const int2* cols, int ncols, const double* x, double* v, cudaStream_t st) {
  if (ncols > 0) gtx_kernel<<<ncols, 256, 0, st>>>(cs, cols, ncols, x, v);
}
void launch_coarse(int nk, const double* C, const double* v, double* z, cudaStream_t st) {
  if (nk > 0) coarse_kernel<<<(nk * 32 + 255) / 256, 256, 0, st>>>(nk, C, v, z);
}
void launch_project(int n_mult, const int* cptr, const int4* cent, const CoarseSub* cs, const double* z,
                    const double* x, double sign, double* out, cudaStream_t st) {
  if (n_mult > 0)
    project_kernel<<<(n_mult + 255) / 256, 256, 0, st>>>(n_mult, cptr, cent, cs, z, x, sign, out);
}

}  // namespace feti
