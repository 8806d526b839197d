// Device numeric factorization ("GPU numeric factorization").
//
// The reference factors K_reg = K + rho Q Q^T on the host (chol_numeric,
// _kernels.py:107-140; regularize, sparse.py:427-454) -- 5.5 minutes per c3
// subdomain in its numba loop, 0.6 s with LAPACK -- and the factor (343 MB
// per c3 subdomain) then has to cross PCIe.  Here only the sparse K (CSR),
// the kernel basis Q and the ordering are uploaded; P K_reg P^T is formed in
// the 128x128 tile layout of the assembly and factored in place by a blocked
// right-looking Cholesky on the FP64 tensor pipe:
//   for k:  L_kk = chol(A_kk), inv(L_kk)          (potrf_diag, one CTA/subdomain)
//           L_ik = A_ik inv(L_kk)^T,   i > k       (tile GEMM, DMMA)
//           A_ij -= L_ik L_jk^T,       k < j <= i  (tile GEMM, DMMA)
// The result is plain L in the tiles (diagonal tiles lower-triangular), which
// the assembly then consumes exactly like a scattered host factor.
//
// solve_kernel: x = K_reg^-1 b through the assembled (block-scaled) factor,
// the full-range version of the implicit sweeps (solve_local, sparse.py:324-337).
#include <cooperative_groups.h>

#include "feti_common.cuh"
#include "feti_dense128.cuh"
#include "feti_factor.h"

namespace feti {

// ---------------------------------------------------------------------------
// K_reg tiles: rho Q Q^T (all lower tiles) + scatter of K
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) kreg_fill_kernel(const SubDev* __restrict__ subs,
                                                        const FactorSub* __restrict__ fs, int ntiles_per_sub) {
  const int sub = blockIdx.x / ntiles_per_sub;
  const int t = blockIdx.x % ntiles_per_sub;
  const SubDev& S = subs[sub];
  const FactorSub& F = fs[sub];
  // tile t of the full lower block triangle, row-major over block rows
  int K = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((K + 1) * (K + 2) / 2 <= t) ++K;
  while (K * (K + 1) / 2 > t) --K;
  const int Lc = t - K * (K + 1) / 2;
  double* tile = tile_ptr(S, K, Lc);
  const int n = S.n, r = F.r;
  for (int idx = threadIdx.x; idx < TILE; idx += 256) {
    const int jl = idx >> 7;
    const int il = (idx & 127) ^ ((jl & 3) << 2);
    const int i = K * TB + il, j = Lc * TB + jl;
    double v = 0.0;
    if (i < n && j < n) {
      if (i >= j) {
        const double* qi = F.Q + F.perm[i] * r;
        const double* qj = F.Q + F.perm[j] * r;
        double sq = 0.0;
        for (int c = 0; c < r; ++c) sq = fma(qi[c], qj[c], sq);
        v = F.rho * sq;
      }
    } else if (i == j) {
      v = 1.0;   // identity padding
    }
    tile[idx] = v;
  }
}

// one CTA per original row a: every K entry (a, b) lands once in the lower
// triangle of P K P^T (the symmetric partner maps to the upper one)
__global__ void __launch_bounds__(128) kreg_scatter_kernel(const SubDev* __restrict__ subs,
                                                           const FactorSub* __restrict__ fs, int n) {
  const int sub = blockIdx.x / n;
  const int a = blockIdx.x % n;
  const SubDev& S = subs[sub];
  const FactorSub& F = fs[sub];
  if (a >= S.n) return;   // max_n grid: smaller subdomains skip the tail rows
  const int pa = F.iperm[a];
  for (int64_t p = F.indptr[a] + threadIdx.x; p < F.indptr[a + 1]; p += blockDim.x) {
    const int pb = F.iperm[F.indices[p]];
    if (pa >= pb) {
      double* tile = tile_ptr(S, pa / TB, pb / TB);
      tile[swz(pb % TB, pa % TB)] += F.data[p];
    }
  }
}

// ---------------------------------------------------------------------------
// diagonal block: L_kk = chol(A_kk) in place, inv(L_kk) -> dinv scratch
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 1) potrf_diag_kernel(const SubDev* __restrict__ subs, double* __restrict__ dinv,
                                                         int* __restrict__ bad, int k) {
  extern __shared__ double fsm[];
  const int sub = blockIdx.x;
  potrf_invert_128(tile_ptr(subs[sub], k, k), dinv + (size_t)sub * TILE, bad + sub, k * TB, fsm);
}

// ---------------------------------------------------------------------------
// tile GEMM on the DMMA pipe: acc = A_tile * B_tile^T over the 128-deep k
// A tile (col-major [kk][m]) and B tile (col-major, read as [kk][n]) are
// bulk-copied slice by slice; 8 DMMA warps + 1 producer warp.
//   PANEL : tile(i,k) = tile(i,k) * dinv_k^T     (in place)
//   UPDATE: tile(i,j) -= tile(i,k) * tile(j,k)^T
// ---------------------------------------------------------------------------
constexpr int FG_STAGES = 3;
constexpr int FG_THREADS = 288;

__device__ __forceinline__ void fg_mma_slice(const double* __restrict__ a_s, const double* __restrict__ b_s,
                                             double (&acc)[8][4][2], int wm, int wn, int g, int t) {
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

// Blocked right-looking Cholesky with a look-ahead group of FG_GROUP block
// columns: inside a group the columns are brought up to date left-looking
// (MODE_ACC) and factored one by one (potrf_diag + MODE_PANEL); the rest of
// the matrix then receives one FG_GROUP*128-deep update (MODE_TRAIL), so every
// trailing tile is read-modified-written once per group.
//   MODE_PANEL (sub, i), i in (c, T):      tile(i,c)  = tile(i,c) dinv_c^T
//   MODE_ACC   (sub, i), i in [c, T):      tile(i,c) -= sum_{kc=k0}^{c-1} tile(i,kc) tile(c,kc)^T
//   MODE_TRAIL (sub, i>=j>=j0):            tile(i,j) -= sum_{kc=k0}^{k0+nk-1} tile(i,kc) tile(j,kc)^T
enum { MODE_PANEL = 0, MODE_ACC = 1, MODE_TRAIL = 2 };
constexpr int FG_GROUP = 16;

template <int MODE>
__global__ void __launch_bounds__(FG_THREADS, 1) factor_gemm_kernel(const SubDev* __restrict__ subs,
                                                                    const double* __restrict__ dinv, int c,
                                                                    int k0, int nk, int T) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sA = reinterpret_cast<double*>(smem_raw);
  double* sB = sA + FG_STAGES * SLICE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + FG_STAGES * SLICE);
  uint64_t* empty = full + FG_STAGES;
  int sub, i, j;
  if (MODE == MODE_PANEL) {
    const int M = T - c - 1;
    sub = blockIdx.x / M;
    i = c + 1 + blockIdx.x % M;
    j = c;
  } else if (MODE == MODE_ACC) {
    const int M = T - c;
    sub = blockIdx.x / M;
    i = c + blockIdx.x % M;
    j = c;
  } else {
    const int M = T - c;                     // c = j0
    const int N = M * (M + 1) / 2;
    sub = blockIdx.x / N;
    const int tt = blockIdx.x % N;
    int ii = (int)((sqrt(8.0 * tt + 1.0) - 1.0) * 0.5);
    while ((ii + 1) * (ii + 2) / 2 <= tt) ++ii;
    while (ii * (ii + 1) / 2 > tt) --ii;
    i = c + ii;
    j = c + (tt - ii * (ii + 1) / 2);
  }
  const SubDev& S = subs[sub];
  double* Ct = tile_ptr(S, i, j);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int st = 0; st < FG_STAGES; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 8);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int nsl = (MODE == MODE_PANEL ? 1 : nk) * (TB / KS);
  if (warp == 8) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int sl = 0; sl < nsl; ++sl) {
        const int kc = k0 + sl / (TB / KS);              // contraction column block
        const double* At = (MODE == MODE_PANEL) ? tile_ptr(S, i, c) : tile_ptr(S, i, kc);
        const double* Bt = (MODE == MODE_PANEL) ? dinv + (size_t)sub * TILE : tile_ptr(S, j, kc);
        const int so = (sl % (TB / KS)) * SLICE;
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_arrive_expect_tx(&full[stage], 2 * SLICE * 8);
        bulk_g2s(sA + stage * SLICE, At + so, SLICE * 8, &full[stage]);
        bulk_g2s(sB + stage * SLICE, Bt + so, SLICE * 8, &full[stage]);
        if (++stage == FG_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t = lane & 3;
  double acc[8][4][2];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  int stage = 0;
  uint32_t phase = 0;
  for (int sl = 0; sl < nsl; ++sl) {
    mbar_wait(&full[stage], phase);
    fg_mma_slice(sA + stage * SLICE, sB + stage * SLICE, acc, wm, wn, g, t);
    fence_proxy_async_shared();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == FG_STAGES) {
      stage = 0;
      phase ^= 1;
    }
  }
  // all slices of A were consumed above, so the in-place panel write is safe
#pragma unroll
  for (int mi = 0; mi < 8; ++mi) {
    const int m = wm * 64 + mi * 8 + g;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int nn = wn * 32 + ni * 8 + 2 * t;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double* cp = Ct + swz(nn + e, m);
        if (MODE == MODE_PANEL)
          *cp = acc[mi][ni][e];
        else
          *cp -= acc[mi][ni][e];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// x = K_reg^-1 b for one or more subdomains through the assembled factor
// (Lhat tiles + inv(L_kk) on the diagonal, all block rows): forward and
// backward sweeps as in the implicit apply, dense right-hand side.
// ---------------------------------------------------------------------------
constexpr int SV_THREADS = 512;
constexpr int SV_GROUPS = SV_THREADS / TB;
constexpr int SV_CLUSTER = 2;

__global__ void __cluster_dims__(SV_CLUSTER, 1, 1) __launch_bounds__(SV_THREADS, 1)
    solve_kernel(const SubDev* __restrict__ subs, const FactorSub* __restrict__ fs, const int* __restrict__ slots,
                 const int64_t* __restrict__ vec_off, const double* __restrict__ b, double* __restrict__ x) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ double ssm[];
  const int rank = (int)cluster.block_rank();
  const int slot = slots[blockIdx.x / SV_CLUSTER];
  const SubDev S = subs[slot];
  const FactorSub& F = fs[slot];
  const int T = S.T;
  double* xs = ssm;
  double* ys = ssm + T * TB;
  double* red = ys + T * TB;
  double* red_peer = cluster.map_shared_rank(red, rank ^ 1);
  const int tid = threadIdx.x;
  const int i = tid & (TB - 1), grp = tid >> 7;
  const int lane_id = rank * SV_GROUPS + grp, nlanes = SV_CLUSTER * SV_GROUPS;
  const double* bv = b + vec_off[blockIdx.x / SV_CLUSTER];
  for (int a = tid; a < T * TB; a += SV_THREADS) xs[a] = a < S.n ? bv[F.perm[a]] : 0.0;
  __syncthreads();
  auto combine = [&](double v) -> double {
    red[grp * TB + i] = v;
    cluster.sync();
    double tsum = 0.0;
    for (int rk = 0; rk < SV_CLUSTER; ++rk) {
      const double* src = (rk == rank) ? red : red_peer;
#pragma unroll
      for (int g2 = 0; g2 < SV_GROUPS; ++g2) tsum += src[g2 * TB + i];
    }
    cluster.sync();
    return tsum;
  };
  for (int k = 0; k < T; ++k) {
    double* bk = xs + k * TB;
    double acc = 0.0;
    for (int w = lane_id; w <= k; w += nlanes) {
      if (w < k) {
        const double* tl = tile_ptr(S, k, w);
        const double* xl = xs + w * TB;
#pragma unroll 8
        for (int jj = 0; jj < TB; ++jj) acc = fma(-__ldcs(tl + swz(jj, i)), xl[jj], acc);
      } else {
        const double* inv = tile_ptr(S, k, k);
#pragma unroll 8
        for (int jj = 0; jj < TB; ++jj) acc = fma(__ldcs(inv + swz(jj, i)), bk[jj], acc);
      }
    }
    const double xk = combine(acc);
    if (grp == 0) bk[i] = xk;
    __syncthreads();
  }
  for (int k = T - 1; k >= 0; --k) {
    double acc = 0.0;
    for (int w = lane_id; w < T - 1 - k; w += nlanes) {
      const int l = k + 1 + w;
      const double* col = tile_ptr(S, l, k) + i * TB;
      const double* ul = xs + l * TB;
#pragma unroll 8
      for (int r = 0; r < TB; ++r) acc = fma(__ldcs(col + (r ^ ((i & 3) << 2))), ul[r], acc);
    }
    double* uk = xs + k * TB;
    const double uk_i = uk[i] - combine(acc);
    __syncthreads();
    if (grp == 0) uk[i] = uk_i;
    __syncthreads();
    const double* col = tile_ptr(S, k, k) + i * TB;
    double y = 0.0;
    const int rb = lane_id * (TB / nlanes);
#pragma unroll 4
    for (int r = rb; r < rb + TB / nlanes; ++r) y = fma(__ldcs(col + (r ^ ((i & 3) << 2))), uk[r], y);
    const double yk = combine(y);
    if (grp == 0) ys[k * TB + i] = yk;
  }
  __syncthreads();
  if (rank == 0) {
    double* xv = x + vec_off[blockIdx.x / SV_CLUSTER];
    for (int a = tid; a < S.n; a += SV_THREADS) xv[F.perm[a]] = ys[a];
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static size_t fg_smem() { return 2 * FG_STAGES * SLICE * sizeof(double) + 8 * 2 * FG_STAGES; }
static size_t potrf_smem() { return POTRF_SMEM_DOUBLES * sizeof(double); }
size_t solve_smem(int T) { return ((size_t)2 * T * TB + SV_GROUPS * TB) * sizeof(double); }

cudaError_t configure_factor(int max_T) {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(factor_gemm_kernel<MODE_PANEL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)fg_smem())))
    return e;
  if ((e = cudaFuncSetAttribute(factor_gemm_kernel<MODE_ACC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)fg_smem())))
    return e;
  if ((e = cudaFuncSetAttribute(factor_gemm_kernel<MODE_TRAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)fg_smem())))
    return e;
  if ((e = cudaFuncSetAttribute(potrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)potrf_smem())))
    return e;
  if (solve_smem(max_T) <= 227 * 1024)
    if ((e = cudaFuncSetAttribute(solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)solve_smem(max_T))))
      return e;
  return cudaSuccess;
}

void launch_kreg_build(const SubDev* subs, const FactorSub* fs, int nsub, int T, int n, cudaStream_t st) {
  const int nt = T * (T + 1) / 2;
  kreg_fill_kernel<<<nsub * nt, 256, 0, st>>>(subs, fs, nt);
  kreg_scatter_kernel<<<nsub * n, 128, 0, st>>>(subs, fs, n);
}

// One look-ahead group starting at block column k0 (FG_GROUP columns):
// returns the next group's first column.
int launch_factor_step(const SubDev* subs, double* dinv, int* bad, int nsub, int k0, int T, cudaStream_t st) {
  const int k1 = k0 + FG_GROUP < T ? k0 + FG_GROUP : T;
  for (int c = k0; c < k1; ++c) {
    if (c > k0)
      factor_gemm_kernel<MODE_ACC><<<nsub * (T - c), FG_THREADS, fg_smem(), st>>>(subs, dinv, c, k0, c - k0, T);
    potrf_diag_kernel<<<nsub, 256, potrf_smem(), st>>>(subs, dinv, bad, c);
    if (T - c - 1 > 0)
      factor_gemm_kernel<MODE_PANEL><<<nsub * (T - c - 1), FG_THREADS, fg_smem(), st>>>(subs, dinv, c, c, 1, T);
  }
  if (k1 < T) {
    const int M = T - k1;
    factor_gemm_kernel<MODE_TRAIL><<<nsub * (M * (M + 1) / 2), FG_THREADS, fg_smem(), st>>>(subs, dinv, k1, k0,
                                                                                             k1 - k0, T);
  }
  return k1;
}

void launch_solve(const SubDev* subs, const FactorSub* fs, const int* slots, int nslots, int max_T,
                  const int64_t* vec_off, const double* b, double* x, cudaStream_t st) {
  if (nslots > 0)
    solve_kernel<<<nslots * SV_CLUSTER, SV_THREADS, solve_smem(max_T), st>>>(subs, fs, slots, vec_off, b, x);
}

}  // namespace feti
