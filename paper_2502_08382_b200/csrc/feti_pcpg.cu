// Device-native PCPG: the reference's projected CG
// (solver.py:195-272) with every vector operation, inner product and the
// stopping test on the device.
//
// One iteration (precond "none") is two launches -- the apply and one
// cooperative kernel doing B, D, F and G below between grid-wide barriers
// (pcpg_iter_coop; FETI_PCPG_COOP=0 falls back to five separate launches) --
// captured in a CUDA graph of several iterations and replayed; the host polls
// a status word once per graph launch.  The phases:
//   A  apply_kernel      SYMV partials of F p_new, gathering p_new = y + beta p
//                        on the fly (the conjugation of the previous iteration)
//   B  reduce_pq         q = F p_new in the reference's gather order, p <- p_new,
//                        p.q; the last block: delta = wy / pq, breakdown test
//   D  gtx_r             G^T (r - delta q) per kernel column; the last block:
//                        kz = (G^T G)^-1 G^T r
//   F  gtx_w             G^T w with w = (r - delta q) - G kz formed on the fly;
//                        the last block: kz2
//   G  update            r, lam, w = P r, y = P w; w.y, w.w; the last block:
//                        k, stopping test, beta, wy
// ("lumped": G1 writes w, the preconditioner apply gives z = M w, then G^T z
// and G2 forms y = z - G kz2 and finalises.)  Reductions are fixed-order
// trees, and the cross-block sums are done by the last block to finish (a
// counter) in block order: bit-reproducible runs.
#include <cooperative_groups.h>

#include <cstdint>

#include "feti_coarse.h"
#include "feti_common.cuh"
#include "feti_apply.cuh"
#include "feti_kernels.h"
#include "feti_pcpg.h"

namespace feti {

constexpr int PT = 256;   // threads per block of the vector kernels

__device__ __forceinline__ double block_sum(double v, double* red) {
  // fixed-order tree over the block: warp shuffles, then the warp sums in order
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < PT / 32; ++i) t += red[i];
  return t;   // valid in thread 0
}

// the last block to arrive (counter) returns true; counters reset themselves
__device__ __forceinline__ bool last_block(unsigned* cnt) {
  __shared__ bool is_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned t = atomicAdd(cnt, 1u);
    is_last = (t == gridDim.x - 1);
    if (is_last) *cnt = 0u;
  }
  __syncthreads();
  return is_last;
}

// sum of n partials in index order by one block (deterministic)
__device__ __forceinline__ double ordered_sum(const double* v, int n, int stride, double* red) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += PT) acc += __ldcg(v + (size_t)i * stride);
  return block_sum(acc, red);
}

// G_s rows of multiplier g times a coarse vector z, in the gather order
__device__ __forceinline__ double gz(const PcpgDev& P, int g, const double* z) {
  double acc = 0.0;
  for (int e = P.cptr[g]; e < P.cptr[g + 1]; ++e) {
    const int4 c = P.cent[e];
    const CoarseSub& S = P.cs[c.w];
    const double* Ga = S.G + (int64_t)c.x * S.r;
    double v = 0.0;
    for (int k = 0; k < S.r; ++k) v = fma(Ga[k], __ldcg(z + S.koff + k), v);
    acc += v;
  }
  return acc;
}

// z = C v by the block (warp per row), C = (G^T G)^-1
__device__ __forceinline__ void coarse_block(const PcpgDev& P, const double* v, double* z) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int row = warp; row < P.nk; row += PT / 32) {
    double acc = 0.0;
    for (int c = lane; c < P.nk; c += 32) acc = fma(P.cinv[(int64_t)row * P.nk + c], __ldcg(v + c), acc);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) z[row] = acc;
  }
}

__device__ __forceinline__ double r_new(const PcpgDev& P, int g, double delta) {
  return __ldcg(P.r + g) - delta * __ldcg(P.q + g);   // r - delta qk (solver.py:250)
}

// B: q = reduce(partials), p <- y + beta p, p.q ; last block: delta
__global__ void __launch_bounds__(PT) pcpg_reduce_pq(PcpgDev P) {
  __shared__ double red[PT / 32];
  PcpgScal* sc = P.sc;
  if (sc->done) return;
  const int g = blockIdx.x * PT + threadIdx.x;
  double v = 0.0;
  if (g < P.n_mult) {
    double qg = 0.0;
    for (int e = P.cptr[g]; e < P.cptr[g + 1]; ++e) {
      const int4 c = P.cent[e];
      double s = 0.0;
      for (int k = c.y; k < c.z; ++k) s += P.part[P.ridx[k]];
      qg += s;
    }
    const double pn = fma(sc->beta, P.p[g], P.y[g]);
    P.q[g] = qg;
    P.p[g] = pn;
    v = pn * qg;
  }
  const double t = block_sum(v, red);
  if (threadIdx.x == 0) P.bpart[blockIdx.x] = t;
  if (!last_block(&sc->cnt[0])) return;
  const double pq = ordered_sum(P.bpart, gridDim.x, 1, red);
  if (threadIdx.x == 0) {
    sc->pq = pq;
    if (!(pq > 0.0)) {   // p^T F p <= 0: BreakdownError (solver.py:246-247)
      sc->status = PCPG_BREAKDOWN;
      sc->done = 1;
    } else {
      sc->delta = sc->wy / pq;
    }
  }
}

// D: kv = G^T (r - delta q), one block per kernel column; last block: kz
__global__ void __launch_bounds__(PT) pcpg_gtx_r(PcpgDev P) {
  __shared__ double red[PT / 32];
  PcpgScal* sc = P.sc;
  if (sc->done) return;
  const int2 col = P.kcols[blockIdx.x];
  const CoarseSub& S = P.cs[col.x];
  const double delta = sc->delta;
  double acc = 0.0;
  for (int a = threadIdx.x; a < S.m; a += PT) acc = fma(S.G[(int64_t)a * S.r + col.y], r_new(P, S.gids[a], delta), acc);
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) P.kv[S.koff + col.y] = t;
  if (!last_block(&sc->cnt[1])) return;
  coarse_block(P, P.kv, P.kz);
}

// F: kv2 = G^T w, w = (r - delta q) - G kz on the fly; last block: kz2
__global__ void __launch_bounds__(PT) pcpg_gtx_w(PcpgDev P) {
  __shared__ double red[PT / 32];
  PcpgScal* sc = P.sc;
  if (sc->done) return;
  const int2 col = P.kcols[blockIdx.x];
  const CoarseSub& S = P.cs[col.x];
  const double delta = sc->delta;
  double acc = 0.0;
  for (int a = threadIdx.x; a < S.m; a += PT) {
    const int g = S.gids[a];
    const double wg = r_new(P, g, delta) - gz(P, g, P.kz);
    acc = fma(S.G[(int64_t)a * S.r + col.y], wg, acc);
  }
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) P.kv2[S.koff + col.y] = t;
  if (!last_block(&sc->cnt[2])) return;
  coarse_block(P, P.kv2, P.kz2);
}

// G^T x for a materialised x (lumped path); last block: kz2
__global__ void __launch_bounds__(PT) pcpg_gtx_x(PcpgDev P, const double* __restrict__ x) {
  __shared__ double red[PT / 32];
  PcpgScal* sc = P.sc;
  if (sc->done) return;
  const int2 col = P.kcols[blockIdx.x];
  const CoarseSub& S = P.cs[col.x];
  double acc = 0.0;
  for (int a = threadIdx.x; a < S.m; a += PT) acc = fma(S.G[(int64_t)a * S.r + col.y], __ldcg(x + S.gids[a]), acc);
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) P.kv2[S.koff + col.y] = t;
  if (!last_block(&sc->cnt[2])) return;
  coarse_block(P, P.kv2, P.kz2);
}

__device__ __forceinline__ void finalize(const PcpgDev& P, double wy_next, double ww) {
  PcpgScal* sc = P.sc;
  const double wn = sqrt(ww);
  sc->k += 1;
  sc->wn = wn;
  if (wn <= sc->tolw0) {                    // solver.py:258-262
    sc->status = PCPG_CONVERGED;
    sc->done = 1;
  } else if (sc->k >= sc->maxit) {          // solver.py:263-267
    sc->status = PCPG_MAXIT;
    sc->done = 1;
  } else {
    sc->beta = wy_next / sc->wy;            // solver.py:268-271
    sc->wy = wy_next;
  }
}

// G (mode 0, "none"): r, lam, w = P r, y = P w, partials of w.y and w.w;
// G1 (mode 1, lumped): r, lam, w written, partial w.w;
// G2 (mode 2, lumped): y = z - G kz2, partial w.y; finalises with G1's w.w
template <int MODE>
__global__ void __launch_bounds__(PT) pcpg_update(PcpgDev P) {
  __shared__ double red[PT / 32];
  PcpgScal* sc = P.sc;
  if (sc->done) return;
  const int g = blockIdx.x * PT + threadIdx.x;
  const double delta = sc->delta;
  double wy = 0.0, ww = 0.0;
  if (g < P.n_mult) {
    if (MODE == 2) {
      const double wg = P.w[g];
      const double yg = P.z[g] - gz(P, g, P.kz2);
      P.y[g] = yg;
      wy = wg * yg;
    } else {
      const double rn = r_new(P, g, delta);
      P.lam[g] = P.lam[g] + delta * P.p[g];   // lam + delta p (solver.py:249)
      const double wg = rn - gz(P, g, P.kz);
      P.r[g] = rn;
      ww = wg * wg;
      if (MODE == 0) {
        const double yg = wg - gz(P, g, P.kz2);
        P.y[g] = yg;
        wy = wg * yg;
      } else {
        P.w[g] = wg;
      }
    }
  }
  const double t_wy = block_sum(wy, red);
  const double t_ww = block_sum(ww, red);
  if (threadIdx.x == 0) {
    P.bpart[2 * blockIdx.x] = t_wy;
    P.bpart[2 * blockIdx.x + 1] = t_ww;
  }
  if (!last_block(&sc->cnt[3])) return;
  const double s_wy = ordered_sum(P.bpart, gridDim.x, 2, red);
  const double s_ww = ordered_sum(P.bpart + 1, gridDim.x, 2, red);
  if (threadIdx.x != 0) return;
  if (MODE == 1) {
    sc->ww = s_ww;
  } else if (MODE == 2) {
    finalize(P, s_wy, sc->ww);
  } else {
    finalize(P, s_wy, s_ww);
  }
}

// ---- the iteration's vector work as ONE cooperative kernel (precond none) --
// grid = one CTA per SM (co-resident), grid-wide barriers between the phases
// of kernels B, D, F and G above; every cross-CTA sum is read back by the CTAs
// that need it in CTA order (deterministic, identical everywhere), so the
// scalar results need no broadcast barrier.
__device__ __forceinline__ double cta_ordered(const double* v, int n, int stride, double* red) {
  const double t = ordered_sum(v, n, stride, red);
  __shared__ double bc;
  if (threadIdx.x == 0) bc = t;
  __syncthreads();
  const double r = bc;
  __syncthreads();
  return r;
}

// piece sums of G^T x (warp per piece, lanes strided over its entries);
// with `qx`, x = r - delta q is formed on the fly (two independent gathers)
__device__ __forceinline__ void gtx_pieces(const PcpgDev& P, const double* x, const double* qx, double delta) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int pc = blockIdx.x * (PT / 32) + warp; pc < P.npieces; pc += gridDim.x * (PT / 32)) {
    const int4 pi = P.pieces[pc];
    double acc = 0.0;
#pragma unroll 4
    for (int e = pi.y + lane; e < pi.z; e += 32) {
      const int g = P.gidx[e];
      const double xv = qx ? __ldcg(x + g) - delta * __ldcg(qx + g) : __ldcg(x + g);
      acc = fma(P.gval[e], xv, acc);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) P.ppart[pc] = acc;
  }
}

// z = C (G^T x) from the piece sums: z[row] = sum_pieces C[row][col(p)] part[p]
// (a row per warp; the pieces of a column are summed in order within the
// warp's fixed lane/tree order: deterministic)
__device__ __forceinline__ void coarse_pieces(const PcpgDev& P, double* z) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int row = blockIdx.x * (PT / 32) + warp; row < P.nk; row += gridDim.x * (PT / 32)) {
    const double* crow = P.cinv + (int64_t)row * P.nk;
    double acc = 0.0;
    for (int pc = lane; pc < P.npieces; pc += 32) acc = fma(crow[P.pieces[pc].x], __ldcg(P.ppart + pc), acc);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) z[row] = acc;
  }
}

// the iteration's vector work after the apply's partials are complete
__device__ __forceinline__ void pcpg_vector_phases(const PcpgDev& P, cooperative_groups::grid_group& grid) {
  __shared__ double red[PT / 32];
  PcpgScal* sc = P.sc;
  const int G = gridDim.x, b = blockIdx.x;
  const int nthr = G * PT, gt = b * PT + threadIdx.x;
  // q = reduce(partials), p <- y + beta p, p.q
  const double beta = sc->beta;
  double v = 0.0;
  for (int g = gt; g < P.n_mult; g += nthr) {
    double qg = 0.0;
    for (int e = P.cptr[g]; e < P.cptr[g + 1]; ++e) {
      const int4 c = P.cent[e];
      double s2 = 0.0;
      for (int k = c.y; k < c.z; ++k) s2 += P.part[P.ridx[k]];
      qg += s2;
    }
    const double pn = fma(beta, P.p[g], P.y[g]);
    P.q[g] = qg;
    P.p[g] = pn;
    v += pn * qg;
  }
  double t = block_sum(v, red);
  if (threadIdx.x == 0) P.bpart[b] = t;
  grid.sync();
  const double pq = cta_ordered(P.bpart, G, 1, red);
  if (!(pq > 0.0)) {                          // BreakdownError (solver.py:246-247)
    if (b == 0 && threadIdx.x == 0) {
      sc->pq = pq;
      sc->status = PCPG_BREAKDOWN;
      sc->done = 1;
    }
    return;                                   // every CTA saw the same pq
  }
  const double delta = sc->wy / pq;
  // kz = (G^T G)^-1 G^T (r - delta q): piece sums, then the coarse rows
  // spread over the grid (the last CTA doing all rows measured slower:
  // 236 vs 220 us per iteration at c3)
  gtx_pieces(P, P.r, P.q, delta);
  grid.sync();
  coarse_pieces(P, P.kz);
  grid.sync();
  // r <- r - delta q, lam <- lam + delta p, w = P r (materialised)
  for (int g = gt; g < P.n_mult; g += nthr) {
    const double rn = __ldcg(P.r + g) - delta * __ldcg(P.q + g);
    P.lam[g] = P.lam[g] + delta * P.p[g];
    P.r[g] = rn;
    P.w[g] = rn - gz(P, g, P.kz);
  }
  grid.sync();
  // kz2 = (G^T G)^-1 G^T w
  gtx_pieces(P, P.w, nullptr, 0.0);
  grid.sync();
  coarse_pieces(P, P.kz2);
  grid.sync();
  // y = P w; w.y, w.w
  double wy = 0.0, ww = 0.0;
  for (int g = gt; g < P.n_mult; g += nthr) {
    const double wg = __ldcg(P.w + g);
    const double yg = wg - gz(P, g, P.kz2);
    P.y[g] = yg;
    wy += wg * yg;
    ww += wg * wg;
  }
  const double a1 = block_sum(wy, red);
  const double a2 = block_sum(ww, red);
  if (threadIdx.x == 0) {
    P.bpart[2 * G + 2 * b] = a1;
    P.bpart[2 * G + 2 * b + 1] = a2;
  }
  grid.sync();
  if (b != 0) return;
  const double s_wy = ordered_sum(P.bpart + 2 * G, G, 2, red);
  const double s_ww = ordered_sum(P.bpart + 2 * G + 1, G, 2, red);
  if (threadIdx.x == 0) {
    sc->pq = pq;
    sc->delta = delta;
    finalize(P, s_wy, s_ww);
  }
}

__global__ void __launch_bounds__(PT) pcpg_iter_coop(PcpgDev P) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  if (P.sc->done) return;                     // uniform: written by the previous launch only
  pcpg_vector_phases(P, grid);
}

// the whole iteration in one cooperative launch: the apply's SYMV on the
// persistent CTAs (gathering p_new = y + beta p), a grid barrier, the vector
// phases -- no launch gap between the apply and the vector work
__global__ void __launch_bounds__(PT, 1) pcpg_iter_fused(PcpgDev P, ApplyArgs A) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  if (P.sc->done) return;
  apply_body<PT / 32>(A.subs, A.segs, A.seg_ptr, A.part, P.p, P.y, &P.sc->beta, nullptr, A.sb);
  grid.sync();
  pcpg_vector_phases(P, grid);
}

int pcpg_fused_grid(int nctas, size_t smem) {
  int per_sm = 0, dev = 0, sms = 0;
  cudaFuncAttributes fa;
  // the dynamic limit excludes the kernel's static shared memory (227 KB per
  // block in total); any failure leaves the two-launch iteration in place and
  // no pending error behind
  bool ok = cudaFuncGetAttributes(&fa, pcpg_iter_fused) == cudaSuccess &&
            smem + fa.sharedSizeBytes <= 227 * 1024 &&
            cudaFuncSetAttribute(pcpg_iter_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(227 * 1024 - fa.sharedSizeBytes)) == cudaSuccess &&
            cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcpg_iter_fused, PT, smem) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    return 0;
  }
  return (per_sm * sms >= nctas) ? nctas : 0;   // every apply CTA co-resident
}

cudaError_t launch_pcpg_iter_fused(const PcpgDev& P, const ApplyArgs& A, int grid, size_t smem, cudaStream_t st) {
  PcpgDev p = P;
  ApplyArgs a = A;
  void* args[] = {&p, &a};
  return cudaLaunchCooperativeKernel((const void*)pcpg_iter_fused, dim3(grid), dim3(PT), args, smem, st);
}

int pcpg_coop_grid(int num_sms) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcpg_iter_coop, PT, 0) != cudaSuccess || per_sm < 1)
    return 0;
  return num_sms;   // one CTA per SM: co-resident by construction
}

cudaError_t launch_pcpg_iter_coop(const PcpgDev& P, int grid, cudaStream_t st) {
  PcpgDev arg = P;
  void* args[] = {&arg};
  return cudaLaunchCooperativeKernel((const void*)pcpg_iter_coop, dim3(grid), dim3(PT), args, 0, st);
}

// ---- setup kernels -----------------------------------------------------
// out = a - b (elementwise)
__global__ void __launch_bounds__(PT) pcpg_sub(int n, const double* __restrict__ a, const double* __restrict__ b,
                                                double* __restrict__ out) {
  const int g = blockIdx.x * PT + threadIdx.x;
  if (g < n) out[g] = a[g] - b[g];
}

// the initial scalars: wy = w.y, w0 = ||w||, ||d||; p = y; beta = 0
__global__ void __launch_bounds__(PT) pcpg_init_dots(PcpgDev P) {
  __shared__ double red[PT / 32];
  const int g = blockIdx.x * PT + threadIdx.x;
  double wy = 0.0, ww = 0.0, dd = 0.0;
  if (g < P.n_mult) {
    const double wg = P.w[g], yg = P.y[g], dg = P.d[g];
    wy = wg * yg;
    ww = wg * wg;
    dd = dg * dg;
    P.p[g] = yg;
  }
  const double a = block_sum(wy, red), b = block_sum(ww, red), c = block_sum(dd, red);
  if (threadIdx.x == 0) {
    P.bpart[3 * blockIdx.x] = a;
    P.bpart[3 * blockIdx.x + 1] = b;
    P.bpart[3 * blockIdx.x + 2] = c;
  }
  if (!last_block(&P.sc->cnt[0])) return;
  const double s_wy = ordered_sum(P.bpart, gridDim.x, 3, red);
  const double s_ww = ordered_sum(P.bpart + 1, gridDim.x, 3, red);
  const double s_dd = ordered_sum(P.bpart + 2, gridDim.x, 3, red);
  if (threadIdx.x == 0) {
    PcpgScal* sc = P.sc;
    sc->wy = s_wy;
    sc->w0 = sqrt(s_ww);
    sc->dnorm = sqrt(s_dd);
    sc->beta = 0.0;
    sc->k = 0;
    sc->status = PCPG_RUNNING;
    sc->done = 0;
  }
}

static int nblocks(int n) { return (n + PT - 1) / PT; }

void launch_pcpg_sub(int n, const double* a, const double* b, double* out, cudaStream_t st) {
  if (n > 0) pcpg_sub<<<nblocks(n), PT, 0, st>>>(n, a, b, out);
}
void launch_pcpg_init_dots(const PcpgDev& P, cudaStream_t st) {
  pcpg_init_dots<<<nblocks(P.n_mult), PT, 0, st>>>(P);
}
void launch_pcpg_reduce_pq(const PcpgDev& P, cudaStream_t st) { pcpg_reduce_pq<<<nblocks(P.n_mult), PT, 0, st>>>(P); }
void launch_pcpg_gtx_r(const PcpgDev& P, cudaStream_t st) {
  if (P.ncols > 0) pcpg_gtx_r<<<P.ncols, PT, 0, st>>>(P);
}
void launch_pcpg_gtx_w(const PcpgDev& P, cudaStream_t st) {
  if (P.ncols > 0) pcpg_gtx_w<<<P.ncols, PT, 0, st>>>(P);
}
void launch_pcpg_gtx_x(const PcpgDev& P, const double* x, cudaStream_t st) {
  if (P.ncols > 0) pcpg_gtx_x<<<P.ncols, PT, 0, st>>>(P, x);
}
void launch_pcpg_update(const PcpgDev& P, int mode, cudaStream_t st) {
  if (mode == 0)
    pcpg_update<0><<<nblocks(P.n_mult), PT, 0, st>>>(P);
  else if (mode == 1)
    pcpg_update<1><<<nblocks(P.n_mult), PT, 0, st>>>(P);
  else
    pcpg_update<2><<<nblocks(P.n_mult), PT, 0, st>>>(P);
}
size_t pcpg_bpart_doubles(int n_mult, int ncols) { return (size_t)3 * (nblocks(n_mult) + ncols + 1) + 4 * 1024; }

}  // namespace feti
