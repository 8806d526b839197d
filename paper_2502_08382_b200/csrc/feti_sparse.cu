// Sparse-factor route on the device (SURVEY.md §7 hard part 4, §8f row 2;
// host side: paper_2502_08382_b200/sparse_route.py).
//
// The reference's K_reg = K + rho Q Q^T (regularize, sparse.py:427-454) is
// dense, so its factor is a full triangle (4.4 GB per config-5 subdomain).
// Here the factor is of K_s = K + rho E E^T (E = fixing DOFs): it keeps K's
// sparsity, and is stored as a pool of 128x128 tiles (the assembly's
// col-major swizzled format) covering the block pattern of L after block
// fill.  With every constrained DOF ordered last, the pool's trailing
// triangle [smin, T) x [smin, T) is dense and laid out exactly as the
// assembly expects, so the unchanged TRSM/SYRK kernels compute
// F_s = B K_s^-1 B^T from it.
//
// Factorization (left-looking, one block column j at a time, all subdomains
// batched in each launch):
//   acc:    L_ij -= sum_k L_ik L_jk^T   over k in rows(i) ∩ rows(j), k < j
//   potrf:  L_jj = chol(A_jj), D = inv(L_jj)
//   panel:  L_ij = A_ij D^T              i in struct(j)
// An extra block row holding (P Q)^T is factored along: its tiles become
// y^T = (L^-1 P Q)^T, and a final accumulation leaves -y^T y in tile (T, T).
//
// Correction (after the assembly):  with U1 = B Q, U2 = B K_s^-1 Q = X^T y_b
// (X = L^-1 P B^T lives in the interface rows only) and C = y^T y + I/rho,
//   F~ = F_s - U1 U2^T - U2 U1^T + U1 C U1^T = F_s + U1 W^T - U2 U1^T,
//   W = U1 C - U2,
// applied in place to the packed 32x32 apply tiles.
#include <algorithm>
#include <cstdlib>

#include "feti_common.cuh"
#include "feti_dense128.cuh"
#include "feti_sparse.h"

namespace feti {

// ---------------------------------------------------------------------------
// pool initialisation: zero tiles, identity on padded diagonal entries, and
// the (P Q)^T block row
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) sp_init_kernel(const SpInit* __restrict__ work, const SpSub* __restrict__ ss) {
  const SpInit w = work[blockIdx.x];
  const SpSub& S = ss[w.sub];
  double* tile = w.tile;
  const int npos = S.npos, r = S.r;
  const bool qrow = (w.K == S.T);
  for (int idx = threadIdx.x; idx < TILE; idx += 256) {
    const int jl = idx >> 7;
    const int il = (idx & 127) ^ ((jl & 3) << 2);
    const int j = w.L * TB + jl;
    const int64_t dof = j < npos ? S.perm[j] : -1;
    double v = 0.0;
    if (qrow) {
      if (w.L < S.T && dof >= 0) {
        if (il < r)
          v = S.Q[dof * r + il];
        else if (il == S.frow)
          v = S.fproj[dof];
      }
    } else if (w.K == w.L && il == jl && dof < 0) {
      v = 1.0;   // identity rows at padding positions keep the diagonal blocks SPD
    }
    tile[idx] = v;
  }
}

// rho = trace(K) / n (regularize, sparse.py:450): one CTA per subdomain,
// strided partial sums reduced in a fixed tree order (bit-reproducible)
__global__ void __launch_bounds__(256) sp_trace_kernel(const SpSub* __restrict__ ss) {
  const SpSub& S = ss[blockIdx.x];
  __shared__ double red[256];
  double acc = 0.0;
  for (int a = threadIdx.x; a < S.n; a += 256) acc += S.kdata[S.kdiag[a]];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *S.rho = red[0] / S.n;
}

// K_s entries into the lower block triangle of P K_s P^T: one warp per
// original row a; the fixing shift rho lands on the diagonal entry.
__global__ void __launch_bounds__(256) sp_scatter_kernel(const SpSub* __restrict__ ss, int sub0) {
  const SpSub& S = ss[sub0 + blockIdx.y];
  const int a = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (a >= S.n) return;
  const int lane = threadIdx.x & 31;
  bool fixed = false;
  for (int f = 0; f < S.nfix; ++f) fixed |= (S.fix[f] == a);
  const int64_t pa = S.iperm[a];
  for (int64_t p = S.kptr[a] + lane; p < S.kptr[a + 1]; p += 32) {
    const int64_t b = S.kind[p];
    const int64_t pb = S.iperm[b];
    if (pa < pb) continue;
    double v = S.kdata[p];
    if (fixed && b == a) v += *S.rho;
    const int slot = S.tmap[(pa / TB) * S.Tq + pb / TB];
    double* tile = S.pool + (size_t)slot * TILE;
    tile[swz((int)(pb % TB), (int)(pa % TB))] += v;
  }
}

// ---------------------------------------------------------------------------
// tile GEMM tasks on the DMMA pipe (8 consumer warps, 1 bulk-copy producer)
// ---------------------------------------------------------------------------
constexpr int SG_STAGES = 3;

// MI = 8: full 128-row tile; MI = 1: "thin" tile of the (P Q)^T block row,
// whose rows >= r <= 8 are zero (only warp row-group 0, first 8 rows)
template <int MI>
__device__ __forceinline__ void sg_mma_slice(const double* __restrict__ a_s, const double* __restrict__ b_s,
                                             double (&acc)[MI][4][2], int wm, int wn, int g, int t) {
#pragma unroll
  for (int kb = 0; kb < KS / 4; ++kb) {
    const int kr = kb * 4 + t;
    double bf[4];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) bf[ni] = b_s[swz(kr, wn * 32 + ni * 8 + g)];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
      const double af = a_s[swz(kr, wm * 64 + mi * 8 + g)];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af, bf[ni]);
    }
  }
}

__global__ void __launch_bounds__(256, 1) sp_potrf_kernel(const SpDiag* __restrict__ d, int* __restrict__ bad) {
  extern __shared__ double psm[];
  const SpDiag w = d[blockIdx.x];
  potrf_invert_128(w.C, w.D, bad + w.sub, w.rowbase, psm);
}

// 8 warps, no dedicated producer warp: lane 0 of warp 0 issues the bulk
// copies PREF slices ahead (after every warp released the stage), so the CTA
// has 255 registers per thread for both the DMMA tiles and potrf_invert_128.
constexpr int SG_THREADS = 256;
constexpr int SG_PREF = SG_STAGES - 1;

__device__ __forceinline__ void sg_issue(const SpPair* __restrict__ pairs, int64_t pair0, int sl, uint32_t pos,
                                          double* sA, double* sB, uint64_t* full, uint64_t* empty) {
  const int st = (int)(pos % SG_STAGES);
  const uint32_t ph = (pos / SG_STAGES) & 1;
  const SpPair pr = pairs[pair0 + sl];
  mbar_wait(&empty[st], ph ^ 1);
  mbar_arrive_expect_tx(&full[st], 2 * SLICE * 8);
  bulk_g2s(sA + st * SLICE, pr.A, SLICE * 8, &full[st]);
  bulk_g2s(sB + st * SLICE, pr.B, SLICE * 8, &full[st]);
}

// One tile task on the ring (positions pos0 ...).  `pre` slices of it were
// already issued by the previous task of this CTA; when `next` is given, its
// first slices are issued before this task's epilogue (cross-task prefetch:
// the next task's fill overlaps this epilogue).  Returns the number issued.
template <int MI>
__device__ __forceinline__ int sg_gemm(const SpPair* __restrict__ pairs, const SpTask& tk, double* sA, double* sB,
                                       uint64_t* full, uint64_t* empty, uint32_t pos0, int warp, int lane, int pre,
                                       const SpTask* next) {
  const int nsl = tk.npairs;
  const int wm = warp >> 2, wn = warp & 3;
  const int gq = lane >> 2, t = lane & 3;
  const bool issuer = (threadIdx.x == 0);
  const bool active = (MI == 8) || wm == 0;
  if (issuer) {
    fence_proxy_async_global();
    fence_proxy_async_shared();
    if (!pre && !(tk.flags & 1)) bulk_prefetch_l2(tk.C, TILE * 8);
    for (int sl = pre; sl < SG_PREF && sl < nsl; ++sl) sg_issue(pairs, tk.pair0, sl, pos0 + sl, sA, sB, full, empty);
  }
  double acc[MI][4][2];
#pragma unroll
  for (int a = 0; a < MI; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  for (int sl = 0; sl < nsl; ++sl) {
    const uint32_t pos = pos0 + sl;
    if (issuer && sl + SG_PREF < nsl)
      sg_issue(pairs, tk.pair0, sl + SG_PREF, pos + SG_PREF, sA, sB, full, empty);
    const int st = (int)(pos % SG_STAGES);
    mbar_wait(&full[st], (pos / SG_STAGES) & 1);
    if (active) sg_mma_slice<MI>(sA + st * SLICE, sB + st * SLICE, acc, wm, wn, gq, t);
    fence_proxy_async_shared();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  int issued = 0;
  if (next) {
    const int nsl2 = next->npairs;
    issued = min(SG_PREF, nsl2);
    if (issuer) {
      if (!(next->flags & 1)) bulk_prefetch_l2(next->C, TILE * 8);
      for (int sl = 0; sl < issued; ++sl) sg_issue(pairs, next->pair0, sl, pos0 + nsl + sl, sA, sB, full, empty);
    }
  }
  if (!active) return issued;
  double* Ct = tk.C;
  const bool panel = tk.flags & 1;
  if (panel) {
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
      const int m = wm * 64 + mi * 8 + gq;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int nn = wn * 32 + ni * 8 + 2 * t;
#pragma unroll
        for (int e = 0; e < 2; ++e) Ct[swz(nn + e, m)] = acc[mi][ni][e];
      }
    }
    return issued;
  }
  tile_sub_acc<MI>(Ct, acc, wm, wn, gq, t);   // C -= acc, loads one fragment row ahead
  return issued;
}

// persistent over the launch's tasks: CTA b runs tasks b, b + grid, ...
// (sorted by decreasing size), the ring continuing across them
__global__ void __launch_bounds__(SG_THREADS, 1) sp_gemm8_kernel(const SpTask* __restrict__ tasks, int ntasks,
                                                                  const SpPair* __restrict__ pairs) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sA = reinterpret_cast<double*>(smem_raw);
  double* sB = sA + SG_STAGES * SLICE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + SG_STAGES * SLICE);
  uint64_t* empty = full + SG_STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int st = 0; st < SG_STAGES; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 8);
    }
    mbar_fence_init();
  }
  __syncthreads();
  uint32_t pos = 0;
  int pre = 0;
  for (int ti = blockIdx.x; ti < ntasks; ti += gridDim.x) {
    const SpTask tk = tasks[ti];
    const SpTask* nx = (ti + (int)gridDim.x < ntasks) ? tasks + ti + gridDim.x : nullptr;
    if (!(tk.flags & 2))
      pre = sg_gemm<8>(pairs, tk, sA, sB, full, empty, pos, warp, lane, pre, nx);
    else
      pre = sg_gemm<1>(pairs, tk, sA, sB, full, empty, pos, warp, lane, pre, nx);
    pos += (uint32_t)tk.npairs;
  }
}

// ---------------------------------------------------------------------------
// correction
// ---------------------------------------------------------------------------
constexpr int MAXR = 8;

// one CTA per (sub, panel c): U2[a] = sum_rows X[row][a] y[row], then
// W[a] = C U1[a] - U2[a] with C = y^T y + I/rho = -tile(T,T) + I/rho
constexpr int U2_GROUPS = 4;   // row groups per CTA (U2_GROUPS x 128 threads)

// NR: accumulator columns (>= every launched subdomain's nr), CH independent
// row chains per thread (loads in flight: the kernel is latency-bound at one
// row per chain step)
template <int NR, int CH>
__global__ void __launch_bounds__(U2_GROUPS * TB) sp_u2_kernel(const SubDev* __restrict__ subs,
                                                              const SpSub* __restrict__ ss,
                                                              const int2* __restrict__ panels) {
  const int2 pc = panels[blockIdx.x];
  const SubDev& S = subs[pc.x];
  const SpSub& Q = ss[pc.x];
  const int c = pc.y, col = threadIdx.x & (TB - 1), rg = threadIdx.x >> 7, r = Q.r;
  const int nr = Q.frow >= 0 ? Q.frow + 1 : r;   // rows of y used: Q columns, then f' (device dual rhs)
  const int a = c * TB + col;
  const int T = Q.T;
  __shared__ double Cm[MAXR * MAXR];
  __shared__ double red[U2_GROUPS][MAXR][TB];
  const double* cq = Q.pool + (size_t)Q.tmap[T * Q.Tq + T] * TILE;
  if (threadIdx.x < r * r) {
    const int q = threadIdx.x / r, q2 = threadIdx.x % r;
    Cm[threadIdx.x] = -cq[swz(q2, q)] + (q == q2 ? 1.0 / *Q.rho : 0.0);
  }
  // rows split over the row groups (row = kb*128 + il, il = rg mod U2_GROUPS),
  // CH independent accumulator chains per group
  double acc[CH][NR];
#pragma unroll
  for (int h = 0; h < CH; ++h)
#pragma unroll
    for (int q = 0; q < NR; ++q) acc[h][q] = 0.0;
  const int r0 = (S.panel_minrow[c] / TB) * TB;
  for (int kb = r0 / TB; kb < T; ++kb) {
    const double* yt = Q.pool + (size_t)Q.tmap[T * Q.Tq + kb] * TILE;
    for (int il = rg; il < TB; il += CH * U2_GROUPS) {
      double x[CH];
#pragma unroll
      for (int h = 0; h < CH; ++h) {
        const int row = kb * TB + il + h * U2_GROUPS;
        x[h] = xrow_ptr(S, c, row)[col ^ ((row & 3) << 2)];
      }
#pragma unroll
      for (int h = 0; h < CH; ++h)
#pragma unroll
        for (int q = 0; q < NR; ++q)
          if (q < nr) acc[h][q] = fma(x[h], yt[swz(il + h * U2_GROUPS, q)], acc[h][q]);
    }
  }
#pragma unroll
  for (int q = 0; q < NR; ++q)
    if (q < nr) {
      double v = 0.0;
#pragma unroll
      for (int h = 0; h < CH; ++h) v += acc[h][q];
      red[rg][q][col] = v;
    }
  __syncthreads();
  if (rg != 0) return;
  double tot[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    double v = 0.0;
    if (q < nr)
      for (int g2 = 0; g2 < U2_GROUPS; ++g2) v += red[g2][q][col];
    tot[q] = (a < S.m) ? v : 0.0;
  }
  if (Q.frow >= 0) {
#pragma unroll
    for (int q = 0; q < NR; ++q)
      if (q == Q.frow) Q.U2f[a] = tot[q];   // X^T y_f = B~ K_s^-1 f'
  }
  if (r == 0) return;
  double* out = Q.U2W + (size_t)a * 2 * r;
  const double* u1 = Q.U1 + (size_t)a * r;
#pragma unroll
  for (int q = 0; q < NR; ++q)
    if (q < r) {
      double w = -tot[q];
      for (int q2 = 0; q2 < r; ++q2) w = fma(Cm[q * r + q2], u1[q2], w);
      out[q] = tot[q];
      out[r + q] = (a < S.m) ? w : 0.0;
    }
}

// F[a][b] += U1[a] . W[b] - U2[a] . U1[b] over every stored apply tile
// (grid: tile row ti x subdomain; diagonal tiles are stored full)
__global__ void __launch_bounds__(256) sp_correct_kernel(const SubDev* __restrict__ subs,
                                                         const SpSub* __restrict__ ss, int sub0) {
  const SubDev& S = subs[sub0 + blockIdx.y];
  const SpSub& Q = ss[sub0 + blockIdx.y];
  const int ti = blockIdx.x, T32 = S.T32, r = Q.r;
  if (ti >= T32 || r == 0) return;
  __shared__ double u1a[AT * MAXR], u2a[AT * MAXR];
  for (int e = threadIdx.x; e < AT * r; e += 256) {
    const int a = ti * AT + e / r, q = e % r;
    u1a[e] = Q.U1[(size_t)a * r + q];
    u2a[e] = Q.U2W[(size_t)a * 2 * r + q];
  }
  __syncthreads();
  for (int tj = ti; tj < T32; ++tj) {
    double* F = S.F + apply_tile_index(ti, tj, T32) * ATILE;
    for (int e = threadIdx.x; e < ATILE; e += 256) {
      const int al = e / AT, b = tj * AT + e % AT;
      const double* u1b = Q.U1 + (size_t)b * r;
      const double* wb = Q.U2W + (size_t)b * 2 * r + r;
      double v = F[e];
      for (int q = 0; q < r; ++q) v += u1a[al * r + q] * wb[q] - u2a[al * r + q] * u1b[q];
      F[e] = v;
    }
  }
}


// d[g] = sum_(s,a) [ (X^T y_f)_a - U1_a . (y^T y_f) + U1_a . (Q^T f) / rho ] - c[g]
// with K_reg^-1 = Pi K_s^-1 Pi + rho^-1 Q Q^T (Pi = I - Q Q^T, f' = Pi f):
//   B~ K_reg^-1 f = B~ K_s^-1 f' - U1 Q^T K_s^-1 f' + rho^-1 U1 Q^T f,
//   Q^T K_s^-1 f' = y^T y_f = -tile(T, T)[q][frow].  Contributions in the
// reference's gather order (assemble_dual_system, solver.py:141-143).
__global__ void __launch_bounds__(256) sp_dual_rhs_kernel(const SpSub* __restrict__ ss, int n_mult,
                                                          const int* __restrict__ cptr, const int4* __restrict__ cent,
                                                          const double* __restrict__ c, double* __restrict__ d) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_mult) return;
  double acc = 0.0;
  for (int e = cptr[g]; e < cptr[g + 1]; ++e) {
    const int4 ce = cent[e];
    const SpSub& S = ss[ce.w];
    const int a = ce.x, r = S.r;
    double v = S.U2f[a];
    if (r > 0) {
      const double* cq = S.pool + (size_t)S.tmap[S.T * S.Tq + S.T] * TILE;
      const double irho = 1.0 / *S.rho;
      double corr = 0.0;
      for (int q = 0; q < r; ++q) {
        const double yyf = -cq[swz(S.frow, q)];
        corr = fma(S.U1[(size_t)a * r + q], irho * S.qtf[q] - yyf, corr);
      }
      v += corr;
    }
    acc += v;
  }
  d[g] = acc - (c ? c[g] : 0.0);
}

// ---------------------------------------------------------------------------
// host: block symbolic factorization and task lists
// ---------------------------------------------------------------------------
void sp_symbolic(int64_t n, const int64_t* indptr, const int64_t* indices, const int64_t* iperm, int64_t npos,
                 int r, int smin, SpPlan* out, bool extra_row) {
  SpPlan& P = *out;
  const int T = (int)((npos + TB - 1) / TB);
  const int Tq = T + ((r > 0 || extra_row) ? 1 : 0);
  P.T = T;
  P.Tq = Tq;
  P.smin = smin = std::min(std::max(smin, 0), T);
  // cs[j][i] = 1: block (i, j), i > j, of L is structurally nonzero
  std::vector<std::vector<char>> cs(T, std::vector<char>(Tq, 0));
  for (int64_t a = 0; a < n; ++a)
    for (int64_t p = indptr[a]; p < indptr[a + 1]; ++p) {
      int I = (int)(iperm[a] / TB), J = (int)(iperm[indices[p]] / TB);
      if (I < J) std::swap(I, J);
      if (I > J) cs[J][I] = 1;
    }
  for (int J = smin; J < T; ++J)
    for (int I = J + 1; I < T; ++I) cs[J][I] = 1;     // dense interface block
  if (Tq > T)
    for (int J = 0; J < T; ++J) cs[J][T] = 1;         // (P Q)^T row: y is dense
  // block fill along the elimination tree: struct(parent) >= struct(k) \ {parent}
  for (int k = 0; k < T; ++k) {
    int par = -1;
    for (int I = k + 1; I < Tq; ++I)
      if (cs[k][I]) {
        par = I;
        break;
      }
    if (par < 0 || par >= T) continue;
    for (int I = par + 1; I < Tq; ++I)
      if (cs[k][I]) cs[par][I] = 1;
  }
  // k-slice masks of the scalar factor per (block row, block column)
  std::vector<uint8_t> smask;
  // scalar work of the same ordering (the algorithmic figure): elimination
  // tree (Liu, path compression) and column counts by row-subtree walks,
  // O(nnz(L)); flops = sum_j c_j (c_j + 3), c_j = nonzeros below the diagonal
  {
    std::vector<int64_t> pos_dof(npos, -1);
    for (int64_t a = 0; a < n; ++a) pos_dof[iperm[a]] = a;
    std::vector<int64_t> parent(npos, -1), anc(npos, -1), mark(npos, -1), cnt(npos, 0);
    for (int64_t i = 0; i < npos; ++i) {
      const int64_t a = pos_dof[i];
      if (a < 0) continue;
      for (int64_t p = indptr[a]; p < indptr[a + 1]; ++p) {
        int64_t k = iperm[indices[p]];
        while (k >= 0 && k < i) {          // etree with path compression
          const int64_t nx = anc[k];
          anc[k] = i;
          if (nx < 0) {
            parent[k] = i;
            break;
          }
          k = nx;
        }
      }
    }
    smask.assign((size_t)Tq * Tq, 0);
    for (int64_t i = 0; i < npos; ++i) {
      smask[(size_t)(i / TB) * Tq + i / TB] |= (uint8_t)(1u << ((i % TB) / KS));   // L(i, i) (identity at padding)
      const int64_t a = pos_dof[i];
      if (a < 0) continue;
      mark[i] = i;
      for (int64_t p = indptr[a]; p < indptr[a + 1]; ++p) {
        for (int64_t j = iperm[indices[p]]; j >= 0 && j < i && mark[j] != i; j = parent[j]) {
          ++cnt[j];                          // L(i, j) != 0
          mark[j] = i;
          smask[(size_t)(i / TB) * Tq + j / TB] |= (uint8_t)(1u << ((j % TB) / KS));
        }
      }
    }
    double fl = 0.0;
    int64_t nl = 0;
    for (int64_t j = 0; j < npos; ++j) {
      fl += (double)cnt[j] * (double)(cnt[j] + 3);
      nl += cnt[j] + (pos_dof[j] >= 0 ? 1 : 0);
    }
    P.nnz_l = nl;
    P.flops_scalar = fl + 4.0 * r * (double)nl;   // + y = L^-1 P Q and y^T y
  }
  // slots: everything outside the trailing triangle first, then the trailing
  // triangle in the assembly's tri_index order
  P.tmap.assign((size_t)Tq * Tq, -1);
  auto stored = [&](int I, int J) { return (I == J && J < T) || (J < T && I > J && cs[J][I]) || (I == T && J == T && Tq > T); };
  auto trailing = [&](int I, int J) { return I < T && J >= smin; };
  int64_t ns = 0;
  for (int J = 0; J < Tq; ++J)
    for (int I = J; I < Tq; ++I)
      if (stored(I, J) && !trailing(I, J)) P.tmap[(size_t)I * Tq + J] = (int)ns++;
  P.trail_base = ns;
  for (int I = smin; I < T; ++I)
    for (int J = smin; J <= I; ++J) P.tmap[(size_t)I * Tq + J] = (int)(ns + tri_index(I - smin, J - smin));
  ns += (int64_t)(T - smin) * (T - smin + 1) / 2;
  P.ntiles = ns;
  const bool kmask = !(getenv("FETI_SP_KMASK") && atoi(getenv("FETI_SP_KMASK")) == 0);
  P.slot_mask.assign((size_t)ns, 0xF);
  if (kmask)
    for (int I = 0; I < T; ++I)
      for (int J = 0; J <= I; ++J) {
        const int sl = P.tmap[(size_t)I * Tq + J];
        if (sl >= 0) P.slot_mask[sl] = smask[(size_t)I * Tq + J];
      }
  auto popc = [](unsigned v) { return (double)__builtin_popcount(v); };
  // row structures (ascending)
  std::vector<std::vector<int>> rows(Tq);
  for (int J = 0; J < T; ++J)
    for (int I = J + 1; I < Tq; ++I)
      if (cs[J][I]) rows[I].push_back(J);
  const double tf = 2.0 * TB * TB * TB;
  P.acc.assign(Tq, {});
  P.panel.assign(Tq, {});
  for (int j = 0; j < Tq; ++j) {
    std::vector<int> targets;
    targets.push_back(j);
    if (j < T)
      for (int I = j + 1; I < Tq; ++I)
        if (cs[j][I]) targets.push_back(I);
    for (int i : targets) {
      std::vector<std::pair<int, int>> pr;
      const std::vector<int>& ri = rows[i];
      const std::vector<int>& rj = rows[j];
      size_t u = 0, v = 0;
      while (u < ri.size() && v < rj.size()) {
        if (ri[u] < rj[v]) {
          ++u;
        } else if (rj[v] < ri[u]) {
          ++v;
        } else {
          const int k = ri[u];
          pr.emplace_back(P.tmap[(size_t)i * Tq + k], P.tmap[(size_t)j * Tq + k]);
          ++u;
          ++v;
        }
      }
      const double tfi = (i == T && Tq > T) ? tf / 16.0 : tf;   // thin (P Q)^T row tiles
      // drop products whose operands share no nonzero k-slice (exact zeros)
      std::vector<std::pair<int, int>> live;
      double sl_count = 0;
      for (const auto& ab : pr) {
        const unsigned mk = P.slot_mask[ab.first] & P.slot_mask[ab.second];
        if (mk) {
          live.push_back(ab);
          sl_count += popc(mk);
        }
      }
      if (!live.empty()) {
        P.flops_exec += tfi * sl_count / (TB / KS);
        P.acc[j].emplace_back(P.tmap[(size_t)i * Tq + j], std::move(live));
      }
      if (i != j) {
        const int cs_slot = P.tmap[(size_t)i * Tq + j];
        P.panel[j].push_back(cs_slot);
        P.flops_exec += tfi * popc(P.slot_mask[cs_slot]) / (TB / KS);
      }
    }
    if (j < T) P.flops_exec += (double)TB * TB * TB / 3.0 + (double)TB * TB * TB / 3.0;  // potrf + inverse
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
static size_t sg_smem() { return 2 * SG_STAGES * SLICE * sizeof(double) + 8 * 2 * SG_STAGES; }
static size_t sp_potrf_smem() { return POTRF_SMEM_DOUBLES * sizeof(double); }

cudaError_t configure_sparse() {
  cudaError_t e;
  static_assert(POTRF_SMEM_DOUBLES * 8 <= 2 * SG_STAGES * SLICE * 8, "potrf scratch must fit the GEMM ring");
  if ((e = cudaFuncSetAttribute(sp_gemm8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sg_smem())))
    return e;
  return cudaFuncSetAttribute(sp_potrf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp_potrf_smem());
}

void launch_sp_init(const SpInit* w, int nw, const SpSub* ss, cudaStream_t st) {
  if (nw > 0) sp_init_kernel<<<nw, 256, 0, st>>>(w, ss);
}

void launch_sp_scatter(const SpSub* ss, int sub0, int nsub, int max_n, cudaStream_t st) {
  if (nsub > 0 && max_n > 0) sp_scatter_kernel<<<dim3((max_n + 7) / 8, nsub), 256, 0, st>>>(ss, sub0);
}

void launch_sp_trace(const SpSub* ss, int nsub, cudaStream_t st) {
  if (nsub > 0) sp_trace_kernel<<<nsub, 256, 0, st>>>(ss);
}

void launch_sp_gemm(const SpTask* tasks, int ntasks, const SpPair* pairs, cudaStream_t st) {
  // tasks per CTA: 1 by default.  Measured (c3, scripts/gpu_exp_tpc.sh):
  // 1/2/3/4 tasks per CTA give 42.3/45.4/49.8/55.9 ms -- fewer, longer CTAs
  // per launch cost more cross-stream concurrency than the cross-task
  // prefetch saves
  static const int tpc = getenv("FETI_SP_TPC") ? std::max(1, atoi(getenv("FETI_SP_TPC"))) : 1;
  if (ntasks > 0) sp_gemm8_kernel<<<(ntasks + tpc - 1) / tpc, SG_THREADS, sg_smem(), st>>>(tasks, ntasks, pairs);
}

void launch_sp_potrf(const SpDiag* d, int nd, int* bad, cudaStream_t st) {
  if (nd > 0) sp_potrf_kernel<<<nd, 256, sp_potrf_smem(), st>>>(d, bad);
}

void launch_sp_dual_rhs(const SpSub* ss, int n_mult, const int* cptr, const int4* cent, const double* c, double* d,
                        cudaStream_t st) {
  if (n_mult > 0) sp_dual_rhs_kernel<<<(n_mult + 255) / 256, 256, 0, st>>>(ss, n_mult, cptr, cent, c, d);
}

void launch_sp_u2(const SubDev* subs, const SpSub* ss, const int2* panels, int npanels, int max_cols,
                  cudaStream_t st) {
  if (npanels <= 0) return;
  // more row chains for narrow y (heat: one kernel column)
  if (max_cols <= 1)
    sp_u2_kernel<1, 8><<<npanels, U2_GROUPS * TB, 0, st>>>(subs, ss, panels);
  else if (max_cols <= 2)
    sp_u2_kernel<2, 8><<<npanels, U2_GROUPS * TB, 0, st>>>(subs, ss, panels);
  else if (max_cols <= 4)
    sp_u2_kernel<4, 4><<<npanels, U2_GROUPS * TB, 0, st>>>(subs, ss, panels);
  else
    sp_u2_kernel<MAXR, 2><<<npanels, U2_GROUPS * TB, 0, st>>>(subs, ss, panels);
}

void launch_sp_correct(const SubDev* subs, const SpSub* ss, const int2* panels, int npanels, int sub0, int nsub,
                       int max_T32, int max_cols, cudaStream_t st) {
  launch_sp_u2(subs, ss, panels, npanels, max_cols, st);
  if (nsub > 0 && max_T32 > 0) sp_correct_kernel<<<dim3(max_T32, nsub), 256, 0, st>>>(subs, ss, sub0);
}

}  // namespace feti
