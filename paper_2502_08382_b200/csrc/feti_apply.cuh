// Batched packed SYMV of the apply (kernel 6 of DESIGN.md §4), shared by
// apply_kernel (feti_kernels.cu) and the fused PCPG iteration
// (feti_pcpg.cu).  Dynamic shared memory: apply_smem(NW, sb).
#pragma once
#include "feti_common.cuh"

namespace feti {

// Work unit: a segment of one super-block (I, J) of SB x SB tiles of a
// subdomain's packed upper triangle (ApplySeg).  The concatenated tile list
// of all super-blocks of all subdomains is cut into one contiguous, equal
// range per CTA (persistent, one CTA per SM), so the load is balanced to a
// tile and the per-warp accumulators span at most 2 x SBE multipliers,
// whatever the subdomain's m (no size limit, and NW warps always fit).
//
// Lane l of a warp owns column l of a 32x32 tile (32 coalesced 256-byte row
// reads per tile); three tiles per warp live in registers so two loads are in
// flight while one is reduced.
__device__ __forceinline__ void apply_tile_load(double (&f)[32], const double* __restrict__ Ft, int lane) {
#pragma unroll
  for (int r = 0; r < 32; ++r) f[r] = __ldcs(Ft + r * AT + lane);
}

// row sums into myr[li], column sums (transposed contribution of an
// off-diagonal tile) into myc[lj]
__device__ __forceinline__ void apply_tile_compute(double (&f)[32], int li, int lj, bool offdiag,
                                                   const double* __restrict__ pr, const double* __restrict__ pc,
                                                   double* __restrict__ myr, double* __restrict__ myc, int lane) {
  if (offdiag) {
    double cs = 0.0;
#pragma unroll
    for (int r = 0; r < 32; ++r) cs = fma(f[r], pr[li * AT + r], cs);
    myc[lj * AT + lane] += cs;
  }
  const double pj = pc[lj * AT + lane];
#pragma unroll
  for (int r = 0; r < 32; ++r) f[r] *= pj;
  // butterfly transpose-reduce: lane r ends with sum_l F[r][l] p_J[l]
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < off; ++i) {
      const double send = up ? f[i] : f[i + off];
      const double keep = up ? f[i + off] : f[i];
      f[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  myr[li * AT + lane] += f[0];
}

// Tile cursor inside a super-block: h x w tiles (rectangle), or for a
// diagonal block the upper triangle of h x h tiles, row-major.  Located once
// per segment, then advanced incrementally (no division or square root on
// the path that computes the next load's address).
struct SbCursor {
  int li, lj;
  __device__ __forceinline__ void locate(int t, int h, int w, bool diag) {
    li = 0;
    lj = diag ? 0 : 0;
    advance(t, h, w, diag);
  }
  __device__ __forceinline__ void advance(int step, int h, int w, bool diag) {
    if (!diag) {
      lj += step;
      while (lj >= w && li < h) {
        lj -= w;
        ++li;
      }
      return;
    }
    int rem = (lj - li) + step;
    while (li < h && rem >= h - li) {
      rem -= h - li;
      ++li;
    }
    lj = li + rem;
  }
};

template <int NW>
__device__ __forceinline__ void apply_body(const SubDev* __restrict__ subs,
                                                        const ApplySeg* __restrict__ segs,
                                                        const int* __restrict__ seg_ptr,
                                                        double* __restrict__ part,
                                                        const double* __restrict__ p,
                                                        const double* __restrict__ py,
                                                        const double* __restrict__ pbeta,
                                                        const int* __restrict__ done, int sb) {
  // PCPG mode (py != nullptr): the gathered vector is p_new = y + beta p
  // (fma, bit-identical to the reduce-side update, feti_pcpg.cu); `done`
  // turns the launch into a no-op once the device loop has finished
  if (done && *done) return;
  extern __shared__ double asmem[];
  const double beta = py ? *pbeta : 0.0;
  auto pval = [&](int gi) -> double { return py ? fma(beta, __ldg(p + gi), __ldg(py + gi)) : __ldg(p + gi); };
  // sb > 0: super-blocks of sb tiles, per warp row + column accumulators;
  // sb < 0: every subdomain is one diagonal block of -sb tiles (compact
  // layout: row accumulators only, as many as fit for small m)
  const bool compact = sb < 0;
  const int SBE = (compact ? -sb : sb) * AT;   // multipliers per super-block edge
  const int WS = compact ? SBE : 2 * SBE;      // accumulator stride per warp
  double* spr = asmem;                  // p of the block's rows
  double* spc = asmem + SBE;            // p of the block's columns (off-diagonal blocks)
  double* acc = asmem + (compact ? SBE : 2 * SBE);   // warp w: rows at acc + w WS, columns at + SBE
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (compact) sb = -sb;
  // accumulators are zeroed once; each combine re-zeroes what it read
  for (int a = tid; a < NW * WS; a += NW * 32) acc[a] = 0.0;
  for (int sg = seg_ptr[blockIdx.x]; sg < seg_ptr[blockIdx.x + 1]; ++sg) {
    const ApplySeg w = segs[sg];
    const SubDev& S = subs[w.sub];
    const int T32 = S.T32;
    const int r0 = w.I * sb, c0 = w.J * sb;
    const int h = min(sb, T32 - r0), wd = min(sb, T32 - c0);
    const bool diag = w.I == w.J;
    const double* Fb = S.F;
    auto tile_ptr = [&](const SbCursor& c) -> const double* {
      return Fb + apply_tile_index(r0 + c.li, c0 + c.lj, T32) * ATILE;
    };
    int tt = w.t0 + warp;
    const int t1 = w.t1;
    // cu: the tile being reduced; ld: the tile two loads ahead.  The first
    // two tile loads are issued before the p gather so their latency
    // overlaps it (each segment restarts the pipeline)
    SbCursor cu, ld;
    cu.locate(tt, h, wd, diag);
    ld = cu;
    double fa[32], fb[32], fc[32];
    if (tt < t1) apply_tile_load(fa, tile_ptr(ld), lane);
    ld.advance(NW, h, wd, diag);
    if (tt + NW < t1) apply_tile_load(fb, tile_ptr(ld), lane);
    ld.advance(NW, h, wd, diag);
    __syncthreads();   // the previous segment's combine is done with smem
    for (int a = tid; a < h * AT; a += NW * 32) {
      const int gi = S.gids_sorted[r0 * AT + a];
      spr[a] = gi >= 0 ? pval(gi) : 0.0;
    }
    if (!diag)
      for (int a = tid; a < wd * AT; a += NW * 32) {
        const int gi = S.gids_sorted[c0 * AT + a];
        spc[a] = gi >= 0 ? pval(gi) : 0.0;
      }
    __syncthreads();
    double* myr = acc + warp * WS;
    double* myc = diag ? myr : myr + SBE;
    const double* pc = diag ? spr : spc;
    while (tt < t1) {
      if (tt + 2 * NW < t1) apply_tile_load(fc, tile_ptr(ld), lane);
      ld.advance(NW, h, wd, diag);
      apply_tile_compute(fa, cu.li, cu.lj, !diag || cu.li != cu.lj, spr, pc, myr, myc, lane);
      cu.advance(NW, h, wd, diag);
      tt += NW;
      if (tt >= t1) break;
      if (tt + 2 * NW < t1) apply_tile_load(fa, tile_ptr(ld), lane);
      ld.advance(NW, h, wd, diag);
      apply_tile_compute(fb, cu.li, cu.lj, !diag || cu.li != cu.lj, spr, pc, myr, myc, lane);
      cu.advance(NW, h, wd, diag);
      tt += NW;
      if (tt >= t1) break;
      if (tt + 2 * NW < t1) apply_tile_load(fb, tile_ptr(ld), lane);
      ld.advance(NW, h, wd, diag);
      apply_tile_compute(fc, cu.li, cu.lj, !diag || cu.li != cu.lj, spr, pc, myr, myc, lane);
      cu.advance(NW, h, wd, diag);
      tt += NW;
    }
    __syncthreads();
    // combine the warps in fixed order (deterministic)
    for (int a = tid; a < h * AT; a += NW * 32) {
      double s = 0.0;
#pragma unroll
      for (int wi = 0; wi < NW; ++wi) {
        s += acc[wi * WS + a];
        acc[wi * WS + a] = 0.0;
      }
      part[w.out_r + a] = s;
    }
    if (!diag)
      for (int a = tid; a < wd * AT; a += NW * 32) {
        double s = 0.0;
#pragma unroll
        for (int wi = 0; wi < NW; ++wi) {
          s += acc[wi * WS + SBE + a];
          acc[wi * WS + SBE + a] = 0.0;
        }
        part[w.out_c + a] = s;
      }
  }
}

}  // namespace feti
