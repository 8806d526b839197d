// Device-native PCPG kernels (feti_pcpg.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "feti_coarse.h"
#include "feti_common.cuh"

namespace feti {

enum { PCPG_RUNNING = 0, PCPG_CONVERGED = 1, PCPG_BREAKDOWN = 2, PCPG_MAXIT = 3 };

// device scalars of one solve (also read by the host once per graph launch)
struct PcpgScal {
  double wy, w0, tolw0, delta, beta, pq, wn, ww, dnorm;
  long long k, maxit;
  int status, done;
  unsigned cnt[4];   // last-block counters (reset by the last block)
};

struct PcpgDev {
  int n_mult, nk, ncols, pad_;
  // apply partials (reduce_kernel's layout) and the coarse space
  const int* cptr;
  const int4* cent;
  const int64_t* ridx;
  const double* part;
  const CoarseSub* cs;
  const int2* kcols;
  const double* cinv;
  const double* d;
  // iteration vectors
  double *lam, *r, *p, *q, *y, *w, *z;
  double *kv, *kz, *kv2, *kz2;
  double* bpart;
  PcpgScal* sc;
  // G flattened by kernel column (entries of a column contiguous) and cut into
  // pieces of <= kPiece entries that never straddle columns: G^T x is one
  // fully parallel pass over the pieces, then rows of (G^T G)^-1 times the
  // piece sums (pcpg_iter_coop)
  const double* gval;       // G entry
  const int* gidx;          // its global multiplier
  const int4* pieces;       // (column, first entry, end entry, -)
  int npieces, pad2_;
  double* ppart;            // per-piece partial sums
};
constexpr int kPiece = 512;

void launch_pcpg_sub(int n, const double* a, const double* b, double* out, cudaStream_t st);
void launch_pcpg_init_dots(const PcpgDev& P, cudaStream_t st);
void launch_pcpg_reduce_pq(const PcpgDev& P, cudaStream_t st);
void launch_pcpg_gtx_r(const PcpgDev& P, cudaStream_t st);
void launch_pcpg_gtx_w(const PcpgDev& P, cudaStream_t st);
void launch_pcpg_gtx_x(const PcpgDev& P, const double* x, cudaStream_t st);
void launch_pcpg_update(const PcpgDev& P, int mode, cudaStream_t st);
size_t pcpg_bpart_doubles(int n_mult, int ncols);
// the apply's work description (apply_kernel's arguments)
struct ApplyArgs {
  const SubDev* subs;
  const ApplySeg* segs;
  const int* seg_ptr;
  double* part;
  int sb, pad_;
};
// the whole iteration (apply + vector work) in one cooperative launch of the
// apply's CTAs (8 warps each); returns 0 when they cannot all be co-resident
int pcpg_fused_grid(int nctas, size_t smem);
cudaError_t launch_pcpg_iter_fused(const PcpgDev& P, const ApplyArgs& A, int grid, size_t smem, cudaStream_t st);
// one cooperative launch for B + D + F + G (grid-wide barriers); grid <= 0: unavailable
int pcpg_coop_grid(int num_sms);
cudaError_t launch_pcpg_iter_coop(const PcpgDev& P, int grid, cudaStream_t st);

}  // namespace feti
