// Host-side launch interface of the device kernels (feti_kernels.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "feti_common.cuh"

namespace feti {

cudaError_t configure_kernels();
int kernel_attributes(char* buf, int len);
void launch_unpack(const SubDev* subs, const int4* work, int nwork, cudaStream_t st);
void launch_scatter_sparse(const SubDev* subs, int sub, int n, cudaStream_t st);
void launch_diag_inverse(const SubDev* subs, const int4* work, int nwork, cudaStream_t st);
void launch_block_scale(const SubDev* subs, const int4* work, int nwork, cudaStream_t st);
void launch_trsm_chain(const SubDev* subs, const int4* work, int nwork, cudaStream_t st);
void launch_syrk(const SubDev* subs, const int4* work, int nwork, cudaStream_t st);
// path "trsm": transpose of the trailing tiles (wd: (sub, block row)), the
// backward chains and the row gather into F (wc: (sub, panel))
void launch_trsm_path(const SubDev* subs, const int4* wd, int nd, const int4* wc, int nc, cudaStream_t st);
constexpr int APPLY_MAX_WARPS = 8;   // 3 tile buffers x 32 doubles: > 8 warps spill
size_t apply_smem(int nw, int sb);
int apply_max_sb(int nw);   // largest super-block edge (tiles) whose accumulators fit 227 KB
int apply_max_compact(int nw);   // largest subdomain (tiles) for the one-block compact layout
// sb: super-block edge in 32x32 tiles (the segments' blocking, chosen at finalize),
//     negative: one block per subdomain of -sb tiles, compact accumulators;
// py/pbeta/done: PCPG mode (gather p_new = y + beta p; no-op once *done)
void launch_apply(int nw, int sb, const SubDev* subs, const ApplySeg* segs, const int* seg_ptr, int nctas,
                  double* part, const double* p, cudaStream_t st, const double* py = nullptr,
                  const double* pbeta = nullptr, const int* done = nullptr);
void launch_reduce(int n_mult, const int* cptr, const int4* cent, const int64_t* ridx, const double* part,
                   double* q, cudaStream_t st);

}  // namespace feti
