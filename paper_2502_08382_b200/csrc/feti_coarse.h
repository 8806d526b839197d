// Coarse-space (projector) kernels for the GPU-resident PCPG; see feti_coarse.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace feti {

struct CoarseSub {
  const double* G;     // m x r, sorted local multiplier order, row-major
  const int* gids;     // m global multiplier ids (sorted local order)
  int m, r;
  int koff;            // offset of this subdomain's kernel columns
  int pad_;
};

void launch_gtx(const CoarseSub* cs, const int2* cols, int ncols, const double* x, double* v, cudaStream_t st);
void launch_coarse(int nk, const double* C, const double* v, double* z, cudaStream_t st);
void launch_project(int n_mult, const int* cptr, const int4* cent, const CoarseSub* cs, const double* z,
                    const double* x, double sign, double* out, cudaStream_t st);

}  // namespace feti
