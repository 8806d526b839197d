// Implicit GPU apply through the assembly's scaled block factor; see feti_implicit.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "feti_common.cuh"

namespace feti {

size_t implicit_smem(int max_blocks);
cudaError_t configure_implicit(int max_blocks);
void launch_implicit_apply(const SubDev* subs, int nsub, int max_blocks, const int64_t* out_off, const double* p,
                           double* part, int n_mult, const int* cptr, const int4* cent, double* q, cudaStream_t st);

}  // namespace feti
