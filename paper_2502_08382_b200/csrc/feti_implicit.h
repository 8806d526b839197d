// Implicit GPU apply through the assembly's scaled block factor; see feti_implicit.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "feti_common.cuh"

namespace feti {

size_t implicit_smem(int max_blocks);
cudaError_t configure_implicit(int max_blocks);
struct SpSub;
// ss: the sparse route's per-subdomain data (adds the rank-2r correction), or nullptr
void launch_implicit_apply(const SubDev* subs, const SpSub* ss, int nsub, int max_blocks, const int64_t* out_off,
                           const double* p, double* part, int n_mult, const int* cptr, const int4* cent, double* q,
                           cudaStream_t st);
// sparse route, once per assembly: U2 = B~ K_s^-1 Q (and U2f = B~ K_s^-1 f')
// of subdomains [sub0, sub0 + nsub) by the backward sweep from y = L^-1 P Q;
// max_cols >= r (+1 with the device dual rhs) of every subdomain
void launch_implicit_u2(const SubDev* subs, const SpSub* ss, int sub0, int nsub, int max_cols, int max_blocks,
                        cudaStream_t st);

}  // namespace feti
