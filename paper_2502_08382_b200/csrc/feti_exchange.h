// Cross-rank exchange fused into the apply's reduction (feti_exchange.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace feti {

struct XchgArgs {
  double* const* peers;     // [world] slab base of every rank (own included), device pointers
  const int* touched;       // multipliers this rank contributes to (ascending)
  const int* cptr;          // contribution CSR of this rank (as reduce_kernel)
  const int4* cent;
  const int64_t* ridx;      // partial positions per contribution (as reduce_kernel)
  const double* part;
  unsigned* done;           // CTA completion counter (own memory)
  int* error;               // set when a peer never arrived
  int64_t epoch;            // 1, 2, ... per apply
  int n_touched, n_mult, rank, world;
};

void launch_exchange(const XchgArgs& a, double* q, cudaStream_t st);

}  // namespace feti
