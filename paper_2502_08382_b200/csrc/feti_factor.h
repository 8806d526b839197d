// Device numeric factorization and full solves; see feti_factor.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "feti_common.cuh"

namespace feti {

// Per-subdomain stiffness data for the device factorization (device pointers).
struct FactorSub {
  const double* Q;          // n x r kernel basis, original DOF order, row-major
  const int64_t* perm;      // permuted position -> original DOF
  const int64_t* iperm;     // original DOF -> permuted position
  const int64_t* indptr;    // K (unregularized) CSR
  const int64_t* indices;
  const double* data;
  double rho;               // trace(K) / n
  int r;
  int pad_;
};

cudaError_t configure_factor(int max_T);
size_t solve_smem(int T);
void launch_kreg_build(const SubDev* subs, const FactorSub* fs, int nsub, int T, int n, cudaStream_t st);
int launch_factor_step(const SubDev* subs, double* dinv, int* bad, int nsub, int k, int T, cudaStream_t st);
void launch_solve(const SubDev* subs, const FactorSub* fs, const int* slots, int nslots, int max_T,
                  const int64_t* vec_off, const double* b, double* x, cudaStream_t st);

}  // namespace feti
