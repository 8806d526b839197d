// Multi-GPU apply with the cross-rank exchange fused into the reduction
// (SURVEY.md §8e): instead of reducing into a full-length vector and then
// calling an all-reduce, each rank's reduction kernel stores its per-
// multiplier sums straight into every peer's receive slab over NVLink (CUDA
// IPC peer memory), the last CTA publishes an epoch flag to every peer, and a
// second kernel waits for all ranks' flags and sums the slabs in rank order.
//
// * Each multiplier touches at most two subdomains (a gluing pair,
//   decomposition.py:184-207), and the sum over ranks runs in fixed rank
//   order, so q is deterministic (identical on every rank and run to run).
// * Slab layout per rank: recv[2][world][n_mult] doubles (double-buffered by
//   epoch parity) followed by flags[world] (int64, last epoch published by
//   each source rank).  Entries of rank r's slab outside r's multipliers are
//   never written and stay zero.
// * Reuse safety: rank r writes slab parity e%2 for epoch e only after its
//   own sum of epoch e-1 returned, which needed every peer's flag e-1, which
//   each peer publishes after its sum of epoch e-2 -- the last reader of
//   that parity.
// * The wait is bounded: after ~10 s without progress the kernel records a
//   sticky error (feti_exchange_status) and writes NaN to its part of q, so
//   a lost peer can never leave stale or half-updated values that look valid.
// * Memory ordering across GPUs: every thread's remote stores of the reduce
//   kernel are ordered before its CTA's __syncthreads; thread 0 then issues
//   __threadfence_system (a fence.sc.sys: cumulative, so it orders the CTA's
//   stores observed through the barrier before everything thread 0 does
//   next) and bumps the CTA counter; the last CTA fences again and publishes
//   the epoch with st.release.sys.  A reader's ld.acquire.sys of that flag
//   therefore synchronises with all CTAs' slab stores (release sequence via
//   the device-scope atomic counter + system fences), so the summing kernel
//   never reads a slab entry older than the epoch it waited for.
#include <cstdint>

#include "feti_common.cuh"
#include "feti_exchange.h"

namespace feti {

__device__ __forceinline__ void st_release_sys_s64(int64_t* p, int64_t v) {
  asm volatile("st.release.sys.global.s64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t ld_acquire_sys_s64(const int64_t* p) {
  int64_t v;
  asm volatile("ld.acquire.sys.global.s64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// local sums of this rank's multipliers -> every peer's slab [parity][rank]
__global__ void __launch_bounds__(256) reduce_exchange_kernel(XchgArgs a) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < a.n_touched) {
    const int g = a.touched[t];
    double acc = 0.0;
    for (int e = a.cptr[g]; e < a.cptr[g + 1]; ++e) {
      const int4 c = a.cent[e];
      double v = 0.0;
      for (int k = c.y; k < c.z; ++k) v += a.part[a.ridx[k]];
      acc += v;
    }
    const size_t off = ((size_t)(a.epoch & 1) * a.world + a.rank) * a.n_mult + g;
    for (int p = 0; p < a.world; ++p) a.peers[p][off] = acc;
  }
  // last CTA to finish publishes the epoch to every peer
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned done = atomicAdd(a.done, 1u);
    if (done == gridDim.x - 1) {
      __threadfence_system();
      for (int p = 0; p < a.world; ++p) {
        int64_t* flags = reinterpret_cast<int64_t*>(a.peers[p] + (size_t)2 * a.world * a.n_mult);
        st_release_sys_s64(flags + a.rank, a.epoch);
      }
      *a.done = 0u;
    }
  }
}

// wait for every rank's epoch, then q = sum over ranks in rank order
__global__ void __launch_bounds__(256) sum_exchange_kernel(XchgArgs a, double* __restrict__ q) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    const int64_t* flags = reinterpret_cast<const int64_t*>(a.peers[a.rank] + (size_t)2 * a.world * a.n_mult);
    int good = 1;
    for (int r = 0; r < a.world && good; ++r) {
      const long long t0 = clock64();
      while (ld_acquire_sys_s64(flags + r) < a.epoch) {
        __nanosleep(200);
        if (clock64() - t0 > 20000000000LL) {   // ~10 s at 2 GHz: a peer never arrived
          atomicExch(a.error, 1);
          good = 0;
          break;
        }
      }
    }
    ok = good;
  }
  __syncthreads();
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= a.n_mult) return;
  if (!ok) {
    q[g] = __longlong_as_double(0x7ff8000000000000LL);   // NaN: never a stale value
    return;
  }
  const double* slab = a.peers[a.rank] + (size_t)(a.epoch & 1) * a.world * a.n_mult;
  double acc = 0.0;
  for (int r = 0; r < a.world; ++r) acc += slab[(size_t)r * a.n_mult + g];
  q[g] = acc;
}

void launch_exchange(const XchgArgs& a, double* q, cudaStream_t st) {
  const int nb = a.n_touched > 0 ? (a.n_touched + 255) / 256 : 1;
  reduce_exchange_kernel<<<nb, 256, 0, st>>>(a);
  if (a.n_mult > 0) sum_exchange_kernel<<<(a.n_mult + 255) / 256, 256, 0, st>>>(a, q);
}

}  // namespace feti
