// Micro-benchmark of the 128x128 tile Cholesky + inverse (potrf_invert_128)
// used by the device factorizations.  Not part of the product: build with
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//        -I paper_2502_08382_b200/csrc scripts/potrf_bench.cu -o /tmp/potrf_bench
// and run on a B200: prints us per launch of NT tiles and the max errors of
// L L^T - A and L Y - I.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "feti_common.cuh"
#include "feti_dense128.cuh"

using namespace feti;

__global__ void __launch_bounds__(256, 1) bench_kernel(double* tiles, double* dinv, int* bad) {
  extern __shared__ double sm[];
  potrf_invert_128(tiles + (size_t)blockIdx.x * TILE, dinv + (size_t)blockIdx.x * TILE, bad, 0, sm);
}

static inline double& at(std::vector<double>& t, int row, int col) { return t[swz(col, row)]; }

int main(int argc, char** argv) {
  const int NT = argc > 1 ? atoi(argv[1]) : 256;
  std::vector<double> A((size_t)TILE);
  // SPD test matrix: diagonally dominant with structure
  srand(1);
  std::vector<double> M(128 * 128);
  for (auto& v : M) v = (rand() / (double)RAND_MAX) - 0.5;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 128; ++j) {
      double s = 0;
      for (int k = 0; k < 128; ++k) s += M[i * 128 + k] * M[j * 128 + k];
      at(A, i, j) = s + (i == j ? 1.0 : 0.0);
    }
  std::vector<double> h((size_t)NT * TILE);
  for (int t = 0; t < NT; ++t) std::copy(A.begin(), A.end(), h.begin() + (size_t)t * TILE);
  double *d_t, *d_d;
  int* d_bad;
  cudaMalloc(&d_t, h.size() * 8);
  cudaMalloc(&d_d, h.size() * 8);
  cudaMalloc(&d_bad, 4);
  const size_t smem = POTRF_SMEM_DOUBLES * sizeof(double);
  cudaFuncSetAttribute(bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaMemcpy(d_t, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    int big = 1 << 30;
    cudaMemcpy(d_bad, &big, 4, cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    bench_kernel<<<NT, 256, smem>>>(d_t, d_d, d_bad);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaError_t err = cudaGetLastError();
  std::vector<double> L(TILE), Y(TILE);
  cudaMemcpy(L.data(), d_t, TILE * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(Y.data(), d_d, TILE * 8, cudaMemcpyDeviceToHost);
  double e_llt = 0, e_ly = 0, anorm = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = 0, p = 0;
      for (int k = 0; k <= j; ++k) s += at(L, i, k) * at(L, j, k);
      for (int k = j; k <= i; ++k) p += at(L, i, k) * at(Y, k, j);
      e_llt = fmax(e_llt, fabs(s - at(A, i, j)));
      e_ly = fmax(e_ly, fabs(p - (i == j ? 1.0 : 0.0)));
      anorm = fmax(anorm, fabs(at(A, i, j)));
    }
  printf("%s  NT=%d  %.1f us/launch  %.2f us/tile-wave  max|LL^T-A|/max|A| = %.2e  max|LY-I| = %.2e\n",
         cudaGetErrorString(err), NT, best * 1e3, best * 1e3 / ((NT + 147) / 148), e_llt / anorm, e_ly);
  return 0;
}
