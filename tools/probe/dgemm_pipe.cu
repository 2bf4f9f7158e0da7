// Probe: packed projection GEMMs (K2a store, K2b subtract+norm) with the
// per-tile mainloop vs the cross-tile pipelined mainloop, random inputs.
#include <cstdio>
#include "../../paper_2506_01120_b200/csrc/dgemm_dmma.cuh"
using namespace liecl_b200;

__global__ void fill(double* p, size_t n, unsigned long long seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long z = seed + i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    p[i] = (double)((z ^ (z >> 31)) >> 11) * 0x1.0p-53 - 0.5;
  }
}

template <bool KC, REpi E, bool PIPE> float run(int M, int N, int K, const double* A, int64_t lda, const double* B,
                                                 const double* X, double* C, double* part, int reps) {
  auto kern = dgemm_dmma_kernel<KC, E, PIPE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, rg::smem_bytes<KC>());
  dim3 grid((M + rg::BM - 1) / rg::BM, (N + rg::BN - 1) / rg::BN);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w)
    kern<<<grid, rg::THREADS, rg::smem_bytes<KC>()>>>(M, N, K, A, lda, B, K, C, M, 1.0, X, M, part, 64, 0, 0);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r)
    kern<<<grid, rg::THREADS, rg::smem_bytes<KC>()>>>(M, N, K, A, lda, B, K, C, M, 1.0, X, M, part, 64, 0, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

int main() {
  const int M = 4096, N = 8192, K = 4096, reps = 10;
  double *A, *B, *X, *C1, *C2, *part;
  cudaMalloc(&A, sizeof(double) * M * K);
  cudaMalloc(&B, sizeof(double) * K * N);
  cudaMalloc(&X, sizeof(double) * M * N);
  cudaMalloc(&C1, sizeof(double) * M * N);
  cudaMalloc(&C2, sizeof(double) * M * N);
  cudaMalloc(&part, sizeof(double) * (M / 128 + 1) * N);
  fill<<<4096, 256>>>(A, (size_t)M * K, 1);
  fill<<<4096, 256>>>(B, (size_t)K * N, 2);
  fill<<<4096, 256>>>(X, (size_t)M * N, 3);
  const double fl = 2.0 * M * N * K;
  for (int round = 0; round < 2; ++round) {
    float a0 = run<true, REpi::kStoreScaled, false>(M, N, K, A, K, B, X, C1, part, reps);
    float a1 = run<true, REpi::kStoreScaled, true>(M, N, K, A, K, B, X, C2, part, reps);
    float b0 = run<false, REpi::kSubtractNorm, false>(M, N, K, A, M, B, X, C1, part, reps);
    float b1 = run<false, REpi::kSubtractNorm, true>(M, N, K, A, M, B, X, C2, part, reps);
    printf("{\"K2a_ms\": [%.3f, %.3f], \"K2a_tf\": [%.2f, %.2f], \"K2b_ms\": [%.3f, %.3f], \"K2b_tf\": [%.2f, %.2f]}\n",
           a0, a1, fl / a0 / 1e9, fl / a1 / 1e9, b0, b1, fl / b0 / 1e9, fl / b1 / 1e9);
  }
  // identical results (same products, same order)
  run<false, REpi::kSubtractNorm, false>(M, N, K, A, M, B, X, C1, part, 1);
  run<false, REpi::kSubtractNorm, true>(M, N, K, A, M, B, X, C2, part, 1);
  cudaDeviceSynchronize();
  double *h1 = (double*)malloc(sizeof(double) * 1024), *h2 = (double*)malloc(sizeof(double) * 1024);
  cudaMemcpy(h1, C1 + 12345, 8192, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2, C2 + 12345, 8192, cudaMemcpyDeviceToHost);
  int diff = 0;
  for (int i = 0; i < 1024; ++i) diff += h1[i] != h2[i];
  printf("{\"bitwise_diffs\": %d, \"err\": \"%s\"}\n", diff, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
