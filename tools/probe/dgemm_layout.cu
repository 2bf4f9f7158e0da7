// Probe: K2b (R = X - V beta, fused weighted norm) with the A operand
// M-contiguous (V as stored, vector-major) vs K-contiguous (a transposed copy).
#include <cstdio>
#include <vector>
#include "../../paper_2506_01120_b200/csrc/dgemm_dmma.cuh"
using namespace liecl_b200;

template <bool KC> float run(int M, int N, int K, const double* A, const double* B, const double* X, double* R,
                             double* part, int reps) {
  auto kern = dgemm_dmma_kernel<KC, REpi::kSubtractNorm>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, rg::smem_bytes<KC>());
  dim3 grid((M + rg::BM - 1) / rg::BM, (N + rg::BN - 1) / rg::BN);
  const int64_t lda = KC ? K : M;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<grid, rg::THREADS, rg::smem_bytes<KC>()>>>(M, N, K, A, lda, B, K, R, M, 1.0, X, M, part, 64, 0, 0);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r)
    kern<<<grid, rg::THREADS, rg::smem_bytes<KC>()>>>(M, N, K, A, lda, B, K, R, M, 1.0, X, M, part, 64, 0, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / reps;
}

int main() {
  const int M = 4096, N = 8192, K = 4096, reps = 10;
  double *A, *B, *X, *R, *part;
  cudaMalloc(&A, sizeof(double) * M * K);
  cudaMalloc(&B, sizeof(double) * K * N);
  cudaMalloc(&X, sizeof(double) * M * N);
  cudaMalloc(&R, sizeof(double) * M * N);
  cudaMalloc(&part, sizeof(double) * (M / 128 + 1) * N);
  cudaMemset(A, 0, sizeof(double) * M * K);
  cudaMemset(B, 0, sizeof(double) * K * N);
  cudaMemset(X, 0, sizeof(double) * M * N);
  const double flops = 2.0 * M * N * K;
  const float mc = run<false>(M, N, K, A, B, X, R, part, reps);
  const float kc = run<true>(M, N, K, A, B, X, R, part, reps);
  printf("{\"m_contiguous_ms\": %.3f, \"m_contiguous_tflops\": %.2f, \"k_contiguous_ms\": %.3f, \"k_contiguous_tflops\": %.2f, \"err\": \"%s\"}\n",
         mc, flops / mc / 1e9, kc, flops / kc / 1e9, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
