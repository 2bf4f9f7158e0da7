// Probe: packed projection GEMMs with the 128x64 CTA tile (64x32 per warp,
// 2 CTAs/SM) vs a 64x64 tile (32x32 per warp, 3 CTAs/SM), random inputs.
#include <cstdio>
#include "../../paper_2506_01120_b200/csrc/dgemm_dmma.cuh"
#include "dgemm64_variant.cuh"
using namespace liecl_b200;

__global__ void fill(double* p, size_t n, unsigned long long seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long z = seed + i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    p[i] = (double)((z ^ (z >> 31)) >> 11) * 0x1.0p-53 - 0.5;
  }
}

template <class F> float timeit(F launch, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  launch();
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch();
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
  cudaMalloc(&part, sizeof(double) * (M / 64 + 1) * N);
  fill<<<4096, 256>>>(A, (size_t)M * K, 1);
  fill<<<4096, 256>>>(B, (size_t)K * N, 2);
  fill<<<4096, 256>>>(X, (size_t)M * N, 3);
  auto k128a = dgemm_dmma_kernel<true, REpi::kStoreScaled>;
  auto k128b = dgemm_dmma_kernel<false, REpi::kSubtractNorm>;
  auto k64a = dgemm_dmma_kernel64<true, REpi::kStoreScaled>;
  auto k64b = dgemm_dmma_kernel64<false, REpi::kSubtractNorm>;
  cudaFuncSetAttribute(k128a, cudaFuncAttributeMaxDynamicSharedMemorySize, rg::smem_bytes<true>());
  cudaFuncSetAttribute(k128b, cudaFuncAttributeMaxDynamicSharedMemorySize, rg::smem_bytes<false>());
  cudaFuncSetAttribute(k64a, cudaFuncAttributeMaxDynamicSharedMemorySize, rg64::smem_bytes<true>());
  cudaFuncSetAttribute(k64b, cudaFuncAttributeMaxDynamicSharedMemorySize, rg64::smem_bytes<false>());
  int occ128 = 0, occ64 = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ128, k128a, rg::THREADS, rg::smem_bytes<true>());
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ64, k64a, rg64::THREADS, rg64::smem_bytes<true>());
  dim3 g128((M + 127) / 128, N / 64), g64((M + 63) / 64, N / 64);
  const double fl = 2.0 * M * N * K;
  for (int round = 0; round < 2; ++round) {
    float a128 = timeit([&] { k128a<<<g128, rg::THREADS, rg::smem_bytes<true>()>>>(M, N, K, A, K, B, K, C1, M, 1.0, X, M, part, 64, 0, 0); }, reps);
    float a64 = timeit([&] { k64a<<<g64, rg64::THREADS, rg64::smem_bytes<true>()>>>(M, N, K, A, K, B, K, C2, M, 1.0, X, M, part, 64, 0, 0); }, reps);
    float b128 = timeit([&] { k128b<<<g128, rg::THREADS, rg::smem_bytes<false>()>>>(M, N, K, A, M, B, K, C1, M, 1.0, X, M, part, 64, 0, 0); }, reps);
    float b64 = timeit([&] { k64b<<<g64, rg64::THREADS, rg64::smem_bytes<false>()>>>(M, N, K, A, M, B, K, C2, M, 1.0, X, M, part, 64, 0, 0); }, reps);
    printf("{\"occupancy\": [%d, %d], \"K2a_tf\": [%.2f, %.2f], \"K2b_tf\": [%.2f, %.2f]}\n", occ128, occ64,
           fl / a128 / 1e9, fl / a64 / 1e9, fl / b128 / 1e9, fl / b64 / 1e9);
  }
  cudaDeviceSynchronize();
  printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
