// Probe: how much DMMA issue time a scalar FP64 instruction costs on sm_100a.
// Each warp runs a loop of 32 DMMA.8x8x4 (16 accumulator pairs) plus K scalar
// FP64 negations of the A operands (as the commutator's main loop has) per
// trip, 8 warps per CTA, 2 CTAs per SM; the same with the sign flipped on the
// integer pipe. Prints the DMMA rate each mix sustains.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o fp64_mix fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int K, bool INT_FLIP>
__global__ void __launch_bounds__(256, 2) mix_kernel(double* out, int trips, double seed) {
  double c[16][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i][0] = c[i][1] = 0.0;
  double a[8], b = seed + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed * (i + 1) + threadIdx.x;
  for (int t = 0; t < trips; ++t) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i < K) {
        if (INT_FLIP) {
          long long v = __double_as_longlong(a[i]) ^ (1ll << 63);
          a[i] = __longlong_as_double(v);
        } else {
          asm volatile("add.f64 %0, %0, %1;\n" : "+d"(a[i]) : "d"(seed));
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int i = 0; i < 16; ++i) dmma(c[i][0], c[i][1], a[(i + r) & 7], b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * 256 + threadIdx.x] = s;
}

template <int K, bool INT_FLIP> void run(const char* name) {
  double* out;
  cudaMalloc(&out, 296 * 256 * 8);
  const int trips = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int it = 0; it < 4; ++it) {
    cudaEventRecord(e0);
    mix_kernel<K, INT_FLIP><<<296, 256>>>(out, trips, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it && ms < best) best = ms;
  }
  const double tf = 296.0 * 8 * trips * 32 * 512 / (best * 1e-3) / 1e12;
  printf("{\"variant\": \"%s\", \"scalar_fp64_per_32_dmma\": %d, \"ms\": %.3f, \"dmma_tflops\": %.2f}\n", name, K, best, tf);
  cudaFree(out);
}

int main() {
  run<0, false>("dmma_only");
  run<1, false>("neg_f64_1");
  run<2, false>("neg_f64_2");
  run<4, false>("neg_f64_4");
  run<8, false>("neg_f64_8");
  run<4, true>("int_flip_4");
  run<8, true>("int_flip_8");
  return 0;
}
