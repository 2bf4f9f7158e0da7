// Shared device helpers for the B200 (sm_100a) Lie-closure kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace liecl_b200 {

// FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col). Lowers to one
// SASS DMMA.8x8x4 on sm_100a (tcgen05 has no kind::f64).
// Fragment ownership, lane = 4*g + t:  a = A[g][t], b = B[t][g],
// c = {C[g][2t], C[g][2t+1]}.
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// 16-byte async global->shared copy; src_bytes = 0 zero-fills (tile edges).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Grouped rasterisation of a linear CTA id over an mt x nt tile grid: runs of
// GROUP M-tiles sweep all N-tiles together, so a wave of CTAs streams GROUP
// basis tiles (instead of the whole basis) while the candidate tiles stay in L2.
template <int GROUP>
__device__ __forceinline__ void grouped_tile(int pid, int mt, int nt, int& m_tile, int& n_tile) {
  const int per_group = GROUP * nt;
  const int group = pid / per_group;
  const int first_m = group * GROUP;
  const int size = min(mt - first_m, GROUP);
  const int in_group = pid % per_group;
  m_tile = first_m + in_group % size;
  n_tile = in_group / size;
}

// Cursor pair (l, m), m < l, from its global index g = l(l-1)/2 + m -- the
// order run_engine visits pairs in (R:src/closure.cpp:412-417).
__host__ __device__ __forceinline__ void pair_from_index(int64_t g, int64_t& l, int64_t& m) {
  int64_t ll = static_cast<int64_t>((1.0 + sqrt(1.0 + 8.0 * static_cast<double>(g))) * 0.5);
  while (ll * (ll - 1) / 2 > g) --ll;
  while ((ll + 1) * ll / 2 <= g) ++ll;
  l = ll;
  m = g - ll * (ll - 1) / 2;
}
__host__ __device__ __forceinline__ int64_t pair_index(int64_t l, int64_t m) { return l * (l - 1) / 2 + m; }

} // namespace liecl_b200
