// Exclusive prefix sums for the PauliSum engine (run and keep positions,
// product offsets): per-1024 block scans (warp shuffles + one shared-memory
// pass over the warp totals), the block totals scanned recursively in place,
// block offsets added back. Any n; 2L - 1 launches for L levels (n <= 1M: 3).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace liecl_b200 {
namespace scan {

constexpr int kBlock = 1024;

template <class T> __device__ __forceinline__ T block_exclusive(T v, T* s_warp, T& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    T w = lane < static_cast<int>(blockDim.x >> 5) ? s_warp[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    s_warp[lane] = w;  // inclusive prefix of the warp totals
  }
  __syncthreads();
  total = s_warp[(blockDim.x >> 5) - 1];
  return (warp > 0 ? s_warp[warp - 1] : T(0)) + x - v;
}

// out[i] = exclusive prefix of in[] within its block; sums[b] = block b's total.
// in == out is allowed (each thread reads its element before writing it).
template <class T>
__global__ void __launch_bounds__(kBlock) blocks_kernel(const T* in, int64_t n, T* out, T* __restrict__ sums) {
  __shared__ T s_warp[32];
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x;
  T total;
  const T e = block_exclusive<T>(i < n ? in[i] : T(0), s_warp, total);
  if (i < n) out[i] = e;
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

template <class T> __global__ void add_kernel(T* __restrict__ out, int64_t n, const T* __restrict__ sums) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && i >= kBlock) out[i] += sums[i / kBlock];
}

// workspace elements for n inputs: the block totals of every level
inline int64_t workspace(int64_t n) {
  int64_t w = 0;
  for (;;) {
    const int64_t nb = (n + kBlock - 1) / kBlock;
    w += nb;
    if (nb <= 1) return w;
    n = nb;
  }
}

// out = exclusive prefix sums of in (n >= 1); ws holds workspace(n) elements.
// Returns the device address of the grand total (inside ws); `launches` counts
// the kernels issued.
template <class T> T* exclusive(const T* in, T* out, int64_t n, T* ws, cudaStream_t stream, int& launches) {
  const int64_t nb = (n + kBlock - 1) / kBlock;
  blocks_kernel<T><<<static_cast<unsigned>(nb), kBlock, 0, stream>>>(in, n, out, ws);
  ++launches;
  if (nb == 1) return ws;
  T* total = exclusive<T>(ws, ws, nb, ws + nb, stream, launches);  // block offsets, in place
  add_kernel<T><<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(out, n, ws);
  ++launches;
  return total;
}

}  // namespace scan
}  // namespace liecl_b200
