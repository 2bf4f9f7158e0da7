// Small HBM-bound kernels around the projection GEMMs: norm finalisation,
// survivor gather, the Gram-Schmidt append (K3) and generator normalisation.
#pragma once

#include "common.cuh"

namespace liecl_b200 {

// rn[b] = sqrt(sum_mt partial[mt*N + b]) / sqrt(d)   (dense_norm, R:src/dense.cpp:61-63)
// Summation over M tiles in fixed order: deterministic across runs.
// sqrt_d <= 0 stores the raw sum (a D-shard's partial, summed over ranks
// before the square root). rn may alias partial when mtiles == 1.
__global__ void norm_finalize_kernel(const double* partial, int mtiles, int N, double sqrt_d, double* rn) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= N) return;
  double s = 0.0;
  for (int mt = 0; mt < mtiles; ++mt) s += partial[static_cast<int64_t>(mt) * N + b];
  rn[b] = sqrt_d > 0.0 ? sqrt(s) / sqrt_d : s;
}

// dst[j] = src[idx[j]] for D-element complex columns.
__global__ void gather_columns_kernel(const double2* __restrict__ src, const int* __restrict__ idx,
                                      int64_t D, double2* __restrict__ dst) {
  const int j = blockIdx.y;
  const double2* s = src + static_cast<int64_t>(idx[j]) * D;
  double2* o = dst + static_cast<int64_t>(j) * D;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < D;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    o[e] = s[e];
}

// from_pauli (R:src/dense.cpp:70-98) on the device, bit-exact: one thread per
// column s of each operator; terms (already sorted by (z, x) as PauliSum keeps
// them) are added in order with the reference's exact phase moves, so every
// entry accumulates the same values in the same order.
__device__ __forceinline__ uint64_t reverse_low_bits_dev(uint64_t v, int n) {
  return __brevll(v) >> (64 - n);
}
__global__ void from_pauli_kernel(const int64_t* __restrict__ offsets, const uint64_t* __restrict__ x,
                                  const uint64_t* __restrict__ z, const double2* __restrict__ coef, int count,
                                  int qubits, double2* __restrict__ out) {
  const int64_t d = int64_t(1) << qubits;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < count * d;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = idx / d;
    const uint64_t s = static_cast<uint64_t>(idx % d);
    double2* col = out + c * d * d + static_cast<int64_t>(s) * d;
    for (int64_t r = 0; r < d; ++r) col[r] = make_double2(0.0, 0.0);
    for (int64_t t = offsets[c]; t < offsets[c + 1]; ++t) {
      const uint64_t xi = reverse_low_bits_dev(x[t], qubits), zi = reverse_low_bits_dev(z[t], qubits);
      double2 v = coef[t];
      switch (__popcll(x[t] & z[t]) & 3) {  // Hermitian phase i^{#Y}
      case 1: v = make_double2(-v.y, v.x); break;
      case 2: v = make_double2(-v.x, -v.y); break;
      case 3: v = make_double2(v.y, -v.x); break;
      default: break;
      }
      if (__popcll(zi & s) & 1) v = make_double2(-v.x, -v.y);
      double2& e = col[s ^ xi];
      e = make_double2(__dadd_rn(e.x, v.x), __dadd_rn(e.y, v.y));
    }
  }
}

// restrict_to_subspace with the zero-magnetization projector (R:src/dense.cpp:
// 167-199): B^H A B for a 0/1 column-selection basis B is the submatrix
// A(s_i, s_j) over the selected basis states s (ascending). count operators,
// full dimension d, m selected states.
__global__ void restrict_states_kernel(const double2* __restrict__ A, int64_t count, int64_t d,
                                       const int64_t* __restrict__ states, int64_t m, double2* __restrict__ out) {
  const int64_t mm = m * m;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < count * mm;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / mm, k = e % mm, i = k % m, j = k / m;
    out[e] = A[c * d * d + states[j] * d + states[i]];
  }
}

// dst[j] = src[idx[j]] for columns of W doubles (either field).
__global__ void gather_words_kernel(const double* __restrict__ src, const int* __restrict__ idx, int64_t W,
                                    double* __restrict__ dst) {
  const int j = blockIdx.y;
  const double* s = src + static_cast<int64_t>(idx[j]) * W;
  double* o = dst + static_cast<int64_t>(j) * W;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < W;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    o[e] = s[e];
}

// K3 append: dst = (s + 0i) * src  -- residual_unit = Complex{1/||r||, 0} * r
// (R:src/closure.cpp:283) written straight into the basis slab slot; with
// `orig_dst` the accepted candidate h_unit is copied to the originals slab
// (Alg. 3 keep_original, R:src/closure.cpp:288-293).
__global__ void append_scaled_kernel(const double2* __restrict__ src, double s, int64_t D,
                                     double2* __restrict__ dst, const double2* __restrict__ orig_src,
                                     double2* __restrict__ orig_dst) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < D;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double2 v = src[e];
    dst[e] = make_double2(v.x * s - v.y * 0.0, v.x * 0.0 + v.y * s);
    if (orig_dst) orig_dst[e] = orig_src[e];
  }
}

// Per-column squared norms of `count` D-element columns, one CTA per column,
// fixed-order tree reduction (deterministic). out[j] = sqrt(sum)/sqrt_d.
__global__ void column_norm_kernel(const double2* __restrict__ x, int64_t D, double sqrt_d,
                                   double* __restrict__ out) {
  __shared__ double red[32];
  const double2* c = x + static_cast<int64_t>(blockIdx.x) * D;
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < D; e += blockDim.x) s += c[e].x * c[e].x + c[e].y * c[e].y;
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) out[blockIdx.x] = sqrt_d > 0.0 ? sqrt(v) / sqrt_d : v;  // <= 0: raw sum
  }
}

// Generator normalisation: g_unit = Complex{1/||g||, 0} * g (R:src/closure.cpp:388),
// null generators (||g|| <= tol) produce zeros and are skipped by the host.
__global__ void scale_columns_kernel(const double2* __restrict__ x, const double* __restrict__ nrm, double tol,
                                     int64_t D, double2* __restrict__ out) {
  const int j = blockIdx.y;
  const double n = nrm[j];
  const double s = n > tol ? 1.0 / n : 0.0;
  const double2* c = x + static_cast<int64_t>(j) * D;
  double2* o = out + static_cast<int64_t>(j) * D;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < D;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double2 v = c[e];
    o[e] = make_double2(v.x * s - v.y * 0.0, v.x * 0.0 + v.y * s);
  }
}

} // namespace liecl_b200
