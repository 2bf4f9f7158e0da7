// Device-resident closure for small operators: the whole cursor loop of
// run_engine (R:src/closure.cpp:378-460) in ONE thread block with the basis,
// the originals and the projection coefficients in shared memory, using the
// reference's sequential semantics (every verdict is CGS2 against the basis
// as it stands -- what the row speculation of :427-444 reproduces).
// Latency-bound closures such as config 0 (d = 8: 36 brackets) pay one launch
// and no host round trip. Used when (cap + 1) basis slots (x2 for Alg. 3)
// fit in shared memory; everything larger runs on the batched engine.
#pragma once

#include "../../include/liecl_b200.h"
#include "common.cuh"

namespace liecl_b200 {

struct TinyState {
  int64_t n_o, n_b;     // orthonormal / commutator-basis sizes
  int64_t g_next;       // pairs processed
  uint64_t commutators, checks, accepted;
  int64_t log_len;
  int32_t status;       // 0 finished, 2 capacity exceeded
  int32_t pad;
};

constexpr int kTinySmemLimit = 200 * 1024;

// dynamic shared memory bytes for d, slots, keep (0 if it does not fit)
inline size_t tiny_smem_bytes(int d, int64_t slots, bool keep) {
  const size_t D2 = static_cast<size_t>(d) * d;
  const size_t bytes = (slots * D2 * (keep ? 2 : 1) + 2 * D2 + slots) * sizeof(double2) + 32 * sizeof(double);
  return bytes <= static_cast<size_t>(kTinySmemLimit) ? bytes : 0;
}

inline int tiny_threads(int d) {
  const int D2 = d * d;
  return std::min(512, std::max(64, (D2 + 31) / 32 * 32));
}

__device__ __forceinline__ double tiny_block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < nw; ++w) s += red[w];  // fixed order: deterministic
  return s;
}

__global__ void tiny_closure_kernel(const double2* __restrict__ gens, int ngens, int d, double tol, int64_t cap,
                                    int keep, int64_t slots, double2* __restrict__ V_out,
                                    double2* __restrict__ O_out, TinyState* __restrict__ st,
                                    liecl_b200_decision* __restrict__ log, int64_t log_cap) {
  extern __shared__ __align__(16) double2 tsm[];
  const int D2 = d * d;
  double2* V = tsm;                                  // slots x D2
  double2* O = keep ? V + slots * D2 : V;            // originals (Alg. 3)
  double2* h = (keep ? O + slots * D2 : V + slots * D2);
  double2* r = h + D2;
  double2* beta = r + D2;                            // slots
  double* red = reinterpret_cast<double*>(beta + slots);
  const int T = blockDim.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = T >> 5;
  const double sqrt_d = sqrt(static_cast<double>(d)), inv_d = 1.0 / d;
  int64_t n_o = 0, n_b = 0, nlog = 0;
  uint64_t commutators = 0, checks = 0, accepted = 0;
  int status = 0;

  auto record = [&](int64_t l, int64_t m, int nul, int ind, double rn) {
    if (threadIdx.x == 0 && nlog < log_cap) log[nlog] = liecl_b200_decision{l, m, nul, ind, 0, 0, rn};
    ++nlog;
  };
  auto norm_of = [&](const double2* x) {
    double s = 0.0;
    for (int k = threadIdx.x; k < D2; k += T) s += x[k].x * x[k].x + x[k].y * x[k].y;
    return sqrt(tiny_block_sum(s, red)) / sqrt_d;
  };
  // one CGS pass of r against V[0:n_o] (R:src/closure.cpp:149-160)
  auto pass = [&]() {
    for (int64_t j = warp; j < n_o; j += nw) {
      const double2* v = V + j * D2;
      double re = 0.0, im = 0.0;
      for (int k = lane; k < D2; k += 32) {
        const double2 a = v[k], b = r[k];
        re += a.x * b.x + a.y * b.y;
        im += a.x * b.y - a.y * b.x;
      }
      re = warp_sum(re);
      im = warp_sum(im);
      if (lane == 0) beta[j] = make_double2(re * inv_d, im * inv_d);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < D2; k += T) {
      double2 acc = r[k];
#pragma unroll 4
      for (int64_t j = 0; j < n_o; ++j) {
        const double2 b = beta[j], v = V[j * D2 + k];
        acc.x -= b.x * v.x - b.y * v.y;
        acc.y -= b.x * v.y + b.y * v.x;
      }
      r[k] = acc;
    }
    __syncthreads();
  };
  // verdict of the unit candidate in h; appends on acceptance (R:src/closure.cpp:276-293)
  auto check_and_apply = [&](int64_t l, int64_t m) -> bool {
    for (int k = threadIdx.x; k < D2; k += T) r[k] = h[k];
    __syncthreads();
    if (n_o > 0) {
      pass();
      pass();
    }
    const double rn = norm_of(r);
    const bool ind = rn > tol;
    ++checks;
    record(l, m, 0, ind, rn);
    if (ind) {
      if ((keep ? n_b : n_o) >= cap) return false;
      const double s = 1.0 / rn;
      for (int k = threadIdx.x; k < D2; k += T) {
        const double2 v = r[k];
        V[n_o * D2 + k] = make_double2(v.x * s, v.y * s);
        if (keep) O[n_b * D2 + k] = h[k];
      }
      ++n_o;
      n_b = keep ? n_b + 1 : n_o;
      ++accepted;
    }
    __syncthreads();
    return true;
  };

  for (int i = 0; i < ngens && status == 0; ++i) {  // generator loop (R:src/closure.cpp:378-403)
    const double2* g = gens + static_cast<int64_t>(i) * D2;
    for (int k = threadIdx.x; k < D2; k += T) h[k] = g[k];
    __syncthreads();
    const double gn = norm_of(h);
    if (gn <= tol) {
      record(i, -1, 1, 0, gn);
      continue;
    }
    const double s = 1.0 / gn;
    for (int k = threadIdx.x; k < D2; k += T) h[k] = make_double2(h[k].x * s, h[k].y * s);
    __syncthreads();
    if (!check_and_apply(i, -1)) status = 2;
  }
  int64_t g = 0;
  for (int64_t l = 1; status == 0 && l < n_b; ++l) {  // cursor loop (R:src/closure.cpp:412-460)
    for (int64_t m = 0; m < l; ++m, ++g) {
      const double2* A = O + l * D2;  // commutator basis (O == V unless Alg. 3)
      const double2* B = O + m * D2;
      for (int e = threadIdx.x; e < D2; e += T) {
        const int i = e % d, j = e / d;
        double re = 0.0, im = 0.0;
        for (int k = 0; k < d; ++k) {
          const double2 aik = A[i + k * d], bkj = B[k + j * d], bik = B[i + k * d], akj = A[k + j * d];
          re += (aik.x * bkj.x - aik.y * bkj.y) - (bik.x * akj.x - bik.y * akj.y);
          im += (aik.x * bkj.y + aik.y * bkj.x) - (bik.x * akj.y + bik.y * akj.x);
        }
        h[e] = make_double2(re, im);
      }
      __syncthreads();
      ++commutators;
      const double hn = norm_of(h);
      if (!(hn > tol)) {
        record(l, m, 1, 0, 0.0);
        continue;
      }
      const double s = 1.0 / hn;
      for (int k = threadIdx.x; k < D2; k += T) h[k] = make_double2(h[k].x * s, h[k].y * s);
      __syncthreads();
      if (!check_and_apply(l, m)) {
        status = 2;
        break;
      }
    }
  }
  for (int64_t k = threadIdx.x; k < n_o * D2; k += T) V_out[k] = V[k];
  if (keep)
    for (int64_t k = threadIdx.x; k < n_b * D2; k += T) O_out[k] = O[k];
  if (threadIdx.x == 0) {
    st->n_o = n_o;
    st->n_b = n_b;
    st->g_next = g;
    st->commutators = commutators;
    st->checks = checks;
    st->accepted = accepted;
    st->log_len = nlog;
    st->status = status;
  }
}

} // namespace liecl_b200
