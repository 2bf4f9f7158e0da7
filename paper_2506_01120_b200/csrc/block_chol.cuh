// In-block decisions from the Gram matrix of the block (the
// re-check rule of R:src/closure.cpp:440-444), replacing the per-survivor
// grid-synchronised walk of block_gs.cuh on the common path.
//
// A block holds up to 64 survivors y_0..y_{nb-1} (residuals already
// re-projected against everything accepted before the block, norms rn2). In
// cursor order, survivor q is decided from rn2_q when nothing was accepted
// earlier in the block, else from its CGS2 residual against the block's
// earlier accepts. With G = <y_i, y_j> (one GEMM) that residual's square is
// the Schur complement s_q = G_qq - sum_a |Z_aq|^2 of a Cholesky factor grown
// one accept at a time (Z = R of the QR of the accepted survivors, extended to
// every later column): O(64^2) work per accept in one CTA.
//
// s_q is exact to ~eps * G_qq, so it CERTIFIES an accept when s_q clears
// 1e-2 G_qq and (100 tol)^2 -- the residual is then far above tol, not
// borderline, and the accepted set well conditioned. A smaller s_q cannot separate 1e-15 from 1e-9: the survivor is
// a TENTATIVE reject, confirmed afterwards by its explicit CGS2 residual
// against exactly the accepts before it (a masked two-pass projection); if
// any explicit residual exceeds tol, the caller redoes the block with the
// exact per-survivor kernel. The accepted vectors are formed by CholQR2 --
// W = Y_A R1^-1, then Q = W R2^-1 with R2 from the Cholesky of W^H W (the
// triangular inverses in one CTA, the products as DMMA GEMMs) --
// the same Q as sequential Gram-Schmidt up to eps * cond (orthonormal to
// eps), and residual norms R2_aa * R1_aa. Included by engine.cu (namespace
// liecl_b200 helpers; anonymous-namespace users in dense_engine.cuh).
#pragma once

#include "common.cuh"

namespace liecl_b200 {

constexpr int kBcMax = 64;  // survivors per block (== kBlockGsMax)

// scalar helpers: double (packed anti-Hermitian field: real Gram) or double2
__device__ __forceinline__ double bc_conj(double a) { return a; }
__device__ __forceinline__ double2 bc_conj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double bc_mul(double a, double b) { return a * b; }
__device__ __forceinline__ double2 bc_mul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double bc_sub(double a, double b) { return a - b; }
__device__ __forceinline__ double2 bc_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double bc_scale(double a, double s) { return a * s; }
__device__ __forceinline__ double2 bc_scale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double bc_abs2(double a) { return a * a; }
__device__ __forceinline__ double bc_abs2(double2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ double bc_re(double a) { return a; }
__device__ __forceinline__ double bc_re(double2 a) { return a.x; }
template <class T> __device__ __forceinline__ T bc_zero();
template <> __device__ __forceinline__ double bc_zero<double>() { return 0.0; }
template <> __device__ __forceinline__ double2 bc_zero<double2>() { return make_double2(0.0, 0.0); }
template <class T> __device__ __forceinline__ T bc_one();
template <> __device__ __forceinline__ double bc_one<double>() { return 1.0; }
template <> __device__ __forceinline__ double2 bc_one<double2>() { return make_double2(1.0, 0.0); }

// The one-CTA kernels below give every column four lanes (kBcThreads =
// 4 kBcMax): a column's dot products are split over its lanes (k = sub, sub+4,
// ...) and summed with two shuffles, so a sequential step costs ~a/4 dependent
// multiply-adds instead of ~a.
constexpr int kBcLanes = 4, kBcThreads = kBcLanes * kBcMax;
// (groups take branches as a whole; the shuffles name only the group's lanes)
__device__ __forceinline__ unsigned bc_group_mask() { return 0xFu << (threadIdx.x & 28); }
__device__ __forceinline__ double bc_group_sum(double v) {
  const unsigned m = bc_group_mask();
  v += __shfl_xor_sync(m, v, 1);
  return v + __shfl_xor_sync(m, v, 2);
}
__device__ __forceinline__ double2 bc_group_sum(double2 v) { return make_double2(bc_group_sum(v.x), bc_group_sum(v.y)); }

struct BcDecision {
  int nacc;          // accepts in the block
  int ntent;         // tentative rejects (explicit check pending)
  int cap_hit;       // survivor whose accept exceeds the cap (-1 none)
  int acc[kBcMax];   // accepted survivors, in order
  int tent[kBcMax];  // tentative rejects, in order
  int tent_before[kBcMax];  // accepts before each tentative reject
};

// One CTA of kBcMax threads: sequential decisions over the block (thread t
// owns column t of Z and s). G: nb x nb, G[i + j*ldg] = <y_i, y_j>. Outputs
// flags (bit 0 independent, 1 re-checked, 2 tentative), rn (decided
// survivors: rn2, or sqrt(s) for certified accepts -- replaced by the CholQR2
// norm later), R1 (accepted x accepted upper factor, ld kBcMax) and `dec`.
template <class T>
__global__ void __launch_bounds__(kBcThreads) bc_decide_kernel(const T* __restrict__ G, int ldg, int nb,
                                                            const double* __restrict__ rn2, double tol,
                                                            int cap_left, int* __restrict__ flags,
                                                            double* __restrict__ rn, T* __restrict__ R1,
                                                            BcDecision* __restrict__ dec) {
  extern __shared__ __align__(16) unsigned char bc_smem[];
  // Z(a, q) = Zs[a * kBcMax + q] and G(i, j) = Gs[i + j * kBcMax]: 2 kBcMax^2 T
  // (dynamic; G staged once -- every step then runs out of shared memory).
  // Flat indexing: the 2-D array-pointer form miscompiled here (a loop-entry
  // register read before its first write in the SASS of nvcc 12.9 / sm_100a;
  // tools/probe/bc_kernels_test.cu)
  T* Zs = reinterpret_cast<T*>(bc_smem);
  T* Gs = Zs + kBcMax * kBcMax;
  __shared__ double s[kBcMax];
  __shared__ double s_rn2[kBcMax];  // rn2 staged: thread 0's serial decisions read shared memory only
  __shared__ int acc_list[kBcMax];
  __shared__ int s_ind, s_stop;
  const int tid = threadIdx.x;
  const int t = tid >> 2, sub = tid & 3;  // column t, lane sub of its group
  for (int e = tid; e < nb * nb; e += blockDim.x) Gs[(e % nb) + (e / nb) * kBcMax] = G[(e % nb) + static_cast<int64_t>(e / nb) * ldg];
  __syncthreads();
  if (sub == 0 && t < nb) {
    s[t] = bc_re(Gs[t + t * kBcMax]);
    s_rn2[t] = rn2[t];
  }
  int acc = 0, tent = 0;
  if (tid == 0) dec->cap_hit = -1;
  __syncthreads();
  for (int q = 0; q < nb; ++q) {
    if (tid == 0) {
      const double r2 = s_rn2[q];
      const bool recheck = acc > 0 && r2 > tol;
      int ind;
      int fl = recheck ? 2 : 0;
      double r = r2;
      if (!recheck) {
        ind = r2 > tol ? 1 : 0;
      } else {
        const double gqq = bc_re(Gs[q + q * kBcMax]);
        const double sq = s[q];
        // certified: the residual keeps >= 10% of the survivor's norm (so the
        // accepted set stays well conditioned, cond <= ~100 per step, and
        // CholQR2 reproduces sequential Gram-Schmidt to ~eps * cond) and is far
        // above tol; anything else is decided explicitly
        // (survivors are residuals of unit candidates, G_qq <= ~1: G_qq >= 1e-6
        // keeps the accepted columns within a few decades of each other)
        ind = (sq > 1e-2 * gqq && gqq > 1e-6 && sq > (100.0 * tol) * (100.0 * tol)) ? 1 : 0;
        r = sqrt(fmax(sq, 0.0));
        if (!ind) {  // tentative: confirmed by an explicit residual
          fl |= 4;
          dec->tent[tent] = q;
          dec->tent_before[tent] = acc;
          ++tent;
        }
      }
      s_stop = 0;
      if (ind && acc >= cap_left) {
        dec->cap_hit = q;
        s_stop = 1;
      }
      flags[q] = fl | ind;
      rn[q] = r;
      s_ind = ind;
    }
    __syncthreads();
    if (s_stop) break;
    if (s_ind) {
      // row `acc` of Z: the new accept's R entries against every later column
      const double lqq = sqrt(s[q]);  // == rn2_q for the block's first accept
      if (tid == 0) acc_list[acc] = q;
      if (t > q && t < nb) {  // whole 4-lane groups: the shuffles stay inside active lanes
        T part = bc_zero<T>();
        for (int a = sub; a < acc; a += kBcLanes) part = bc_sub(part, bc_mul(bc_conj(Zs[a * kBcMax + q]), Zs[a * kBcMax + t]));
        part = bc_group_sum(part);
        if (sub == 0) {
          const T z = bc_scale(bc_sub(Gs[q + t * kBcMax], bc_scale(part, -1.0)), 1.0 / lqq);
          Zs[acc * kBcMax + t] = z;
          s[t] -= bc_abs2(z);
        }
      }
      if (tid == 0) {  // the diagonal (real, positive); no thread reads row `acc` in this phase
        if constexpr (sizeof(T) == sizeof(double)) Zs[acc * kBcMax + q] = lqq;
        else Zs[acc * kBcMax + q] = T{lqq, 0.0};
      }
      ++acc;
      __syncthreads();
    }
  }
  __syncthreads();
  // R1[a'][a] = Z[a'][q_a] (upper triangular, ld kBcMax)
  for (int e = tid; e < acc * acc; e += blockDim.x) {
    const int ap = e % acc, a = e / acc;
    R1[ap + a * kBcMax] = ap <= a ? Zs[ap * kBcMax + acc_list[a]] : bc_zero<T>();
  }
  if (tid < acc) dec->acc[tid] = acc_list[tid];
  if (tid == 0) {
    dec->nacc = acc;
    dec->ntent = tent;
  }
}

// Cholesky G = R^H R (upper R, ld kBcMax) of an a x a Hermitian matrix
// (a <= 64), one CTA; diag[a] receives R_aa. Right-looking: step i reads row i
// of the current Schur complement (every thread recomputes R_ii), writes R's
// row i and takes conj(R_iu) R_iv off the trailing upper triangle -- one
// barrier per step, every thread's work independent.
template <class T>
__global__ void __launch_bounds__(kBcThreads) bc_cholesky_kernel(const T* __restrict__ G, int ldg, int a,
                                                                  T* __restrict__ R, double* __restrict__ diag) {
  extern __shared__ __align__(16) unsigned char bc_smem[];
  T* Rs = reinterpret_cast<T*>(bc_smem);  // R(i, j) = Rs[i * kBcMax + j]: kBcMax^2 T (dynamic), flat (see above)
  T* Gs = Rs + kBcMax * kBcMax;            // G staged in shared memory, then its Schur complements
  const int tid = threadIdx.x;
  for (int e = tid; e < a * a; e += blockDim.x) Gs[(e % a) + (e / a) * kBcMax] = G[(e % a) + static_cast<int64_t>(e / a) * ldg];
  __syncthreads();
  for (int i = 0; i < a; ++i) {
    const double r = sqrt(fmax(bc_re(Gs[i + i * kBcMax]), 0.0));
    const double ir = 1.0 / r;
    for (int j = i + tid; j < a; j += blockDim.x) {
      if (j == i) {
        if constexpr (sizeof(T) == sizeof(double)) Rs[i * kBcMax + i] = r;
        else Rs[i * kBcMax + i] = T{r, 0.0};
        diag[i] = r;
      } else {
        Rs[i * kBcMax + j] = bc_scale(Gs[i + j * kBcMax], ir);
      }
    }
    const int m = a - i - 1;
    for (int e = tid; e < m * m; e += blockDim.x) {
      const int u = i + 1 + e % m, v = i + 1 + e / m;
      if (u > v) continue;
      const T ru = bc_scale(Gs[i + u * kBcMax], ir), rv = bc_scale(Gs[i + v * kBcMax], ir);
      Gs[u + v * kBcMax] = bc_sub(Gs[u + v * kBcMax], bc_mul(bc_conj(ru), rv));
    }
    __syncthreads();
  }
  for (int e = tid; e < a * a; e += blockDim.x) {
    const int i = e % a, j = e / a;
    R[i + j * kBcMax] = i <= j ? Rs[i * kBcMax + j] : bc_zero<T>();
  }
}

// masked overlaps: beta[a][t] = 0 for a >= before[t] (tentative reject t is
// checked against the accepts that preceded it only); P column-major, ld ldp,
// `scalars` doubles per entry (1 packed, 2 complex)
__global__ void bc_mask_kernel(double* __restrict__ P, int64_t ldp, int rows, int cols,
                               const int* __restrict__ before, int scalars) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols; e += gridDim.x * blockDim.x) {
    const int a = e % rows, c = e / rows;
    if (a >= before[c])
      for (int k = 0; k < scalars; ++k) P[(static_cast<int64_t>(c) * ldp + a) * scalars + k] = 0.0;
  }
}

// T = R^-1 for an a x a upper-triangular R (ld kBcMax), one CTA, right-looking
// from the bottom row: B starts as I; step i (a-1 down to 0) fixes row i,
// T(i, j) = B(i, j) / R_ii, and takes R(u, i) T(i, j) off every row u < i --
// one barrier per step, every thread's updates independent (no dot-product
// chains). Rows a .. 2*ceil(a/2)-1 of T are zero (the real GEMM reads an even K).
template <class T>
__global__ void __launch_bounds__(kBcThreads) bc_tri_inverse_kernel(const T* __restrict__ R, int a, T* __restrict__ Tinv) {
  extern __shared__ __align__(16) unsigned char bc_smem[];
  T* Rs = reinterpret_cast<T*>(bc_smem);  // R(i, j) = Rs[i + j * kBcMax]
  T* Bs = Rs + kBcMax * kBcMax;           // B(i, j) = Bs[i + j * kBcMax]; T written back in place per row
  const int tid = threadIdx.x;
  for (int e = tid; e < a * a; e += blockDim.x) {
    const int i = e % a, j = e / a;
    Rs[i + j * kBcMax] = R[i + j * kBcMax];
    Bs[i + j * kBcMax] = i == j ? bc_one<T>() : bc_zero<T>();
  }
  __syncthreads();
  for (int i = a - 1; i >= 0; --i) {
    const double ir = 1.0 / bc_re(Rs[i + i * kBcMax]);
    // rows u < i, columns j >= i: B(u, j) -= R(u, i) B(i, j) / R_ii (row i is final)
    const int w = a - i;
    for (int e = tid; e < i * w; e += blockDim.x) {
      const int u = e % i, j = i + e / i;
      Bs[u + j * kBcMax] = bc_sub(Bs[u + j * kBcMax], bc_mul(Rs[u + i * kBcMax], bc_scale(Bs[i + j * kBcMax], ir)));
    }
    __syncthreads();
    for (int j = i + tid; j < a; j += blockDim.x) Bs[i + j * kBcMax] = bc_scale(Bs[i + j * kBcMax], ir);
    // (row i is read again only by steps < i, after the next barrier)
  }
  __syncthreads();
  const int rows = (a + 1) & ~1;
  for (int e = threadIdx.x; e < rows * a; e += blockDim.x) {
    const int i = e % rows, c = e / rows;
    Tinv[i + c * kBcMax] = (i <= c && i < a) ? Bs[i + c * kBcMax] : bc_zero<T>();
  }
}

// max |(Q^H Q)_ij - delta_ij| of the new block (G ld ldg, a x a): the
// a-posteriori orthogonality check of CholQR2 (the caller falls back to the
// exact per-survivor kernel above a bound)
template <class T>
__global__ void bc_orth_error_kernel(const T* __restrict__ G, int ldg, int a, double* __restrict__ out) {
  __shared__ double red[32];
  double m = 0.0;
  for (int e = threadIdx.x; e < a * a; e += blockDim.x) {
    const int i = e % a, j = e / a;
    T v = G[i + static_cast<int64_t>(j) * ldg];
    if (i == j) v = bc_sub(v, bc_scale(bc_one<T>(), 1.0));
    m = fmax(m, sqrt(bc_abs2(v)));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) *out = m;
  }
}

// accepted survivors that were re-checked report the CGS2 norm R_aa = R2_aa R1_aa
// (R1_aa = sqrt(s) is already in rn); the block's first accept keeps rn2
__global__ void bc_rn_kernel(const BcDecision* __restrict__ dec, const double* __restrict__ diag2,
                             const int* __restrict__ flags, double* __restrict__ rn) {
  const int a = threadIdx.x;
  if (a >= dec->nacc) return;
  const int q = dec->acc[a];
  if (flags[q] & 2) rn[q] *= diag2[a];
}

// zero every element outside [lo, hi) (doubles) of n vectors of W doubles
__global__ void bc_zero_outside_kernel(double* __restrict__ v, int64_t n, int64_t W, int64_t lo, int64_t hi) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n * W;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k = e % W;
    if (k < lo || k >= hi) v[e] = 0.0;
  }
}

template <class T> constexpr int bc_smem_bytes() { return 2 * kBcMax * kBcMax * static_cast<int>(sizeof(T)); }

} // namespace liecl_b200
