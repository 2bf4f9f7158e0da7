// Real-FP64 projection GEMMs on DMMA.8x8x4 for the anti-Hermitian path.
//
// Anti-Hermitian operators (every generator i*H of the BASELINE dense
// configs, and everything their closure produces) are stored packed real:
// a d x d real matrix M with, for i < j, M(i,j) = Re A(i,j), M(j,i) = Im A(i,j)
// and M(i,i) = Im A(i,i) -- d^2 reals instead of d^2 complex numbers. The
// reference inner product (1/d) sum conj(A) B (R:src/dense.cpp:53-59) is real
// for two anti-Hermitian operators and equals (1/d) sum_k w_k a_k b_k with
// w = 2 off the diagonal and 1 on it (exact scalings), so one projection pass
// (R:src/closure.cpp:149-160) becomes two real GEMMs:
//
//   K2a_r  beta = (1/d) Vw^T X          (Vw = w .* V, kept beside V)
//   K2b_r  R    = X - V beta, sum_k w_k R_k^2 partials (the weighted norm)
//
// 2 N D flops each per candidate instead of 8 N D. Tile: BM x BN = 128 x 64
// real per CTA, 4 warps as 2 x 2 of 64 x 32, two CTAs per SM, BK = 16,
// 3-stage cp.async pipeline. Inside a BK tile the k order is permuted so a
// thread's fragments for two consecutive k-steps are adjacent (128-bit loads);
// row paddings keep every fragment access bank-conflict free.
#pragma once

#include "common.cuh"

namespace liecl_b200 {

namespace rg {
constexpr int BM = 128, BN = 64, BK = 16, STAGES = 3;
constexpr int GROUP = 16;  // M-tiles per raster group: 16 x 4 MB basis tiles stay in L2 while the candidates stream
constexpr int WM = 2, WN = 2, THREADS = 32 * WM * WN;  // 4 warps, 2 CTAs per SM
constexpr int WTM = BM / WM, WTN = BN / WN;  // 64 x 32 warp tile
constexpr int MT = WTM / 8, NT = WTN / 8;    // 8 x 4 m8n8 tiles
constexpr int LDK = BK + 8;                  // K-contiguous rows (doubles): == 8 mod 16 for 128-bit loads
constexpr int LDM = BM + 2;                  // M-contiguous rows (doubles): 2*LDM == 4 mod 16
constexpr int A_KC = BM * LDK, A_MC = BK * LDM, B_KC = BN * LDK;
template <bool KC> constexpr int a_elems() { return KC ? A_KC : A_MC; }
template <bool KC> constexpr int smem_bytes() { return STAGES * (a_elems<KC>() + B_KC) * 8; }
} // namespace rg

// weight of packed element k of a d x d matrix: 1 on the diagonal, 2 elsewhere.
// Kernels working on a slice [lo, hi) of the packed vector pass k = local row +
// wofs, wofs = lo mod (d + 1).
__device__ __forceinline__ double packed_weight(int64_t k, int d) {
  return (k % (d + 1)) == 0 ? 1.0 : 2.0;
}

enum class REpi { kStoreScaled, kSubtractNorm };

// C(m, n) = epi( sum_k A(m, k) B(k, n) ), all real:
//   A_KCONTIG: A(m, k) = A[m*lda + k]; else A(m, k) = A[k*lda + m]
//   B(k, n) = B[n*ldb + k]
//   kStoreScaled : C[n*ldc + m] = alpha * acc        (split-K: raw partial slices)
//   kSubtractNorm: C[n*ldc + m] = X[n*ldx + m] - acc;
//                  partial[blockIdx.x*N + n] = sum_rows w(m) C^2 (w: packed_weight, dim)
template <bool A_KCONTIG, REpi EPI>
__global__ void __launch_bounds__(rg::THREADS, 2)
dgemm_dmma_kernel(int M, int N, int K, const double* __restrict__ A, int64_t lda, const double* __restrict__ B,
                  int64_t ldb, double* __restrict__ Cout, int64_t ldc, double alpha, const double* __restrict__ X,
                  int64_t ldx, double* __restrict__ partial, int dim, int k_chunk, int64_t split_stride,
                  int wofs = 0) {
  using namespace rg;
  extern __shared__ __align__(16) double rsm[];
  double* As = rsm;
  double* Bs = rsm + STAGES * a_elems<A_KCONTIG>();

  if (k_chunk > 0) {
    const int kb = blockIdx.z * k_chunk;
    A += A_KCONTIG ? static_cast<int64_t>(kb) : static_cast<int64_t>(kb) * lda;
    B += kb;
    K = min(K - kb, k_chunk);
    Cout += blockIdx.z * split_stride;
  }
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % WM, wn = warp / WM;
  int m_tile, n_tile;
  grouped_tile<GROUP>(blockIdx.x + blockIdx.y * gridDim.x, gridDim.x, gridDim.y, m_tile, n_tile);
  const int m0 = m_tile * BM, n0 = n_tile * BN;
  const int KT = K > 0 ? (K + BK - 1) / BK : 0;

  // 16-byte chunks (2 doubles); K and the M extent are even on this path
  auto load_stage = [&](int stage, int kt) {
    const int k0 = kt * BK;
    double* as = As + stage * a_elems<A_KCONTIG>();
    double* bs = Bs + stage * B_KC;
    if (A_KCONTIG) {
#pragma unroll
      for (int i = 0; i < (BM * BK / 2) / THREADS; ++i) {
        const int e = tid + i * THREADS;
        const int r = e / (BK / 2), c = (e % (BK / 2)) * 2;
        const int gm = m0 + r, gk = k0 + c;
        const bool ok = gm < M && gk < K;
        cp_async16(as + r * LDK + c, ok ? A + static_cast<int64_t>(gm) * lda + gk : A, ok ? 16 : 0);
      }
    } else {
#pragma unroll
      for (int i = 0; i < (BM * BK / 2) / THREADS; ++i) {
        const int e = tid + i * THREADS;
        const int r = e / (BM / 2), c = (e % (BM / 2)) * 2;
        const int gk = k0 + r, gm = m0 + c;
        const bool ok = gm < M && gk < K;
        cp_async16(as + r * LDM + c, ok ? A + static_cast<int64_t>(gk) * lda + gm : A, ok ? 16 : 0);
      }
    }
#pragma unroll
    for (int i = 0; i < (BN * BK / 2) / THREADS; ++i) {
      const int e = tid + i * THREADS;
      const int r = e / (BK / 2), c = (e % (BK / 2)) * 2;
      const int gn = n0 + r, gk = k0 + c;
      const bool ok = gn < N && gk < K;
      cp_async16(bs + r * LDK + c, ok ? B + static_cast<int64_t>(gn) * ldb + gk : B, ok ? 16 : 0);
    }
  };

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < KT) load_stage(nk % STAGES, nk);
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * a_elems<A_KCONTIG>();
    const double* bs = Bs + (kt % STAGES) * B_KC;
    // K permutation inside the tile: k-step 2p+q uses k = 8p + 2t + q, so a
    // thread's fragments for the step pair are adjacent (one 128-bit load on
    // K-contiguous tiles); A and B use the same permutation, so the dot
    // products are unchanged. Fragments of the next pair are loaded before
    // the DMMAs of the current pair are issued.
    double2 af[2][MT], bf[2][NT];
    auto load_frags = [&](int p, double2 (&a)[MT], double2 (&b)[NT]) {
      const int kc = 8 * p + 2 * t;
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int mr = wm * WTM + i * 8 + g;
        if (A_KCONTIG) {
          a[i] = *reinterpret_cast<const double2*>(as + mr * LDK + kc);
        } else {
          a[i].x = as[kc * LDM + mr];
          a[i].y = as[(kc + 1) * LDM + mr];
        }
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = *reinterpret_cast<const double2*>(bs + (wn * WTN + j * 8 + g) * LDK + kc);
    };
    load_frags(0, af[0], bf[0]);
#pragma unroll
    for (int p = 0; p < BK / 8; ++p) {
      const int cur = p & 1;
      if (p + 1 < BK / 8) load_frags(p + 1, af[cur ^ 1], bf[cur ^ 1]);
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cur][i].x, bf[cur][j].x);
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[cur][i].y, bf[cur][j].y);
    }
  }
  cp_async_wait<0>();

  if (EPI == REpi::kStoreScaled) {
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int gm = m0 + wm * WTM + i * 8 + g;
      if (gm >= M) {
        // pad rows M <= row < ldc (the even leading dimension of beta) are
        // written as zeros: the subtract GEMM reads one row past an odd basis
        // count, where V is zero and beta must be finite (0 * NaN from a
        // recycled workspace would poison the residual)
        if (gm < ldc) {
#pragma unroll
          for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int gn = n0 + wn * WTN + j * 8 + 2 * t + h;
              if (gn < N) Cout[static_cast<int64_t>(gn) * ldc + gm] = 0.0;
            }
        }
        continue;
      }
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gn = n0 + wn * WTN + j * 8 + 2 * t + h;
          if (gn < N) Cout[static_cast<int64_t>(gn) * ldc + gm] = alpha * acc[i][j][h];
        }
    }
  } else {
    __shared__ double red[WM][BN];
    double colsum[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j) colsum[j][0] = colsum[j][1] = 0.0;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int gm = m0 + wm * WTM + i * 8 + g;
      if (gm >= M) continue;
      const double w = packed_weight(gm + wofs, dim);
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gn = n0 + wn * WTN + j * 8 + 2 * t + h;
          if (gn < N) {
            const double r = X[static_cast<int64_t>(gn) * ldx + gm] - acc[i][j][h];
            Cout[static_cast<int64_t>(gn) * ldc + gm] = r;
            colsum[j][h] += w * r * r;
          }
        }
    }
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double v = colsum[j][h];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        if (g == 0) red[wm][wn * WTN + j * 8 + 2 * t + h] = v;
      }
    __syncthreads();
    for (int c = tid; c < BN; c += THREADS) {
      const int gn = n0 + c;
      if (gn < N) {
        double s = 0.0;
#pragma unroll
        for (int w2 = 0; w2 < WM; ++w2) s += red[w2][c];
        partial[static_cast<int64_t>(m_tile) * N + gn] = s;
      }
    }
  }
}

// split-K reductions for the real GEMMs (fixed slice order)
__global__ void rsplitk_reduce_scale_kernel(const double* __restrict__ ws, int slices, int64_t stride, int64_t total,
                                            double alpha, double* __restrict__ P) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < slices; ++z) s += ws[z * stride + i];
    P[i] = alpha * s;
  }
}

// one CTA of rg::BM threads per (row tile, column); partial layout as the GEMM's
__global__ void rsplitk_reduce_subtract_kernel(const double* __restrict__ ws, int slices, int64_t stride, int M,
                                               int N, const double* __restrict__ X, double* __restrict__ R,
                                               double* __restrict__ partial, int dim, int64_t ldx,
                                               int wofs = 0) {
  __shared__ double red[rg::BM / 32];
  const int mt = blockIdx.x, b = blockIdx.y;
  const int m = mt * rg::BM + threadIdx.x;
  double s = 0.0;
  if (m < M) {
    const int64_t i = static_cast<int64_t>(b) * M + m;  // the workspace is packed (ld M)
    const int64_t ix = static_cast<int64_t>(b) * ldx + m;
    double acc = 0.0;
    for (int z = 0; z < slices; ++z) acc += ws[z * stride + i];
    const double r = X[ix] - acc;
    R[ix] = r;
    s = packed_weight(m + wofs, dim) * r * r;
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < rg::BM / 32; ++w) tot += red[w];
    partial[static_cast<int64_t>(mt) * N + b] = tot;
  }
}

} // namespace liecl_b200
