// Complex-FP64 projection GEMMs on the FP64 tensor pipe (DMMA.8x8x4).
//
// These are the two halves of one projection pass of project_residual
// (R:src/closure.cpp:142-162) applied to a whole batch of candidates:
//
//   K2a  beta = (1/d) V^H X           inner_product x |V| (R:src/dense.cpp:53-59)
//   K2b  R    = X - V beta, ||R_b||^2  linear_combination (R:src/operator.cpp:155-162)
//                                       + norm (R:src/dense.cpp:61-63) partials
//
// V is the basis slab, D x N column-major (basis vector n = column n =
// column-major vec of the d x d operator); X and R are D x B candidate slabs;
// beta is N x B. All complex128, interleaved (double2).
//
// Tiling: BM x BN complex outputs per CTA, 2 x 2 warps of 32 x 32, BK complex
// per stage, STAGES-deep cp.async pipeline. Each complex MAC is 4 DMMAs on
// re/im fragments (8 real flops). Shared-memory rows are padded so every
// 128-bit fragment load is bank-conflict free:
//   K-contiguous tile [row][k], LD = BK + 4   (== 4 mod 8 complex)
//   M-contiguous tile [k][row], LD = BM + 2   (== 2 mod 8 complex)
#pragma once

#include "common.cuh"

namespace liecl_b200 {

namespace zg {
constexpr int BM = 64, BN = 64, BK = 8, STAGES = 4;
constexpr int WM = 2, WN = 2, THREADS = 32 * WM * WN;
constexpr int WTM = BM / WM, WTN = BN / WN;  // warp tile 32 x 32
constexpr int MT = WTM / 8, NT = WTN / 8;    // 4 x 4 m8n8 tiles per warp
constexpr int LDK = BK + 4;                  // K-contiguous rows
constexpr int LDM = BM + 2;                  // M-contiguous rows
constexpr int A_KC_ELEMS = BM * LDK;
constexpr int A_MC_ELEMS = BK * LDM;
constexpr int B_ELEMS = BN * LDK;

template <bool A_KCONTIG> constexpr int a_elems() { return A_KCONTIG ? A_KC_ELEMS : A_MC_ELEMS; }
template <bool A_KCONTIG> constexpr int smem_bytes() {
  return STAGES * (a_elems<A_KCONTIG>() + B_ELEMS) * static_cast<int>(sizeof(double2));
}
} // namespace zg

enum class Epilogue { kStoreScaled, kSubtractNorm };

// C(m, n) = epilogue( sum_k op(A)(m, k) * B(k, n) )
//   A_KCONTIG: A(m, k) = A[m*lda + k] (V^H side: m = basis index, k = element)
//   else     : A(m, k) = A[k*lda + m] (V side:   m = element,     k = basis index)
//   CONJ_A   : use conj(A(m, k))
//   B(k, n) = B[n*ldb + k]
//   kStoreScaled : C[n*ldc + m] = alpha * acc
//   kSubtractNorm: C[n*ldc + m] = X[n*ldx + m] - acc, and
//                  partial[blockIdx.x * N + n] = sum over this CTA's rows of |C|^2
//
// Split-K (k_chunk > 0, small grids): CTA z covers k in [z*k_chunk, (z+1)*k_chunk)
// and stores its raw partial product at Cout + z*split_stride (kStoreScaled only);
// splitk_reduce_* below sum the slices in fixed order (deterministic).
template <bool A_KCONTIG, bool CONJ_A, Epilogue EPI>
__global__ void __launch_bounds__(zg::THREADS)
zgemm_dmma_kernel(int M, int N, int K, const double2* __restrict__ A, int64_t lda,
                  const double2* __restrict__ B, int64_t ldb, double2* __restrict__ Cout,
                  int64_t ldc, double alpha, const double2* __restrict__ X, int64_t ldx,
                  double* __restrict__ partial, int k_chunk, int64_t split_stride) {
  using namespace zg;
  extern __shared__ __align__(16) double2 smem[];
  double2* As = smem;
  double2* Bs = smem + STAGES * a_elems<A_KCONTIG>();

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
  grouped_tile<8>(blockIdx.x + blockIdx.y * gridDim.x, gridDim.x, gridDim.y, m_tile, n_tile);
  const int m0 = m_tile * BM, n0 = n_tile * BN;
  const int KT = K > 0 ? (K + BK - 1) / BK : 0;

  auto load_stage = [&](int stage, int kt) {
    const int k0 = kt * BK;
    double2* as = As + stage * a_elems<A_KCONTIG>();
    double2* bs = Bs + stage * B_ELEMS;
    if (A_KCONTIG) {
#pragma unroll
      for (int i = 0; i < (BM * BK) / THREADS; ++i) {
        const int e = tid + i * THREADS;
        const int r = e / BK, c = e % BK;
        const int gm = m0 + r, gk = k0 + c;
        const bool ok = gm < M && gk < K;
        const double2* src = ok ? A + static_cast<int64_t>(gm) * lda + gk : A;
        cp_async16(as + r * LDK + c, src, ok ? 16 : 0);
      }
    } else {
#pragma unroll
      for (int i = 0; i < (BM * BK) / THREADS; ++i) {
        const int e = tid + i * THREADS;
        const int r = e / BM, c = e % BM;
        const int gk = k0 + r, gm = m0 + c;
        const bool ok = gm < M && gk < K;
        const double2* src = ok ? A + static_cast<int64_t>(gk) * lda + gm : A;
        cp_async16(as + r * LDM + c, src, ok ? 16 : 0);
      }
    }
#pragma unroll
    for (int i = 0; i < (BN * BK) / THREADS; ++i) {
      const int e = tid + i * THREADS;
      const int r = e / BK, c = e % BK;
      const int gn = n0 + r, gk = k0 + c;
      const bool ok = gn < N && gk < K;
      const double2* src = ok ? B + static_cast<int64_t>(gn) * ldb + gk : B;
      cp_async16(bs + r * LDK + c, src, ok ? 16 : 0);
    }
  };

  double acc_re[MT][NT][2], acc_im[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      acc_re[i][j][0] = acc_re[i][j][1] = 0.0;
      acc_im[i][j][0] = acc_im[i][j][1] = 0.0;
    }

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
    const double2* as = As + (kt % STAGES) * a_elems<A_KCONTIG>();
    const double2* bs = Bs + (kt % STAGES) * B_ELEMS;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      const int kc = kk * 4 + t;
      double2 af[MT], bf[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int mr = wm * WTM + i * 8 + g;
        af[i] = A_KCONTIG ? as[mr * LDK + kc] : as[kc * LDM + mr];
        if (CONJ_A) af[i].y = -af[i].y;
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) bf[j] = bs[(wn * WTN + j * 8 + g) * LDK + kc];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const double a_re = af[i].x, a_im = af[i].y, a_nim = -af[i].y;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          dmma_8x8x4(acc_re[i][j][0], acc_re[i][j][1], a_re, bf[j].x);
          dmma_8x8x4(acc_re[i][j][0], acc_re[i][j][1], a_nim, bf[j].y);
          dmma_8x8x4(acc_im[i][j][0], acc_im[i][j][1], a_re, bf[j].y);
          dmma_8x8x4(acc_im[i][j][0], acc_im[i][j][1], a_im, bf[j].x);
        }
      }
    }
  }
  cp_async_wait<0>();

  if (EPI == Epilogue::kStoreScaled) {
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int gm = m0 + wm * WTM + i * 8 + g;
      if (gm >= M) continue;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gn = n0 + wn * WTN + j * 8 + 2 * t + h;
          if (gn < N)
            Cout[static_cast<int64_t>(gn) * ldc + gm] = make_double2(alpha * acc_re[i][j][h], alpha * acc_im[i][j][h]);
        }
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
#pragma unroll
      for (int j = 0; j < NT; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gn = n0 + wn * WTN + j * 8 + 2 * t + h;
          if (gn < N) {
            const double2 x = X[static_cast<int64_t>(gn) * ldx + gm];
            const double2 r = make_double2(x.x - acc_re[i][j][h], x.y - acc_im[i][j][h]);
            Cout[static_cast<int64_t>(gn) * ldc + gm] = r;
            colsum[j][h] += r.x * r.x + r.y * r.y;
          }
        }
      }
    }
    // reduce over g (lanes sharing t), then over the WM warps of this column strip
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
        for (int w = 0; w < WM; ++w) s += red[w][c];
        partial[static_cast<int64_t>(m_tile) * N + gn] = s;
      }
    }
  }
}

// P[i] = alpha * sum_z ws[z*stride + i], i < total (fixed slice order)
__global__ void splitk_reduce_scale_kernel(const double2* __restrict__ ws, int slices, int64_t stride, int64_t total,
                                           double alpha, double2* __restrict__ P) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double re = 0.0, im = 0.0;
    for (int z = 0; z < slices; ++z) {
      const double2 v = ws[z * stride + i];
      re += v.x;
      im += v.y;
    }
    P[i] = make_double2(alpha * re, alpha * im);
  }
}

// R[b*M + m] = X[b*M + m] - sum_z ws[z*stride + b*M + m]; one CTA of zg::BM
// threads per (row tile, column) also writes partial[mt*N + b] = sum |R|^2 over
// its rows, the layout norm_finalize_kernel expects.
__global__ void splitk_reduce_subtract_kernel(const double2* __restrict__ ws, int slices, int64_t stride, int M,
                                              int N, const double2* __restrict__ X, double2* __restrict__ R,
                                              double* __restrict__ partial, int64_t ldx) {
  __shared__ double red[zg::BM / 32];
  const int mt = blockIdx.x, b = blockIdx.y;
  const int m = mt * zg::BM + threadIdx.x;
  double s = 0.0;
  if (m < M) {
    const int64_t i = static_cast<int64_t>(b) * M + m;  // the workspace is packed (ld M)
    const int64_t ix = static_cast<int64_t>(b) * ldx + m;
    double re = 0.0, im = 0.0;
    for (int z = 0; z < slices; ++z) {
      const double2 v = ws[z * stride + i];
      re += v.x;
      im += v.y;
    }
    const double2 x = X[ix];
    const double2 r = make_double2(x.x - re, x.y - im);
    R[ix] = r;
    s = r.x * r.x + r.y * r.y;
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < zg::BM / 32; ++w) tot += red[w];
    partial[static_cast<int64_t>(mt) * N + b] = tot;
  }
}

} // namespace liecl_b200
