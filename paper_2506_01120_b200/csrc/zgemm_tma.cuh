// Complex-FP64 projection GEMMs (K2a / K2b, see zgemm_dmma.cuh) with TMA
// staging, the complex counterpart of dgemm_tma.cuh: a 128-byte smem row holds
// 8 complex values (one 16-byte swizzle chunk each, chunk c of row r at
// c ^ (r & 7)), stages complete on an expect_tx mbarrier and are released per
// warp on an "empty" mbarrier, thread 0 issues the copies two k-tiles ahead.
// Inside a k-tile of 8 complex the lane order is k = 2t + s (k-step s of lane
// t), the same for A and B:
//   K-contiguous rows: a quarter-warp (rows g, g^1) reads chunks
//     (2t + s) ^ g -- disjoint sets, conflict-free;
//   M-contiguous A (K2b: A(m, k) = V[k][m]): 3-D box [m / 8][k][m % 8],
//     row (m / 8) * 8 + k, chunk (m % 8) ^ k: four lanes per chunk, the minimum
//     for 16-byte loads.
// Tile: 64 x 64 complex per CTA (4 warps of 32 x 32), BK = 8 complex, 4 stages
// of 16 KB.
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "dgemm_tma.cuh"
#include "zgemm_dmma.cuh"

namespace liecl_b200 {

namespace ztg {
constexpr int BM = 64, BN = 64, BK = 8, STAGES = 4, AHEAD = 2;
constexpr int WM = 2, WN = 2, THREADS = 32 * WM * WN;
constexpr int WTM = BM / WM, WTN = BN / WN;
constexpr int MT = WTM / 8, NT = WTN / 8;
constexpr int A_BYTES = BM * BK * 16, B_BYTES = BN * BK * 16, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024;
}  // namespace ztg

// swizzled complex offsets inside a stage tile
__device__ __forceinline__ int zsw_kc(int r, int k) { return r * 8 + ((k ^ r) & 7); }
__device__ __forceinline__ int zsw_mc(int m, int k) { return ((m >> 3) * 8 + k) * 8 + (((m & 7) ^ k) & 7); }

// Same contract as zgemm_dmma_kernel without split-K. mapA: A_KCONTIG -- 2-D
// {2K, M} doubles, box {16, 64}; else 3-D {16, K, M / 8} (doubles, complex
// rows; M a multiple of 8), box {16, 8, 8}. mapB: 2-D {2K, N}, box {16, 64}.
template <bool A_KCONTIG, bool CONJ_A, Epilogue EPI>
__global__ void __launch_bounds__(ztg::THREADS)
zgemm_tma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int M, int N,
                 int K, double2* __restrict__ Cout, int64_t ldc, double alpha, const double2* __restrict__ X,
                 int64_t ldx, double* __restrict__ partial) {
  using namespace ztg;
  extern __shared__ __align__(16) unsigned char ztsm_raw[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  unsigned char* tsm = ztsm_raw + ((1024 - (smem_u32(ztsm_raw) & 1023)) & 1023);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % WM, wn = warp / WM;
  int m_tile, n_tile;
  grouped_tile<8>(blockIdx.x + blockIdx.y * gridDim.x, gridDim.x, gridDim.y, m_tile, n_tile);
  const int m0 = m_tile * BM, n0 = n_tile * BN;
  const int KT = K > 0 ? (K + BK - 1) / BK : 0;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], WM * WN);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](int kt) {
    const int s = kt % STAGES;
    if (kt >= STAGES) mbar_wait(&empty[s], ((kt / STAGES) - 1) & 1);
    unsigned char* a = tsm + s * STAGE_BYTES;
    mbar_expect_tx(&full[s], STAGE_BYTES);
    if (A_KCONTIG) tma_load_2d(a, &mapA, 2 * kt * BK, m0, &full[s]);
    else tma_load_3d(a, &mapA, 0, kt * BK, m0 / 8, &full[s]);
    tma_load_2d(a + A_BYTES, &mapB, 2 * kt * BK, n0, &full[s]);
  };
  if (tid == 0)
    for (int kt = 0; kt < AHEAD && kt < KT; ++kt) issue(kt);

  double acc_re[MT][NT][2], acc_im[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      acc_re[i][j][0] = acc_re[i][j][1] = 0.0;
      acc_im[i][j][0] = acc_im[i][j][1] = 0.0;
    }

  for (int kt = 0; kt < KT; ++kt) {
    if (tid == 0 && kt + AHEAD < KT) issue(kt + AHEAD);
    const int s = kt % STAGES;
    mbar_wait(&full[s], (kt / STAGES) & 1);
    const double2* as = reinterpret_cast<const double2*>(tsm + s * STAGE_BYTES);
    const double2* bs = reinterpret_cast<const double2*>(tsm + s * STAGE_BYTES + A_BYTES);
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      const int kc = 2 * t + kk;
      double2 af[MT], bf[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int mr = wm * WTM + i * 8 + g;
        af[i] = A_KCONTIG ? as[zsw_kc(mr, kc)] : as[zsw_mc(mr, kc)];
        if (CONJ_A) af[i].y = -af[i].y;
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) bf[j] = bs[zsw_kc(wn * WTN + j * 8 + g, kc)];
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
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  if (EPI == Epilogue::kStoreScaled) {
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int gm = m0 + wm * WTM + i * 8 + g;
      if (gm >= M) continue;
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gn = n0 + wn * WTN + j * 8 + 2 * t + h;
          if (gn < N)
            Cout[static_cast<int64_t>(gn) * ldc + gm] = make_double2(alpha * acc_re[i][j][h], alpha * acc_im[i][j][h]);
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
      for (int j = 0; j < NT; ++j)
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
        double s2 = 0.0;
#pragma unroll
        for (int w = 0; w < WM; ++w) s2 += red[w][c];
        partial[static_cast<int64_t>(m_tile) * N + gn] = s2;
      }
    }
  }
}

}  // namespace liecl_b200
