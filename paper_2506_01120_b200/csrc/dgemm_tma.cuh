// Real-FP64 projection GEMMs (K2a_r / K2b_r, see dgemm_dmma.cuh) with TMA
// staging: operand tiles arrive by cp.async.bulk.tensor into 128-byte-swizzled
// shared memory, completion is tracked per stage by an mbarrier (expect_tx),
// and each warp releases a stage with one arrive on the stage's "empty"
// mbarrier -- no CTA-wide barrier in the main loop and no per-thread copy
// instructions. One elected thread (thread 0) issues the copies two k-tiles
// ahead into a 4-stage ring.
//
// DMMA.8x8x4 takes its operands from registers, so fragments are still read
// from shared memory with ld.shared; the swizzle (16-byte chunk c of 128-byte
// row r lands at chunk c ^ (r & 7)) and the k order inside a 16-wide tile
// (k-step 2p+q of lane t uses k = 4t + 2p + q, the same permutation for A and
// B, so dot products are unchanged up to rounding order) make every fragment
// load conflict-free:
//   K-contiguous tile (rows of 16 k): lane (g, t) reads the 16-byte chunk
//     (2t + p) ^ (row & 7): rows g and g^1 of a quarter-warp hit disjoint chunks;
//   M-contiguous A (K2b: A(m, k) = V[k][m]): the 3-D box [m/16][k][m%16]
//     (sw_mc3) leaves half-warps of 8-byte loads 2-way conflicted; the 5-D box
//     (sw_mc, MC_BOX = 5) orders k's bits so lane t lands in the swizzle row
//     and the loads are conflict-free -- measured 0.5 % slower (the TMA
//     gathers 16 lines from 4 row groups), so the engine launches MC_BOX = 3.
// Tile: BM x BN = 128 x 64 per CTA (4 warps of 64 x 32), BK = 16, two CTAs per
// SM (96 KB of stages each).
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "dgemm_dmma.cuh"

namespace liecl_b200 {

namespace tg {
constexpr int BM = 128, BN = 64, BK = 16, STAGES = 4, AHEAD = 2;
constexpr int WM = 2, WN = 2, THREADS = 32 * WM * WN;
constexpr int WTM = BM / WM, WTN = BN / WN;
constexpr int MT = WTM / 8, NT = WTN / 8;
constexpr int A_BYTES = BM * BK * 8, B_BYTES = BN * BK * 8, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024;  // + slack for 1024-byte alignment
}  // namespace tg

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            int c4, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}

// swizzled element offsets (doubles) inside a stage tile
__device__ __forceinline__ int sw_kc(int r, int k) { return r * 16 + ((((k >> 1) ^ r) & 7) << 1) + (k & 1); }
// M-contiguous tile as the 5-D box [m/16][p][t][q][m%16] of k = 4t + 2p + q:
// line (m/16)*16 + 8p + 2t + q, so line & 7 = 2t + q and the swizzled chunk
// ((m%16)/2) ^ (2t + q) spreads each half-warp's fragment loads over 16 banks
// (a [m/16][k][m%16] box leaves t's high bit out of line & 7: 2-way conflicts)
__device__ __forceinline__ int sw_mc(int m, int k) {
  const int line = (m >> 4) * 16 + ((k >> 1) & 1) * 8 + (k >> 2) * 2 + (k & 1);
  return line * 16 + ((((m & 15) >> 1) ^ line) & 7) * 2 + (m & 1);
}
// the 3-D box [m/16][k][m%16] (line (m/16)*16 + k): half-warps 2-way conflicted
__device__ __forceinline__ int sw_mc3(int m, int k) {
  return ((m >> 4) * 16 + k) * 16 + ((((m & 15) >> 1) ^ k) & 7) * 2 + (m & 1);
}

// Same contract as dgemm_dmma_kernel without split-K: C(m, n) = epi(sum_k
// A(m, k) B(k, n)). mapA: A_KCONTIG -- 2-D {K, M} box {16, 128}; else 5-D
// {16 (m%16), 2 (q), ceil(K/4) (t), 2 (p), M/16} box {16, 2, 4, 2, 8} (M a
// multiple of 16; rows up to 4 ceil(K/4) are read and must be zero past K).
// mapB: 2-D {K, N} box {16, 64}. All 128-byte swizzled, out-of-bounds
// elements read as zeros.
template <bool A_KCONTIG, REpi EPI, int MC_BOX = 5, int GROUP = rg::GROUP>
__global__ void __launch_bounds__(tg::THREADS, 2)
dgemm_tma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int M, int N,
                 int K, double* __restrict__ Cout, int64_t ldc, double alpha, const double* __restrict__ X,
                 int64_t ldx, double* __restrict__ partial, int dim, int wofs = 0) {
  using namespace tg;
  extern __shared__ __align__(16) unsigned char tsm_raw[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  unsigned char* tsm = tsm_raw + ((1024 - (smem_u32(tsm_raw) & 1023)) & 1023);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % WM, wn = warp / WM;
  int m_tile, n_tile;
  grouped_tile<GROUP>(blockIdx.x + blockIdx.y * gridDim.x, gridDim.x, gridDim.y, m_tile, n_tile);
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

  auto issue = [&](int kt) {  // thread 0: tile kt into stage kt % STAGES
    const int s = kt % STAGES;
    if (kt >= STAGES) mbar_wait(&empty[s], ((kt / STAGES) - 1) & 1);
    unsigned char* a = tsm + s * STAGE_BYTES;
    mbar_expect_tx(&full[s], STAGE_BYTES);
    if (A_KCONTIG) tma_load_2d(a, &mapA, kt * BK, m0, &full[s]);
    else if (MC_BOX == 5) tma_load_5d(a, &mapA, 0, 0, kt * (BK / 4), 0, m0 / 16, &full[s]);
    else tma_load_3d(a, &mapA, 0, kt * BK, m0 / 16, &full[s]);
    tma_load_2d(a + A_BYTES, &mapB, kt * BK, n0, &full[s]);
  };
  if (tid == 0)
    for (int kt = 0; kt < AHEAD && kt < KT; ++kt) issue(kt);

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int kt = 0; kt < KT; ++kt) {
    if (tid == 0 && kt + AHEAD < KT) issue(kt + AHEAD);
    const int s = kt % STAGES;
    mbar_wait(&full[s], (kt / STAGES) & 1);
    const double* as = reinterpret_cast<const double*>(tsm + s * STAGE_BYTES);
    const double* bs = reinterpret_cast<const double*>(tsm + s * STAGE_BYTES + A_BYTES);
    double2 af[2][MT], bf[2][NT];
    auto load_frags = [&](int p, double2 (&a)[MT], double2 (&b)[NT]) {
      const int kc = 4 * t + 2 * p;
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int mr = wm * WTM + i * 8 + g;
        if (A_KCONTIG) {
          a[i] = *reinterpret_cast<const double2*>(as + sw_kc(mr, kc));
        } else {
          a[i].x = as[MC_BOX == 5 ? sw_mc(mr, kc) : sw_mc3(mr, kc)];
          a[i].y = as[MC_BOX == 5 ? sw_mc(mr, kc + 1) : sw_mc3(mr, kc + 1)];
        }
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = *reinterpret_cast<const double2*>(bs + sw_kc(wn * WTN + j * 8 + g, kc));
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
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
  }

  if (EPI == REpi::kStoreScaled) {
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int gm = m0 + wm * WTM + i * 8 + g;
      if (gm >= M) {
        if (gm < ldc) {  // pad rows of beta: zeros (see dgemm_dmma_kernel)
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
      const double w = packed_weight(gm + wofs, dim);  // wofs: the slice's first packed index mod (d + 1)
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

}  // namespace liecl_b200
