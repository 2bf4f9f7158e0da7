// K1: batched dense commutator with the fused norm / null-test / normalise
// epilogue of run_engine's hot loop A (R:src/closure.cpp:416-424):
//
//   h = B[l] B[m] - B[m] B[l]        dense_commutator   (R:src/dense.cpp:65-68)
//   ||h|| = sqrt(sum |h|^2)/sqrt(d)  dense_norm         (R:src/dense.cpp:61-63)
//   null iff ||h|| <= tol; else h_unit = (1/||h||) h    (R:src/closure.cpp:420-422)
//
// One cursor pair per group of warps; the two d x d operands sit in shared
// memory as split re/im planes (row stride d+4 doubles, so both the row- and
// the column-operand fragment loads of DMMA.8x8x4 are bank-conflict free) and
// h accumulates in registers as the single K = 2d product [A | -B] [B ; A].
// Pairs come from global cursor indices g (l(l-1)/2 + m), so a batch may span
// any number of rows.
#pragma once

#include "common.cuh"

namespace liecl_b200 {

template <int DIM> struct CommShape {
  static constexpr int TILES = (DIM / 8) * (DIM / 8);            // m8n8 output tiles
  static constexpr int WARPS_PER_PAIR = TILES >= 8 ? 8 : TILES;  // <= 8 warps per pair
  static constexpr int PAIRS_PER_CTA = 8 / WARPS_PER_PAIR;
  static constexpr int TILES_PER_WARP = TILES / WARPS_PER_PAIR;
  static constexpr int LD = DIM + 4;                             // doubles; == 4 mod 16 for DIM>=16
  static constexpr int PLANE = DIM * LD;
  static constexpr int SMEM_PER_PAIR = 4 * PLANE * 8 + WARPS_PER_PAIR * 8;
  static constexpr int SMEM = PAIRS_PER_CTA * SMEM_PER_PAIR;
};

// basis: commutator basis slab (vec layout, ld = DIM*DIM); pairs [g0, g0+count)
// write h_unit to out[j] (ld DIM*DIM), hnorm[j], is_null[j].
template <int DIM>
__global__ void __launch_bounds__(256)
commutator_norm_kernel(const double2* __restrict__ basis, int64_t g0, int count, double tol, bool normalize,
                       double2* __restrict__ out, double* __restrict__ hnorm, int* __restrict__ is_null) {
  using S = CommShape<DIM>;
  constexpr int D2 = DIM * DIM;
  extern __shared__ __align__(16) double csm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int slot = warp / S::WARPS_PER_PAIR;     // pair within CTA
  const int wip = warp % S::WARPS_PER_PAIR;      // warp within pair
  const int j = blockIdx.x * S::PAIRS_PER_CTA + slot;
  const bool active = j < count;

  double* base = csm + slot * (S::SMEM_PER_PAIR / 8);
  double* are = base;
  double* aim = are + S::PLANE;
  double* bre = aim + S::PLANE;
  double* bim = bre + S::PLANE;
  double* red = bim + S::PLANE;

  int64_t l = 0, m = 0;
  if (active) pair_from_index(g0 + j, l, m);
  // stage operands: element (row i, col k) of a column-major matrix -> plane[i*LD + k]
  if (active) {
    const double2* pa = basis + l * D2;
    const double2* pb = basis + m * D2;
    const int tip = threadIdx.x - slot * S::WARPS_PER_PAIR * 32;
    for (int e = tip; e < D2; e += S::WARPS_PER_PAIR * 32) {
      const int i = e % DIM, k = e / DIM;
      const double2 va = pa[e], vb = pb[e];
      are[i * S::LD + k] = va.x;
      aim[i * S::LD + k] = va.y;
      bre[i * S::LD + k] = vb.x;
      bim[i * S::LD + k] = vb.y;
    }
  }
  __syncthreads();

  double cre[S::TILES_PER_WARP][2], cim[S::TILES_PER_WARP][2];
  double sumsq = 0.0;
  if (active) {
#pragma unroll
    for (int q = 0; q < S::TILES_PER_WARP; ++q) {
      const int tile = wip * S::TILES_PER_WARP + q;
      const int ti = (tile / (DIM / 8)) * 8, tj = (tile % (DIM / 8)) * 8;
      double c0r = 0.0, c1r = 0.0, c0i = 0.0, c1i = 0.0;
      // h(i,j) = sum_k A(i,k) B(k,j) - B(i,k) A(k,j)
#pragma unroll 4
      for (int k0 = 0; k0 < DIM; k0 += 4) {
        const int k = k0 + t;
        // first product: row operand A(ti+g, k), column operand B(k, tj+g)
        double xr = are[(ti + g) * S::LD + k], xi = aim[(ti + g) * S::LD + k];
        double yr = bre[k * S::LD + tj + g], yi = bim[k * S::LD + tj + g];
        dmma_8x8x4(c0r, c1r, xr, yr);
        dmma_8x8x4(c0r, c1r, -xi, yi);
        dmma_8x8x4(c0i, c1i, xr, yi);
        dmma_8x8x4(c0i, c1i, xi, yr);
        // second product, negated: row operand -B(ti+g, k), column operand A(k, tj+g)
        xr = -bre[(ti + g) * S::LD + k];
        xi = -bim[(ti + g) * S::LD + k];
        yr = are[k * S::LD + tj + g];
        yi = aim[k * S::LD + tj + g];
        dmma_8x8x4(c0r, c1r, xr, yr);
        dmma_8x8x4(c0r, c1r, -xi, yi);
        dmma_8x8x4(c0i, c1i, xr, yi);
        dmma_8x8x4(c0i, c1i, xi, yr);
      }
      cre[q][0] = c0r; cre[q][1] = c1r; cim[q][0] = c0i; cim[q][1] = c1i;
      sumsq += c0r * c0r + c0i * c0i + c1r * c1r + c1i * c1i;
    }
  }
  sumsq = warp_sum(sumsq);
  if (lane == 0) red[wip] = sumsq;
  __syncthreads();
  if (!active) return;
  double total = 0.0;
#pragma unroll
  for (int w = 0; w < S::WARPS_PER_PAIR; ++w) total += red[w];
  const double hn = sqrt(total) / sqrt(static_cast<double>(DIM));
  const bool nul = !(hn > tol);
  if (wip == 0 && lane == 0) {
    hnorm[j] = hn;
    is_null[j] = nul ? 1 : 0;
  }
  const double s = !normalize ? 1.0 : (nul ? 0.0 : 1.0 / hn);
  double2* o = out + static_cast<int64_t>(j) * D2;
#pragma unroll
  for (int q = 0; q < S::TILES_PER_WARP; ++q) {
    const int tile = wip * S::TILES_PER_WARP + q;
    const int ti = (tile / (DIM / 8)) * 8, tj = (tile % (DIM / 8)) * 8;
    // thread owns h(ti+g, tj+2t+h): column-major index (tj+2t+h)*DIM + ti+g
#pragma unroll
    for (int h = 0; h < 2; ++h)
      o[static_cast<int64_t>(tj + 2 * t + h) * DIM + ti + g] = make_double2(cre[q][h] * s, cim[q][h] * s);
  }
}

// Any other dimension (subspace-restricted operators, d = 2, 6, 20, 128, ...):
// one CTA per pair, plain FP64 FMAs with operands through L1/L2, same fused
// norm / null / normalise epilogue. Off the BASELINE configs' hot path.
__global__ void __launch_bounds__(256)
commutator_generic_kernel(const double2* __restrict__ basis, int dim, int64_t g0, int count, double tol,
                          bool normalize, double2* __restrict__ out, double* __restrict__ hnorm,
                          int* __restrict__ is_null) {
  __shared__ double red[8];
  const int j = blockIdx.x;
  if (j >= count) return;
  int64_t l, m;
  pair_from_index(g0 + j, l, m);
  const int64_t D2 = static_cast<int64_t>(dim) * dim;
  const double2* pa = basis + l * D2;
  const double2* pb = basis + m * D2;
  double2* o = out + static_cast<int64_t>(j) * D2;
  double sumsq = 0.0;
  for (int64_t e = threadIdx.x; e < D2; e += blockDim.x) {
    const int i = static_cast<int>(e % dim), c = static_cast<int>(e / dim);
    double re = 0.0, im = 0.0;
    for (int k = 0; k < dim; ++k) {
      const double2 aik = pa[i + static_cast<int64_t>(k) * dim], bkc = pb[k + static_cast<int64_t>(c) * dim];
      const double2 bik = pb[i + static_cast<int64_t>(k) * dim], akc = pa[k + static_cast<int64_t>(c) * dim];
      re += aik.x * bkc.x - aik.y * bkc.y - (bik.x * akc.x - bik.y * akc.y);
      im += aik.x * bkc.y + aik.y * bkc.x - (bik.x * akc.y + bik.y * akc.x);
    }
    o[e] = make_double2(re, im);
    sumsq += re * re + im * im;
  }
  sumsq = warp_sum(sumsq);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sumsq;
  __syncthreads();
  double total = 0.0;
  for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) total += red[w];
  const double hn = sqrt(total) / sqrt(static_cast<double>(dim));
  const bool nul = !(hn > tol);
  if (threadIdx.x == 0) {
    hnorm[j] = hn;
    is_null[j] = nul ? 1 : 0;
  }
  if (!normalize) return;
  const double s = nul ? 0.0 : 1.0 / hn;
  for (int64_t e = threadIdx.x; e < D2; e += blockDim.x) {
    const double2 v = o[e];
    o[e] = make_double2(v.x * s, v.y * s);
  }
}

} // namespace liecl_b200
