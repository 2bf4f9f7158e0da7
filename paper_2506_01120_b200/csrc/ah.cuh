// Anti-Hermitian (su(d) / u(d)) path: packed-real layout kernels.
//
// Packed layout of an anti-Hermitian d x d matrix A (d^2 reals, column-major
// like the complex vec layout): M(i,j) = Re A(i,j) and M(j,i) = Im A(i,j) for
// i < j, M(i,i) = Im A(i,i). The reference inner product is
// <A,B> = (1/d) sum_k w_k M_A(k) M_B(k) with w = 2 off the diagonal, 1 on it,
// and ||A||^2 = <A,A> -- the same numbers the complex formulas give
// (R:src/dense.cpp:53-63) for anti-Hermitian inputs.
//
// The commutator of two anti-Hermitian matrices needs one complex product:
// with P = A B, B A = (A B)^dagger, so h = P - P^dagger (R:src/dense.cpp:65-68),
// and h is again anti-Hermitian: half the flops of the general kernel.
#pragma once

#include "commutator.cuh"
#include "common.cuh"

namespace liecl_b200 {

// exact structure test: x(j,i) == -conj(x(i,j)) for all i <= j (diag: Re == 0)
__global__ void antiherm_violations_kernel(const double2* __restrict__ x, int64_t count, int d,
                                           unsigned long long* __restrict__ viol) {
  const int64_t D2 = static_cast<int64_t>(d) * d;
  const int64_t total = count * D2;
  unsigned long long bad = 0;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / D2, k = e % D2;
    const int i = static_cast<int>(k % d), j = static_cast<int>(k / d);
    if (i > j) continue;
    const double2 a = x[c * D2 + i + static_cast<int64_t>(j) * d];
    const double2 b = x[c * D2 + j + static_cast<int64_t>(i) * d];
    if (!(b.x == -a.x && b.y == a.y)) ++bad;
  }
  if (bad) atomicAdd(viol, bad);
}

__global__ void pack_ah_kernel(const double2* __restrict__ in, int64_t count, int d, double* __restrict__ out) {
  const int64_t D2 = static_cast<int64_t>(d) * d;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < count * D2;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / D2, k = e % D2;
    const int i = static_cast<int>(k % d), j = static_cast<int>(k / d);
    double v;
    if (i < j) v = in[c * D2 + k].x;                                   // Re A(i,j)
    else if (i > j) v = in[c * D2 + j + static_cast<int64_t>(i) * d].y;  // Im A(j,i)
    else v = in[c * D2 + k].y;                                         // Im A(i,i)
    out[e] = v;
  }
}

__global__ void unpack_ah_kernel(const double* __restrict__ in, int64_t count, int d, double2* __restrict__ out) {
  const int64_t D2 = static_cast<int64_t>(d) * d;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < count * D2;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / D2, k = e % D2;
    const int i = static_cast<int>(k % d), j = static_cast<int>(k / d);
    const double* m = in + c * D2;
    double2 v;
    if (i < j) v = make_double2(m[k], m[j + static_cast<int64_t>(i) * d]);
    else if (i > j) v = make_double2(-m[j + static_cast<int64_t>(i) * d], m[k]);
    else v = make_double2(0.0, m[k]);
    out[e] = v;
  }
}

// weighted column norms: out[j] = sqrt(sum_k w_k x_k^2) / sqrt(d)
__global__ void column_norm_ah_kernel(const double* __restrict__ x, int d, double* __restrict__ out) {
  __shared__ double red[32];
  const int64_t D2 = static_cast<int64_t>(d) * d;
  const double* c = x + static_cast<int64_t>(blockIdx.x) * D2;
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < D2; e += blockDim.x) s += ((e % (d + 1)) == 0 ? 1.0 : 2.0) * c[e] * c[e];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) out[blockIdx.x] = sqrt(v) / sqrt(static_cast<double>(d));
  }
}

// out = x * (1/nrm) per column (null: zeros)
__global__ void scale_columns_ah_kernel(const double* __restrict__ x, const double* __restrict__ nrm, double tol,
                                        int64_t D2, double* __restrict__ out) {
  const int j = blockIdx.y;
  const double n = nrm[j];
  const double s = n > tol ? 1.0 / n : 0.0;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < D2;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[static_cast<int64_t>(j) * D2 + e] = x[static_cast<int64_t>(j) * D2 + e] * s;
}

// K3 on the packed path: V slot = r * s, Vw slot = w .* (r * s) (exact
// doubling), originals slot = h_unit copy (Alg. 3).
__global__ void append_ah_kernel(const double* __restrict__ src, double s, int d, double* __restrict__ v,
                                 double* __restrict__ vw, const double* __restrict__ orig_src,
                                 double* __restrict__ orig_dst) {
  const int64_t D2 = static_cast<int64_t>(d) * d;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < D2;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double x = src[e] * s;
    v[e] = x;
    vw[e] = ((e % (d + 1)) == 0 ? 1.0 : 2.0) * x;
    if (orig_dst) orig_dst[e] = orig_src[e];
  }
}

// Vw = w .* V for n packed vectors (set_basis on the packed path)
__global__ void weight_ah_kernel(const double* __restrict__ v, int64_t count, int d, double* __restrict__ vw) {
  const int64_t D2 = static_cast<int64_t>(d) * d;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < count * D2;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    vw[e] = (((e % D2) % (d + 1)) == 0 ? 1.0 : 2.0) * v[e];
}

// VT[m * ldvt + k] = V[k * D + m] for basis rows k in [k0, k1): the transposed
// (K-contiguous) copy K2b reads through TMA (dense_engine.cuh ensure_vt).
// 32 x 32 tiles through shared memory, both sides coalesced.
__global__ void transpose_rows_kernel(const double* __restrict__ V, int64_t D, int64_t k0, int64_t k1,
                                      double* __restrict__ VT, int64_t ldvt) {
  __shared__ double tile[32][33];
  const int64_t kb = k0 + static_cast<int64_t>(blockIdx.y) * 32, mb = static_cast<int64_t>(blockIdx.x) * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t k = kb + r, m = mb + threadIdx.x;
    tile[r][threadIdx.x] = (k < k1 && m < D) ? V[k * D + m] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t m = mb + r, k = kb + threadIdx.x;
    if (m < D && k < k1) VT[m * ldvt + k] = tile[threadIdx.x][r];
  }
}

// Warp layout of one pair's product P = A B (TR x TR tiles of 8 x 8): a warp
// owns WR x WC tiles (WR row tiles sharing A fragments, WC column tiles
// sharing B fragments). d < 64: one row of tiles per warp, several pairs per
// CTA; d = 64: eight warps per pair, WR x WC per warp (default 2 x 4: 12
// fragment loads per 32 DMMAs, 64 accumulator registers).
template <int DIM, int WR_ = (DIM == 64 ? 2 : 1), int WC_ = (DIM == 64 ? 4 : DIM / 8)> struct CommAhShape {
  static constexpr int TR = DIM / 8;                 // tile rows (and columns)
  static constexpr int WR = WR_, WC = WC_;
  static constexpr int WARPS_PER_PAIR = (TR / WR) * (TR / WC);
  static constexpr int CTA_WARPS = WARPS_PER_PAIR > 8 ? WARPS_PER_PAIR : 8;  // 256 threads, or one pair
  static constexpr int THREADS = 32 * CTA_WARPS;
  static_assert(CTA_WARPS % WARPS_PER_PAIR == 0, "warp layout");
  static constexpr int PAIRS_PER_CTA = CTA_WARPS / WARPS_PER_PAIR;
  static constexpr int LDP = DIM + 4;                // == 4 (mod 16): conflict-free fragment gathers
  static constexpr int PACKED = DIM * LDP;
  static constexpr int SMEM_PER_PAIR = (2 * PACKED * 8 + WARPS_PER_PAIR * 8 + 15) / 16 * 16;  // 16-byte slots
  static constexpr int SMEM = PAIRS_PER_CTA * SMEM_PER_PAIR;
};

// P-plane offset of (r, c): the fragment writes (rows g, columns 2t + h), the
// row reads and the column reads of the epilogue are all conflict-free with
// the XOR swizzle c ^ sw(r), sw(r) = r & 7 | ((r >> 1 ^ r >> 3) & 1) << 3 on the
// low four column bits (found by exhaustive search over GF(2) row maps; a
// plain padded stride leaves the writes 3-4-way conflicted). d < 16: padded.
template <int DIM> __device__ __forceinline__ int p_at(int r, int c) {
  if constexpr (DIM >= 16) return r * DIM + (c ^ ((r & 7) | ((((r >> 1) ^ (r >> 3)) & 1) << 3)));
  else return r * (DIM + 1) + c;
}

// complex element (i, k) of the anti-Hermitian matrix stored packed at p (stride LDP)
template <int LDP>
__device__ __forceinline__ void ah_elem(const double* p, int i, int k, double& re, double& im) {
  const double u = p[i + k * LDP], v = p[k + i * LDP];
  if (i < k) { re = u; im = v; }
  else if (i > k) { re = -v; im = u; }
  else { re = 0.0; im = u; }
}

// One pair's pieces, shared by the kernels below (same arithmetic in the same
// order, so every variant gives bit-identical h and norms).
//
// Operands of pair `pair` into pa / pb (stride LDP): 16-byte pieces (DIM
// even; i even and LDP even keep them 16-byte aligned in shared memory).
// cp.async issues every piece before waiting: one memory latency per pair.
template <int DIM, int LDP, int NT, bool ASYNC>
__device__ __forceinline__ void ah_load_pair(const double* __restrict__ basis, int64_t pair, double* pa, double* pb,
                                             int tip) {
  constexpr int D2 = DIM * DIM;
  int64_t l, m;
  pair_from_index(pair, l, m);
  const double2* ga = reinterpret_cast<const double2*>(basis + l * D2);
  const double2* gb = reinterpret_cast<const double2*>(basis + m * D2);
#pragma unroll
  for (int e = tip; e < D2 / 2; e += NT) {
    const int i = (2 * e) % DIM, k = (2 * e) / DIM;
    if constexpr (ASYNC) {
      cp_async16(pa + i + k * LDP, ga + e, 16);
      cp_async16(pb + i + k * LDP, gb + e, 16);
    } else {
      const double2 va = ga[e], vb = gb[e];
      *reinterpret_cast<double2*>(pa + i + k * LDP) = va;
      *reinterpret_cast<double2*>(pb + i + k * LDP) = vb;
    }
  }
  if constexpr (ASYNC) {
    cp_async_commit();
    cp_async_wait<0>();
  }
}

// This warp's WR x WC tiles of P = A B, fragments gathered straight from the
// packed inputs (A fragments reused across the WC column tiles, B fragments
// across the WR row tiles).
template <int DIM, int LDP, int WR, int WC>
__device__ __forceinline__ void ah_product(const double* pa, const double* pb, int wr0, int wc0, int g, int t,
                                           double (&cre)[WR][WC][2], double (&cim)[WR][WC][2]) {
#pragma unroll 2
  for (int k0 = 0; k0 < DIM; k0 += 4) {
    const int k = k0 + t;
    double br[WC], bi[WC], ar[WR], ai[WR];
#pragma unroll
    for (int c = 0; c < WC; ++c) ah_elem<LDP>(pb, k, (wc0 + c) * 8 + g, br[c], bi[c]);  // B(k, tj + g)
#pragma unroll
    for (int r = 0; r < WR; ++r) ah_elem<LDP>(pa, (wr0 + r) * 8 + g, k, ar[r], ai[r]);  // A(ti + g, k)
    // four sweeps over the warp's tiles: two DMMAs into the same
    // accumulator are WR*WC*2 - 1 instructions apart (no back-to-back
    // dependency on the DMMA latency); each accumulator still adds its
    // terms in the same order (re: ar br, then -ai bi; im: ar bi, then ai br)
#pragma unroll
    for (int r = 0; r < WR; ++r)
#pragma unroll
      for (int c = 0; c < WC; ++c) dmma_8x8x4(cre[r][c][0], cre[r][c][1], ar[r], br[c]);
#pragma unroll
    for (int r = 0; r < WR; ++r)
#pragma unroll
      for (int c = 0; c < WC; ++c) dmma_8x8x4(cim[r][c][0], cim[r][c][1], ar[r], bi[c]);
#pragma unroll
    for (int r = 0; r < WR; ++r)
#pragma unroll
      for (int c = 0; c < WC; ++c) dmma_8x8x4(cre[r][c][0], cre[r][c][1], -ai[r], bi[c]);
#pragma unroll
    for (int r = 0; r < WR; ++r)
#pragma unroll
      for (int c = 0; c < WC; ++c) dmma_8x8x4(cim[r][c][0], cim[r][c][1], ai[r], br[c]);
  }
}

// P(i, k) re at pre[p_at(i, k)]: the epilogue reads P(k, i) along a row and
// P(i, k) down a column
template <int DIM, int WR, int WC>
__device__ __forceinline__ void ah_store_p(double* pre, double* pim, int wr0, int wc0, int g, int t,
                                           const double (&cre)[WR][WC][2], const double (&cim)[WR][WC][2]) {
#pragma unroll
  for (int r = 0; r < WR; ++r) {
    const int ti = (wr0 + r) * 8;
#pragma unroll
    for (int c = 0; c < WC; ++c)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        pre[p_at<DIM>(ti + g, (wc0 + c) * 8 + 2 * t + h)] = cre[r][c][h];
        pim[p_at<DIM>(ti + g, (wc0 + c) * 8 + 2 * t + h)] = cim[r][c][h];
      }
  }
}

// packed h = P - P^dagger for this thread's elements; returns its part of sum w h^2
template <int DIM, int NT>
__device__ __forceinline__ double ah_h_values(const double* pre, const double* pim, int tip,
                                              double (&hv)[(DIM * DIM + NT - 1) / NT]) {
  constexpr int D2 = DIM * DIM;
  double sumsq = 0.0;
#pragma unroll
  for (int q = 0; q < (D2 + NT - 1) / NT; ++q) {
    const int e = tip + q * NT;
    if (e >= D2) break;
    const int i = e % DIM, k = e / DIM;
    double v;
    if (i < k) v = pre[p_at<DIM>(i, k)] - pre[p_at<DIM>(k, i)];
    else if (i > k) v = pim[p_at<DIM>(k, i)] + pim[p_at<DIM>(i, k)];
    else v = 2.0 * pim[p_at<DIM>(i, i)];
    hv[q] = v;
    sumsq += (i == k ? 1.0 : 2.0) * v * v;
  }
  return sumsq;
}

// norm, null flag and the (normalised) packed h of pair j from the warps' partial sums
template <int DIM, int NT, int WARPS>
__device__ __forceinline__ void ah_finish(const double* red, const double (&hv)[(DIM * DIM + NT - 1) / NT], int j,
                                          int tip, double tol, bool normalize, double* __restrict__ out,
                                          double* __restrict__ hnorm, int* __restrict__ is_null) {
  constexpr int D2 = DIM * DIM;
  double total = 0.0;
#pragma unroll
  for (int w = 0; w < WARPS; ++w) total += red[w];
  const double hn = sqrt(total) / sqrt(static_cast<double>(DIM));
  const bool nul = !(hn > tol);
  if (tip == 0) {
    hnorm[j] = hn;
    is_null[j] = nul ? 1 : 0;
  }
  const double sc = !normalize ? 1.0 : (nul ? 0.0 : 1.0 / hn);
  double* o = out + static_cast<int64_t>(j) * D2;
#pragma unroll
  for (int q = 0; q < (D2 + NT - 1) / NT; ++q) {
    const int e = tip + q * NT;
    if (e < D2) o[e] = hv[q] * sc;
  }
}

// K1 on the packed path: pairs [g0, g0+count) of the packed commutator basis;
// writes packed h_unit, ||h||, null flag. One DMMA product P = A B per pair;
// P is written back over the consumed inputs and h = P - P^dagger is read out
// in the packed layout. ~70 KB per pair at d = 64.
template <int DIM, int MINB = 2, int WR = CommAhShape<DIM>::WR, int WC = CommAhShape<DIM>::WC, bool ASYNC = true>
__global__ void __launch_bounds__(CommAhShape<DIM, WR, WC>::THREADS, MINB)
commutator_ah_kernel(const double* __restrict__ basis, int64_t g0, int count, double tol, bool normalize,
                     double* __restrict__ out, double* __restrict__ hnorm, int* __restrict__ is_null) {
  using S = CommAhShape<DIM, WR, WC>;
  constexpr int D2 = DIM * DIM;
  constexpr int LDP = S::LDP;
  constexpr int NT = S::WARPS_PER_PAIR * 32;
  extern __shared__ __align__(16) double csm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int slot = warp / S::WARPS_PER_PAIR;
  const int wip = warp % S::WARPS_PER_PAIR;
  const int wr0 = (wip / (S::TR / WC)) * WR;  // first row tile of this warp
  const int wc0 = (wip % (S::TR / WC)) * WC;  // first column tile
  const int j = blockIdx.x * S::PAIRS_PER_CTA + slot;
  const bool active = j < count;
  const int tip = threadIdx.x - slot * NT;

  double* pa = csm + slot * (S::SMEM_PER_PAIR / 8);
  double* pb = pa + S::PACKED;
  double* red = pb + S::PACKED;

  if (active) ah_load_pair<DIM, LDP, NT, ASYNC>(basis, g0 + j, pa, pb, tip);
  __syncthreads();

  double cre[WR][WC][2], cim[WR][WC][2];
#pragma unroll
  for (int r = 0; r < WR; ++r)
#pragma unroll
    for (int c = 0; c < WC; ++c) cre[r][c][0] = cre[r][c][1] = cim[r][c][0] = cim[r][c][1] = 0.0;
  if (active) ah_product<DIM, LDP, WR, WC>(pa, pb, wr0, wc0, g, t, cre, cim);
  __syncthreads();  // inputs consumed: P planes reuse the packed buffers
  if (active) ah_store_p<DIM, WR, WC>(pa, pb, wr0, wc0, g, t, cre, cim);
  __syncthreads();
  double hv[(D2 + NT - 1) / NT];
  double sumsq = active ? ah_h_values<DIM, NT>(pa, pb, tip, hv) : 0.0;
  sumsq = warp_sum(sumsq);
  if (lane == 0) red[wip] = sumsq;
  __syncthreads();
  if (!active) return;
  ah_finish<DIM, NT, S::WARPS_PER_PAIR>(red, hv, j, tip, tol, normalize, out, hnorm, is_null);
}

// K1 of a D-sharded rank ("GPU p computes only the columns
// J_p of h"): packed columns [8 tc0, 8 tc1) of h = P - P^dagger, i.e. packed
// elements [64 * 8 tc0, 64 * 8 tc1) at d = 64. They need P's tile columns
// [tc0, tc1) and tile rows [tc0, tc1) only: 8w + w(8 - w) of the 64 tiles for
// w = tc1 - tc0 (15 at eight ranks). Tiles go round-robin over the eight
// warps, up to six per warp, each accumulating in the engine kernel's order
// (re: ar br, then -ai bi; im: ar bi, then ai br), so the unnormalised slice
// has the bits of the whole-operator kernel. Writes the UNNORMALISED slice
// and this rank's part of sum w h^2; the norm is a sum over ranks
// (commutator_ah_cols_finish_kernel).
template <int DIM>
__global__ void __launch_bounds__(256, 2)
commutator_ah_cols_kernel(const double* __restrict__ basis, int64_t g0, int count, int tc0, int tc1,
                          double* __restrict__ out, double* __restrict__ sumsq_out) {
  static_assert(DIM == 64, "tile bookkeeping below is for 8 x 8 tiles");
  using S = CommAhShape<DIM, 2, 4>;
  constexpr int D2 = DIM * DIM, LDP = S::LDP, NT = 256, TR = 8, MAXT = 6;
  extern __shared__ __align__(16) double csm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int j = blockIdx.x, tip = threadIdx.x;
  if (j >= count) return;
  double* pa = csm;
  double* pb = pa + S::PACKED;
  double* red = pb + S::PACKED;
  const int w = tc1 - tc0, ntile = TR * w + w * (TR - w);
  auto tile_of = [&](int idx, int& r, int& c) {
    if (idx < TR * w) {  // the tile columns of the slice
      r = idx % TR;
      c = tc0 + idx / TR;
    } else {  // the rest of its tile rows
      const int u = idx - TR * w, cc = u % (TR - w);
      r = tc0 + u / (TR - w);
      c = cc < tc0 ? cc : cc + w;
    }
  };
  ah_load_pair<DIM, LDP, NT, true>(basis, g0 + j, pa, pb, tip);
  __syncthreads();
  double cre[MAXT][2], cim[MAXT][2];
#pragma unroll
  for (int q = 0; q < MAXT; ++q) cre[q][0] = cre[q][1] = cim[q][0] = cim[q][1] = 0.0;
#pragma unroll
  for (int q = 0; q < MAXT; q += 2) {  // two tiles at a time: independent accumulators
    const int i0 = warp + 8 * q, i1 = warp + 8 * (q + 1);
    if (i0 >= ntile) break;
    int r0, c0, r1 = 0, c1 = 0;
    tile_of(i0, r0, c0);
    const bool two = i1 < ntile;
    if (two) tile_of(i1, r1, c1);
    for (int k0 = 0; k0 < DIM; k0 += 4) {
      const int k = k0 + t;
      double ar, ai, br, bi;
      ah_elem<LDP>(pa, r0 * 8 + g, k, ar, ai);
      ah_elem<LDP>(pb, k, c0 * 8 + g, br, bi);
      dmma_8x8x4(cre[q][0], cre[q][1], ar, br);
      dmma_8x8x4(cim[q][0], cim[q][1], ar, bi);
      dmma_8x8x4(cre[q][0], cre[q][1], -ai, bi);
      dmma_8x8x4(cim[q][0], cim[q][1], ai, br);
      if (two) {
        ah_elem<LDP>(pa, r1 * 8 + g, k, ar, ai);
        ah_elem<LDP>(pb, k, c1 * 8 + g, br, bi);
        dmma_8x8x4(cre[q + 1][0], cre[q + 1][1], ar, br);
        dmma_8x8x4(cim[q + 1][0], cim[q + 1][1], ar, bi);
        dmma_8x8x4(cre[q + 1][0], cre[q + 1][1], -ai, bi);
        dmma_8x8x4(cim[q + 1][0], cim[q + 1][1], ai, br);
      }
    }
  }
  __syncthreads();  // inputs consumed: the P planes reuse the packed buffers
#pragma unroll
  for (int q = 0; q < MAXT; ++q) {
    const int idx = warp + 8 * q;
    if (idx < ntile) {
      int r, c;
      tile_of(idx, r, c);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        pa[p_at<DIM>(r * 8 + g, c * 8 + 2 * t + h)] = cre[q][h];
        pb[p_at<DIM>(r * 8 + g, c * 8 + 2 * t + h)] = cim[q][h];
      }
    }
  }
  __syncthreads();
  // packed elements of columns [8 tc0, 8 tc1): e = i + k * DIM
  const int e0 = tc0 * 8 * DIM, ne = w * 8 * DIM;
  double sumsq = 0.0;
  double* o = out + static_cast<int64_t>(j) * D2 + e0;
  for (int x = tip; x < ne; x += NT) {
    const int e = e0 + x, i = e % DIM, k = e / DIM;
    double v;
    if (i < k) v = pa[p_at<DIM>(i, k)] - pa[p_at<DIM>(k, i)];
    else if (i > k) v = pb[p_at<DIM>(k, i)] + pb[p_at<DIM>(i, k)];
    else v = 2.0 * pb[p_at<DIM>(i, i)];
    o[x] = v;
    sumsq += (i == k ? 1.0 : 2.0) * v * v;
  }
  sumsq = warp_sum(sumsq);
  if (lane == 0) red[warp] = sumsq;
  __syncthreads();
  if (tip == 0) {
    double total = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) total += red[q];
    sumsq_out[j] = total;
  }
}

// After the sum of sumsq over ranks: ||h||, the null flag, and the slice
// [e0, e0 + ne) of every bracket scaled by 1/||h|| (null: zeros), as the
// whole-operator kernel's epilogue does.
__global__ void commutator_ah_cols_finish_kernel(const double* __restrict__ sumsq, int d, double tol, int64_t e0,
                                                 int64_t ne, double* __restrict__ out, double* __restrict__ hnorm,
                                                 int* __restrict__ is_null) {
  const int j = blockIdx.y;
  const double hn = sqrt(sumsq[j]) / sqrt(static_cast<double>(d));
  const bool nul = !(hn > tol);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    hnorm[j] = hn;
    is_null[j] = nul ? 1 : 0;
  }
  const double sc = nul ? 0.0 : 1.0 / hn;
  double* o = out + static_cast<int64_t>(j) * d * d + e0;
  for (int64_t x = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; x < ne;
       x += static_cast<int64_t>(gridDim.x) * blockDim.x)
    o[x] *= sc;
}

// packed path, any even d: one CTA per pair, operands through L1/L2
__global__ void __launch_bounds__(256)
commutator_ah_generic_kernel(const double* __restrict__ basis, int dim, int64_t g0, int count, double tol,
                             bool normalize, double* __restrict__ out, double* __restrict__ hnorm,
                             int* __restrict__ is_null) {
  __shared__ double red[8];
  const int j = blockIdx.x;
  if (j >= count) return;
  int64_t l, m;
  pair_from_index(g0 + j, l, m);
  const int64_t D2 = static_cast<int64_t>(dim) * dim;
  const double* ma = basis + l * D2;
  const double* mb = basis + m * D2;
  auto elem = [&](const double* mp, int i, int k, double& re, double& im) {
    if (i < k) { re = mp[i + static_cast<int64_t>(k) * dim]; im = mp[k + static_cast<int64_t>(i) * dim]; }
    else if (i > k) { re = -mp[k + static_cast<int64_t>(i) * dim]; im = mp[i + static_cast<int64_t>(k) * dim]; }
    else { re = 0.0; im = mp[i + static_cast<int64_t>(i) * dim]; }
  };
  // P(i,k) = sum_q A(i,q) B(q,k); packed h needs P(i,k) and P(k,i)
  auto pval = [&](int i, int k, double& re, double& im) {
    re = 0.0;
    im = 0.0;
    for (int q = 0; q < dim; ++q) {
      double ar, ai, br, bi;
      elem(ma, i, q, ar, ai);
      elem(mb, q, k, br, bi);
      re += ar * br - ai * bi;
      im += ar * bi + ai * br;
    }
  };
  double* o = out + static_cast<int64_t>(j) * D2;
  double sumsq = 0.0;
  for (int64_t e = threadIdx.x; e < D2; e += blockDim.x) {
    const int i = static_cast<int>(e % dim), k = static_cast<int>(e / dim);
    double r1, i1, r2, i2;
    double v;
    if (i < k) { pval(i, k, r1, i1); pval(k, i, r2, i2); v = r1 - r2; }
    else if (i > k) { pval(k, i, r1, i1); pval(i, k, r2, i2); v = i1 + i2; }
    else { pval(i, i, r1, i1); v = 2.0 * i1; }
    o[e] = v;
    sumsq += (i == k ? 1.0 : 2.0) * v * v;
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
  for (int64_t e = threadIdx.x; e < D2; e += blockDim.x) o[e] *= s;
}

} // namespace liecl_b200
