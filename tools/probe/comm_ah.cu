// Probe: warp layouts / register bounds of commutator_ah_kernel<64> on a
// random packed anti-Hermitian basis (4095 x 4096), 8192 cursor pairs from
// row 1024 (a saturated-window batch). Prints ms and TFLOP/s (8 d^3 per pair)
// per variant; every variant must give bit-identical h and norms.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o comm_ah comm_ah.cu
#include <cstdio>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <vector>

#include "../../paper_2506_01120_b200/csrc/ah.cuh"

using namespace liecl_b200;

// ---- experiment: a ping-pong K1 (measured slower than the engine kernel; kept here, not in the product) ----
namespace liecl_b200 {
// Named barriers of the ping-pong kernel (0 is __syncthreads).
__device__ __forceinline__ void named_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int threads) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(threads) : "memory");
}

// packed h(i, k) from the P planes (the same expression as ah_h_values)
template <int DIM>
__device__ __forceinline__ double ah_h_at(const double* pre, const double* pim, int i, int k) {
  if (i < k) return pre[p_at<DIM>(i, k)] - pre[p_at<DIM>(k, i)];
  if (i > k) return pim[p_at<DIM>(k, i)] + pim[p_at<DIM>(i, k)];
  return 2.0 * pim[p_at<DIM>(i, i)];
}

// One group's loop of the ping-pong kernel (GRP constant: the named barrier
// ids are immediates). The epilogue reads h from the P planes twice (norm,
// then scaled store) instead of holding it in registers across the reduction.
template <int DIM, int GRP>
__device__ __forceinline__ void ah_pp_group(const double* __restrict__ basis, int64_t g0, int count, double tol,
                                            bool normalize, double* __restrict__ out, double* __restrict__ hnorm,
                                            int* __restrict__ is_null, double* csm) {
  using S = CommAhShape<DIM>;
  constexpr int D2 = DIM * DIM;
  constexpr int NT = 256;
  constexpr int BAR_TURN = 1 + GRP, BAR_GIVE = 2 - GRP, BAR_GRP = 3 + GRP;
  const int warp = (threadIdx.x >> 5) & 7, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wr0 = (warp / (S::TR / S::WC)) * S::WR;
  const int wc0 = (warp % (S::TR / S::WC)) * S::WC;
  const int tip = threadIdx.x & (NT - 1);
  double* pa = csm + GRP * (S::SMEM_PER_PAIR / 8);
  double* pb = pa + S::PACKED;
  double* red = pb + S::PACKED;
  const int n_it = (count + 2 * static_cast<int>(gridDim.x) - 1) / (2 * static_cast<int>(gridDim.x));
  if (GRP == 1 && n_it > 0) named_arrive(1, 512);  // group 0 multiplies first
  for (int it = 0; it < n_it; ++it) {
    const int j = (it * static_cast<int>(gridDim.x) + static_cast<int>(blockIdx.x)) * 2 + GRP;
    const bool active = j < count;
    if (active) ah_load_pair<DIM, S::LDP, NT, true>(basis, g0 + j, pa, pb, tip);
    named_sync(BAR_GRP, NT);   // operands visible to the group
    named_sync(BAR_TURN, 512);  // the pipe is ours
    double cre[S::WR][S::WC][2], cim[S::WR][S::WC][2];
#pragma unroll
    for (int r = 0; r < S::WR; ++r)
#pragma unroll
      for (int c = 0; c < S::WC; ++c) cre[r][c][0] = cre[r][c][1] = cim[r][c][0] = cim[r][c][1] = 0.0;
    if (active) ah_product<DIM, S::LDP, S::WR, S::WC>(pa, pb, wr0, wc0, g, t, cre, cim);
    // hand the pipe over (group 1's last hand-over would have no taker)
    if (!(GRP == 1 && it == n_it - 1)) named_arrive(BAR_GIVE, 512);
    named_sync(BAR_GRP, NT);  // inputs consumed: P planes reuse the pair buffer
    if (active) ah_store_p<DIM, S::WR, S::WC>(pa, pb, wr0, wc0, g, t, cre, cim);
    named_sync(BAR_GRP, NT);
    double sumsq = 0.0;
    if (active) {
#pragma unroll 4
      for (int e = tip; e < D2; e += NT) {
        const int i = e % DIM, k = e / DIM;
        const double v = ah_h_at<DIM>(pa, pb, i, k);
        sumsq += (i == k ? 1.0 : 2.0) * v * v;
      }
    }
    sumsq = warp_sum(sumsq);
    if (lane == 0) red[warp] = sumsq;
    named_sync(BAR_GRP, NT);
    if (active) {
      double total = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) total += red[w];
      const double hn = sqrt(total) / sqrt(static_cast<double>(DIM));
      const bool nul = !(hn > tol);
      if (tip == 0) {
        hnorm[j] = hn;
        is_null[j] = nul ? 1 : 0;
      }
      const double sc = !normalize ? 1.0 : (nul ? 0.0 : 1.0 / hn);
      double* o = out + static_cast<int64_t>(j) * D2;
#pragma unroll 4
      for (int e = tip; e < D2; e += NT) o[e] = ah_h_at<DIM>(pa, pb, e % DIM, e / DIM) * sc;
    }
    named_sync(BAR_GRP, NT);  // P planes and red read before the next load
  }
}

// K1 at d = 64, ping-pong: one persistent 512-thread CTA per SM holding two
// 8-warp groups, each with its own ~70 KB pair buffer. The groups take turns
// on the DMMA pipe (named barriers 1 and 2 hand the turn over), so one group's
// operand load, P write-back and epilogue run while the other group's product
// runs. With two independent 256-thread CTAs per SM both CTAs drift into the
// same phase (load together, multiply together at half rate, epilogue
// together) and the pipe idles during the shared load/epilogue phases.
// Pair j = (it * gridDim.x + blockIdx.x) * 2 + group; per pair the arithmetic
// is commutator_ah_kernel's (bit-identical results). Dynamic shared memory:
// 2 * CommAhShape<DIM>::SMEM_PER_PAIR.
template <int DIM>
__global__ void __launch_bounds__(512, 1)
commutator_ah_pp_kernel(const double* __restrict__ basis, int64_t g0, int count, double tol, bool normalize,
                        double* __restrict__ out, double* __restrict__ hnorm, int* __restrict__ is_null) {
  using S = CommAhShape<DIM>;
  static_assert(S::WARPS_PER_PAIR == 8 && S::PAIRS_PER_CTA == 1, "ping-pong groups are one 8-warp pair each");
  extern __shared__ __align__(16) double csm[];
  if (threadIdx.x < 256) ah_pp_group<DIM, 0>(basis, g0, count, tol, normalize, out, hnorm, is_null, csm);
  else ah_pp_group<DIM, 1>(basis, g0, count, tol, normalize, out, hnorm, is_null, csm);
}

}  // namespace liecl_b200

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int DIM = 64, D2 = DIM * DIM, NB = 4095, CNT = 8192;

// ---- phase clocks of the engine kernel (thread 0 of every CTA): load, product, P store, h values, finish
template <int MINB>
__global__ void __launch_bounds__(256, MINB)
commutator_ah_clock_kernel(const double* __restrict__ basis, int64_t g0, int count, double tol, double* __restrict__ out,
                           double* __restrict__ hnorm, int* __restrict__ is_null, long long* __restrict__ clk) {
  using S = CommAhShape<DIM, 2, 4>;
  constexpr int LDP = S::LDP, NT = 256, WR = 2, WC = 4;
  extern __shared__ __align__(16) double csm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int wr0 = (warp / (S::TR / WC)) * WR, wc0 = (warp % (S::TR / WC)) * WC;
  const int j = blockIdx.x, tip = threadIdx.x;
  double* pa = csm;
  double* pb = pa + S::PACKED;
  double* red = pb + S::PACKED;
  long long c[7];
  c[0] = clock64();
  ah_load_pair<DIM, LDP, NT, true>(basis, g0 + j, pa, pb, tip);
  __syncthreads();
  c[1] = clock64();
  double cre[WR][WC][2], cim[WR][WC][2];
#pragma unroll
  for (int r = 0; r < WR; ++r)
#pragma unroll
    for (int cc = 0; cc < WC; ++cc) cre[r][cc][0] = cre[r][cc][1] = cim[r][cc][0] = cim[r][cc][1] = 0.0;
  ah_product<DIM, LDP, WR, WC>(pa, pb, wr0, wc0, g, t, cre, cim);
  c[2] = clock64();
  __syncthreads();
  c[3] = clock64();
  ah_store_p<DIM, WR, WC>(pa, pb, wr0, wc0, g, t, cre, cim);
  __syncthreads();
  c[4] = clock64();
  double hv[(D2 + NT - 1) / NT];
  double sumsq = ah_h_values<DIM, NT>(pa, pb, tip, hv);
  sumsq = warp_sum(sumsq);
  if (lane == 0) red[warp] = sumsq;
  __syncthreads();
  c[5] = clock64();
  ah_finish<DIM, NT, 8>(red, hv, j, tip, tol, true, out, hnorm, is_null);
  c[6] = clock64();
  if (threadIdx.x == 0)
    for (int q = 0; q < 7; ++q) clk[static_cast<int64_t>(blockIdx.x) * 7 + q] = c[q];
}

// ---- experiment: the epilogue's FP64 work as independent operations (trees
// instead of the 16-term and 8-term dependent chains); differs from the
// engine kernel in the last bits of the norm
template <int DIM_, int NT>
__device__ __forceinline__ double ah_h_values_tree(const double* pre, const double* pim, int tip,
                                                   double (&hv)[(DIM_ * DIM_ + NT - 1) / NT]) {
  constexpr int D2_ = DIM_ * DIM_, Q = (D2_ + NT - 1) / NT;
  double sq[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int e = tip + q * NT;
    double v = 0.0, w = 0.0;
    if (e < D2_) {
      const int i = e % DIM_, k = e / DIM_;
      if (i < k) v = pre[p_at<DIM_>(i, k)] - pre[p_at<DIM_>(k, i)];
      else if (i > k) v = pim[p_at<DIM_>(k, i)] + pim[p_at<DIM_>(i, k)];
      else v = 2.0 * pim[p_at<DIM_>(i, i)];
      w = i == k ? 1.0 : 2.0;
    }
    hv[q] = v;
    sq[q] = w * (v * v);
  }
#pragma unroll
  for (int s2 = 1; s2 < Q; s2 <<= 1)
#pragma unroll
    for (int q = 0; q + s2 < Q; q += 2 * s2) sq[q] += sq[q + s2];
  return sq[0];
}

// fewest FP64 instructions: S = sum of all v^2 (one DFMA each), the diagonal
// element (at most one per thread) picked by integer selects, thread total
// 2 S - v_diag^2
template <int DIM_, int NT>
__device__ __forceinline__ double ah_h_values_lean(const double* pre, const double* pim, int tip,
                                                   double (&hv)[(DIM_ * DIM_ + NT - 1) / NT]) {
  constexpr int D2_ = DIM_ * DIM_, Q = (D2_ + NT - 1) / NT;
  double s0 = 0.0, s1 = 0.0, vd = 0.0;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int e = tip + q * NT;
    double v = 0.0;
    if (e < D2_) {
      const int i = e % DIM_, k = e / DIM_;
      if (i < k) v = pre[p_at<DIM_>(i, k)] - pre[p_at<DIM_>(k, i)];
      else if (i > k) v = pim[p_at<DIM_>(k, i)] + pim[p_at<DIM_>(i, k)];
      else { v = pim[p_at<DIM_>(i, i)]; v += v; vd = v; }
    }
    hv[q] = v;
    if (q & 1) s1 = fma(v, v, s1);
    else s0 = fma(v, v, s0);
  }
  return fma(2.0, s0 + s1, -(vd * vd));
}

template <int MINB, int VARIANT>
__global__ void __launch_bounds__(256, MINB)
commutator_ah_tree_kernel(const double* __restrict__ basis, int64_t g0, int count, double tol, double* __restrict__ out,
                          double* __restrict__ hnorm, int* __restrict__ is_null) {
  using S = CommAhShape<DIM, 2, 4>;
  constexpr int LDP = S::LDP, NT = 256, WR = 2, WC = 4;
  extern __shared__ __align__(16) double csm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int wr0 = (warp / (S::TR / WC)) * WR, wc0 = (warp % (S::TR / WC)) * WC;
  const int j = blockIdx.x, tip = threadIdx.x;
  double* pa = csm;
  double* pb = pa + S::PACKED;
  double* red = pb + S::PACKED;
  ah_load_pair<DIM, LDP, NT, true>(basis, g0 + j, pa, pb, tip);
  __syncthreads();
  double cre[WR][WC][2], cim[WR][WC][2];
#pragma unroll
  for (int r = 0; r < WR; ++r)
#pragma unroll
    for (int cc = 0; cc < WC; ++cc) cre[r][cc][0] = cre[r][cc][1] = cim[r][cc][0] = cim[r][cc][1] = 0.0;
  ah_product<DIM, LDP, WR, WC>(pa, pb, wr0, wc0, g, t, cre, cim);
  __syncthreads();
  ah_store_p<DIM, WR, WC>(pa, pb, wr0, wc0, g, t, cre, cim);
  __syncthreads();
  double hv[(D2 + NT - 1) / NT];
  double sumsq = VARIANT == 3 ? ah_h_values_lean<DIM, NT>(pa, pb, tip, hv) : ah_h_values_tree<DIM, NT>(pa, pb, tip, hv);
  sumsq = warp_sum(sumsq);
  if (lane == 0) red[warp] = sumsq;
  __syncthreads();
  double hn, sc;
  if (VARIANT == 3) {  // warp partials summed by three shuffle levels, one reciprocal square root
    double total = red[lane & 7];
    total += __shfl_xor_sync(0xffffffffu, total, 1);
    total += __shfl_xor_sync(0xffffffffu, total, 2);
    total += __shfl_xor_sync(0xffffffffu, total, 4);
    const double rs = rsqrt(total);
    hn = total > 0.0 ? (total * rs) * (1.0 / sqrt(static_cast<double>(DIM))) : 0.0;
    sc = !(hn > tol) ? 0.0 : rs * sqrt(static_cast<double>(DIM));
  } else if (VARIANT == 0) {  // every thread: tree over the warp partials, sqrt, reciprocal
    const double total = ((red[0] + red[1]) + (red[2] + red[3])) + ((red[4] + red[5]) + (red[6] + red[7]));
    hn = sqrt(total) / sqrt(static_cast<double>(DIM));
    sc = !(hn > tol) ? 0.0 : 1.0 / hn;
  } else if (VARIANT == 2) {  // one reciprocal square root instead of sqrt and a reciprocal
    const double total = ((red[0] + red[1]) + (red[2] + red[3])) + ((red[4] + red[5]) + (red[6] + red[7]));
    const double rs = rsqrt(total);
    hn = total > 0.0 ? (total * rs) * (1.0 / sqrt(static_cast<double>(DIM))) : 0.0;
    sc = !(hn > tol) ? 0.0 : rs * sqrt(static_cast<double>(DIM));
  } else {  // one thread computes norm and scale, the rest pick them up
    if (threadIdx.x == 0) {
      const double total = ((red[0] + red[1]) + (red[2] + red[3])) + ((red[4] + red[5]) + (red[6] + red[7]));
      const double h1 = sqrt(total) / sqrt(static_cast<double>(DIM));
      red[8] = h1;
      red[9] = !(h1 > tol) ? 0.0 : 1.0 / h1;
    }
    __syncthreads();
    hn = red[8];
    sc = red[9];
  }
  if (tip == 0) {
    hnorm[j] = hn;
    is_null[j] = !(hn > tol) ? 1 : 0;
  }
  double* o = out + static_cast<int64_t>(j) * D2;
#pragma unroll
  for (int q = 0; q < (D2 + NT - 1) / NT; ++q) o[tip + q * NT] = hv[q] * sc;
}

template <int MINB, int VARIANT>
void run_tree(const char* name, const double* basis, int64_t g0, double* out, double* hn, int* nul,
              const std::vector<double>& ro, const std::vector<double>& rh) {
  using S = CommAhShape<DIM, 2, 4>;
  auto k = commutator_ah_tree_kernel<MINB, VARIANT>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM + 64));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, k));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int it = 0; it < 12; ++it) {
    cudaEventRecord(e0);
    k<<<CNT, 256, S::SMEM + 64>>>(basis, g0, CNT, 1e-10, out, hn, nul);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it >= 2 && ms < best) best = ms;
  }
  CK(cudaGetLastError());
  std::vector<double> o(static_cast<size_t>(CNT) * D2), h(CNT);
  CK(cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h.data(), hn, CNT * 8, cudaMemcpyDeviceToHost));
  double dmax = 0.0, hmax = 0.0;
  for (size_t e = 0; e < o.size(); ++e) dmax = std::max(dmax, std::abs(o[e] - ro[e]));
  for (int e = 0; e < CNT; ++e) hmax = std::max(hmax, std::abs(h[e] - rh[e]) / rh[e]);
  printf("{\"variant\": \"%s\", \"regs\": %d, \"local_bytes\": %zu, \"ms\": %.4f, \"tflops\": %.2f, "
         "\"max_abs_dh\": %.3g, \"max_rel_dnorm\": %.3g}\n",
         name, fa.numRegs, fa.localSizeBytes, best, 8.0 * DIM * DIM * DIM * CNT / (best * 1e-3) / 1e12, dmax, hmax);
}

template <int MINB> void run_clock(const double* basis, int64_t g0, double* out, double* hn, int* nul) {
  using S = CommAhShape<DIM, 2, 4>;
  auto k = commutator_ah_clock_kernel<MINB>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM));
  long long* clk;
  CK(cudaMalloc(&clk, static_cast<size_t>(CNT) * 7 * sizeof(long long)));
  for (int it = 0; it < 3; ++it) k<<<CNT, 256, S::SMEM>>>(basis, g0, CNT, 1e-10, out, hn, nul, clk);
  CK(cudaDeviceSynchronize());
  std::vector<long long> h(static_cast<size_t>(CNT) * 7);
  CK(cudaMemcpy(h.data(), clk, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
  double ph[6] = {0, 0, 0, 0, 0, 0};
  for (int b = 2000; b < 6000; ++b)
    for (int q = 0; q < 6; ++q) ph[q] += static_cast<double>(h[b * 7 + q + 1] - h[b * 7 + q]) / 4000.0;
  printf("{\"variant\": \"clock_minb%d\", \"cycles\": {\"load\": %.0f, \"product\": %.0f, \"barrier\": %.0f, "
         "\"store_p\": %.0f, \"h_values\": %.0f, \"finish\": %.0f, \"total\": %.0f}}\n",
         MINB, ph[0], ph[1], ph[2], ph[3], ph[4], ph[5], ph[0] + ph[1] + ph[2] + ph[3] + ph[4] + ph[5]);
  cudaFree(clk);
}

template <int MINB, int WR, int WC, bool ASYNC = true>
double run(const char* name, const double* basis, int64_t g0, double* out, double* hn, int* nul,
           std::vector<double>& h_out, std::vector<double>& h_hn) {
  using S = CommAhShape<DIM, WR, WC>;
  auto k = commutator_ah_kernel<DIM, MINB, WR, WC, ASYNC>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM));
  CK(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, k));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, S::THREADS, S::SMEM));
  const int blocks = (CNT + S::PAIRS_PER_CTA - 1) / S::PAIRS_PER_CTA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int it = 0; it < 12; ++it) {
    cudaEventRecord(e0);
    k<<<blocks, S::THREADS, S::SMEM>>>(basis, g0, CNT, 1e-10, true, out, hn, nul);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it >= 2 && ms < best) best = ms;
  }
  CK(cudaGetLastError());
  h_out.resize(static_cast<size_t>(CNT) * D2);
  h_hn.resize(CNT);
  CK(cudaMemcpy(h_out.data(), out, h_out.size() * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h_hn.data(), hn, CNT * 8, cudaMemcpyDeviceToHost));
  const double tf = 8.0 * DIM * DIM * DIM * CNT / (best * 1e-3) / 1e12;
  printf("{\"variant\": \"%s\", \"minb\": %d, \"wr\": %d, \"wc\": %d, \"regs\": %d, \"local_bytes\": %zu, "
         "\"ctas_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.2f}\n",
         name, MINB, WR, WC, fa.numRegs, fa.localSizeBytes, occ, best, tf);
  return best;
}

// the ping-pong kernel: one persistent 512-thread CTA per SM (two 8-warp groups)
double run_pp(const char* name, const double* basis, int64_t g0, double* out, double* hn, int* nul,
              std::vector<double>& h_out, std::vector<double>& h_hn) {
  using S = CommAhShape<DIM>;
  auto k = commutator_ah_pp_kernel<DIM>;
  const int smem = 2 * S::SMEM_PER_PAIR;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, k));
  int occ = 0, sms = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 512, smem));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int blocks = std::min(sms * occ, (CNT + 1) / 2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int it = 0; it < 12; ++it) {
    cudaEventRecord(e0);
    k<<<blocks, 512, smem>>>(basis, g0, CNT, 1e-10, true, out, hn, nul);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it >= 2 && ms < best) best = ms;
  }
  CK(cudaGetLastError());
  h_out.resize(static_cast<size_t>(CNT) * D2);
  h_hn.resize(CNT);
  CK(cudaMemcpy(h_out.data(), out, h_out.size() * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h_hn.data(), hn, CNT * 8, cudaMemcpyDeviceToHost));
  const double tf = 8.0 * DIM * DIM * DIM * CNT / (best * 1e-3) / 1e12;
  printf("{\"variant\": \"%s\", \"regs\": %d, \"local_bytes\": %zu, \"ctas_per_sm\": %d, \"blocks\": %d, "
         "\"ms\": %.4f, \"tflops\": %.2f}\n",
         name, fa.numRegs, fa.localSizeBytes, occ, blocks, best, tf);
  return best;
}

int main() {
  std::vector<double> hb(static_cast<size_t>(NB) * D2);
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  for (auto& v : hb) v = nd(rng) / 64.0;
  double *basis, *out, *hn;
  int* nul;
  CK(cudaMalloc(&basis, hb.size() * 8));
  CK(cudaMalloc(&out, static_cast<size_t>(CNT) * D2 * 8));
  CK(cudaMalloc(&hn, CNT * 8));
  CK(cudaMalloc(&nul, CNT * 4));
  CK(cudaMemcpy(basis, hb.data(), hb.size() * 8, cudaMemcpyHostToDevice));
  const int64_t g0 = pair_index(1024, 0);
  std::vector<double> ro, rh, o, h;
  run<2, 2, 4, false>("2x4_minb2_sync", basis, g0, out, hn, nul, ro, rh);
  auto same = [&](const char* n) {
    const bool eq = !std::memcmp(o.data(), ro.data(), o.size() * 8) && !std::memcmp(h.data(), rh.data(), h.size() * 8);
    printf("  %s bit-identical: %s\n", n, eq ? "yes" : "NO");
  };
  run<2, 2, 4>("2x4_minb2", basis, g0, out, hn, nul, o, h); same("2x4_minb2");
  run_pp("pingpong_2x8warps", basis, g0, out, hn, nul, o, h); same("pingpong_2x8warps");
  run<2, 2, 4>("2x4_minb2_again", basis, g0, out, hn, nul, o, h); same("2x4_minb2_again");
  run_pp("pingpong_again", basis, g0, out, hn, nul, o, h); same("pingpong_again");
  run_tree<2, 0>("tree_all_threads", basis, g0, out, hn, nul, ro, rh);
  run_tree<2, 1>("tree_one_thread", basis, g0, out, hn, nul, ro, rh);
  run_tree<2, 2>("tree_rsqrt", basis, g0, out, hn, nul, ro, rh);
  run_tree<2, 3>("lean_rsqrt", basis, g0, out, hn, nul, ro, rh);
  run_clock<1>(basis, g0, out, hn, nul);
  run_clock<2>(basis, g0, out, hn, nul);
  return 0;
}
