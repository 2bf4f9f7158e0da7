// Probe: warp layouts / register bounds of commutator_ah_kernel<64> on a
// random packed anti-Hermitian basis (4095 x 4096), 8192 cursor pairs from
// row 1024 (a saturated-window batch). Prints ms and TFLOP/s (8 d^3 per pair)
// per variant; every variant must give bit-identical h and norms.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o comm_ah comm_ah.cu
#include <cstdio>
#include <algorithm>
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
  return 0;
}
