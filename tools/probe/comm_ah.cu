// Probe: warp layouts / register bounds of commutator_ah_kernel<64> on a
// random packed anti-Hermitian basis (4095 x 4096), 8192 cursor pairs from
// row 1024 (a saturated-window batch). Prints ms and TFLOP/s (8 d^3 per pair)
// per variant; every variant must give bit-identical h and norms.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o comm_ah comm_ah.cu
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "../../paper_2506_01120_b200/csrc/ah.cuh"

using namespace liecl_b200;

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
  run<3, 1, 8, false>("row_strip_minb3_sync", basis, g0, out, hn, nul, ro, rh);
  auto same = [&](const char* n) {
    const bool eq = !std::memcmp(o.data(), ro.data(), o.size() * 8) && !std::memcmp(h.data(), rh.data(), h.size() * 8);
    printf("  %s bit-identical: %s\n", n, eq ? "yes" : "NO");
  };
  run<3, 1, 8>("row_strip_minb3", basis, g0, out, hn, nul, o, h); same("row_strip_minb3");
  run<2, 1, 8>("row_strip_minb2", basis, g0, out, hn, nul, o, h); same("row_strip_minb2");
  run<2, 2, 4, false>("2x4_minb2_sync", basis, g0, out, hn, nul, o, h); same("2x4_minb2_sync");
  run<2, 2, 4>("2x4_minb2", basis, g0, out, hn, nul, o, h); same("2x4_minb2");
  run<3, 2, 4>("2x4_minb3", basis, g0, out, hn, nul, o, h); same("2x4_minb3");
  run<2, 4, 2>("4x2_minb2", basis, g0, out, hn, nul, o, h); same("4x2_minb2");
  run<1, 2, 4>("2x4_minb1", basis, g0, out, hn, nul, o, h); same("2x4_minb1");
  run<2, 8, 1>("8x1_minb2", basis, g0, out, hn, nul, o, h); same("8x1_minb2");
  run<2, 1, 4>("1x4_16warps_minb2", basis, g0, out, hn, nul, o, h); same("1x4_16warps_minb2");
  run<2, 2, 2>("2x2_16warps_minb2", basis, g0, out, hn, nul, o, h); same("2x2_16warps_minb2");
  run<3, 2, 2>("2x2_16warps_minb3", basis, g0, out, hn, nul, o, h); same("2x2_16warps_minb3");
  return 0;
}
