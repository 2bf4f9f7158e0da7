// Probe: TMA-staged complex projection GEMMs (zgemm_tma.cuh) against the
// cp.async kernels (zgemm_dmma.cuh): K2a beta = V^H X / d (M = n = 4096,
// N = 4096 candidates, K = D = 16384) and K2b R = X - V beta (M = D, K = n).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o zgemm_tma zgemm_tma.cu
#include <cudaTypedefs.h>

#include <cstdio>
#include <random>
#include <vector>

#include "../../paper_2506_01120_b200/csrc/zgemm_tma.cuh"

using namespace liecl_b200;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

static PFN_cuTensorMapEncodeTiled_v12000 encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&fn), cudaEnableDefault, &q));
  }
  return fn;
}
static CUtensorMap zmap_kc(const double2* p, int64_t len, int64_t rows, int64_t ld) {
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(2 * len), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 16)};
  cuuint32_t box[2] = {16, 64}, es[2] = {1, 1};
  if (encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double2*>(p), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encode kc\n"); exit(1); }
  return m;
}
static CUtensorMap zmap_mc(const double2* p, int64_t M, int64_t K, int64_t ld) {
  CUtensorMap m;
  cuuint64_t dims[3] = {16, static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(M / 8)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld * 16), 128};
  cuuint32_t box[3] = {16, 8, 8}, es[3] = {1, 1, 1};
  if (encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double2*>(p), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encode mc\n"); exit(1); }
  return m;
}
template <class F> float best_ms(F f, int reps = 6) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int i = 0; i < reps + 2; ++i) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (i >= 2 && ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}
static double maxdiff(const void* a, const void* b, size_t n) {
  std::vector<double> ha(n), hb(n);
  CK(cudaMemcpy(ha.data(), a, n * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hb.data(), b, n * 8, cudaMemcpyDeviceToHost));
  double md = 0, mr = 0;
  for (size_t i = 0; i < n; ++i) {
    md = std::max(md, std::abs(ha[i] - hb[i]));
    mr = std::max(mr, std::abs(hb[i]));
  }
  return md / std::max(mr, 1e-300);
}

int main() {
  const int64_t NBASIS = 4095, D = 16384, NC = 4096;
  std::mt19937_64 rng(5);
  std::normal_distribution<double> nd;
  std::vector<double2> hv(NBASIS * D), hx(NC * D);
  for (auto& v : hv) v = make_double2(nd(rng) / 128, nd(rng) / 128);
  for (auto& v : hx) v = make_double2(nd(rng) / 128, nd(rng) / 128);
  double2 *V, *X, *b1, *b2, *R1, *R2;
  double *p1, *p2;
  CK(cudaMalloc(&V, hv.size() * 16));
  CK(cudaMalloc(&X, hx.size() * 16));
  CK(cudaMalloc(&b1, NBASIS * NC * 16));
  CK(cudaMalloc(&b2, NBASIS * NC * 16));
  CK(cudaMalloc(&R1, hx.size() * 16));
  CK(cudaMalloc(&R2, hx.size() * 16));
  CK(cudaMalloc(&p1, 512 * NC * 8));
  CK(cudaMalloc(&p2, 512 * NC * 8));
  CK(cudaMemcpy(V, hv.data(), hv.size() * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(X, hx.data(), hx.size() * 16, cudaMemcpyHostToDevice));
  const double flops = 8.0 * NBASIS * D * NC;
  {
    auto k = zgemm_dmma_kernel<true, true, Epilogue::kStoreScaled>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, zg::smem_bytes<true>()));
    dim3 grid((NBASIS + 63) / 64, (NC + 63) / 64);
    float ms = best_ms([&] { k<<<grid, zg::THREADS, zg::smem_bytes<true>()>>>(NBASIS, NC, D, V, D, X, D, b1, NBASIS, 1.0 / 128, nullptr, 0, nullptr, 0, 0); });
    printf("{\"gemm\": \"K2a\", \"kernel\": \"cp.async\", \"ms\": %.3f, \"tflops\": %.2f}\n", ms, flops / ms / 1e9);
    auto kt = zgemm_tma_kernel<true, true, Epilogue::kStoreScaled>;
    CK(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, ztg::SMEM));
    CUtensorMap ma = zmap_kc(V, D, NBASIS, D), mb = zmap_kc(X, D, NC, D);
    float ms2 = best_ms([&] { kt<<<grid, ztg::THREADS, ztg::SMEM>>>(ma, mb, NBASIS, NC, D, b2, NBASIS, 1.0 / 128, nullptr, 0, nullptr); });
    printf("{\"gemm\": \"K2a\", \"kernel\": \"tma\", \"ms\": %.3f, \"tflops\": %.2f, \"rel_diff\": %.3e}\n", ms2, flops / ms2 / 1e9,
           maxdiff(b2, b1, NBASIS * NC * 2));
  }
  {
    auto k = zgemm_dmma_kernel<false, false, Epilogue::kSubtractNorm>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, zg::smem_bytes<false>()));
    dim3 grid((D + 63) / 64, (NC + 63) / 64);
    float ms = best_ms([&] { k<<<grid, zg::THREADS, zg::smem_bytes<false>()>>>(D, NC, NBASIS, V, D, b1, NBASIS, R1, D, 1.0, X, D, p1, 0, 0); });
    printf("{\"gemm\": \"K2b\", \"kernel\": \"cp.async\", \"ms\": %.3f, \"tflops\": %.2f}\n", ms, flops / ms / 1e9);
    auto kt = zgemm_tma_kernel<false, false, Epilogue::kSubtractNorm>;
    CK(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, ztg::SMEM));
    CUtensorMap ma = zmap_mc(V, D, NBASIS, D), mb = zmap_kc(b1, NBASIS, NC, NBASIS);
    float ms2 = best_ms([&] { kt<<<grid, ztg::THREADS, ztg::SMEM>>>(ma, mb, D, NC, NBASIS, R2, D, 1.0, X, D, p2); });
    printf("{\"gemm\": \"K2b\", \"kernel\": \"tma\", \"ms\": %.3f, \"tflops\": %.2f, \"rel_diff\": %.3e, \"partial_rel_diff\": %.3e}\n",
           ms2, flops / ms2 / 1e9, maxdiff(R2, R1, hx.size() * 2), maxdiff(p2, p1, 256 * NC));
  }
  return 0;
}
