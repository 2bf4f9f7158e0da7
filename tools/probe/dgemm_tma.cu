// Probe: TMA-staged projection GEMMs (dgemm_tma.cuh) against the cp.async
// kernels (dgemm_dmma.cuh) on the saturated-window shapes: K2a beta = Vw^T X / d
// (M = 4095 basis, N = 8192 candidates, K = 4096) and K2b R = X - V beta
// (M = 4096, N = 8192, K = 4095). Prints ms, TFLOP/s and max |diff| / max |ref|.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o dgemm_tma dgemm_tma.cu
#include <cudaTypedefs.h>

#include <cstdio>
#include <random>
#include <vector>

#include "../../paper_2506_01120_b200/csrc/dgemm_tma.cuh"

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
// rows of `len` doubles (K-contiguous), row stride ld doubles: box {16, box_rows}
static CUtensorMap map_kc(const double* p, int64_t len, int64_t rows, int64_t ld, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(len), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 8)};
  cuuint32_t box[2] = {16, static_cast<cuuint32_t>(box_rows)}, es[2] = {1, 1};
  CUresult r = encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(p), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode kc failed %d\n", r); exit(1); }
  return m;
}
// A(m, k) = p[k*ld + m], M a multiple of 16, k = 4t + 2p + q: 5-D {16, 2, ceil(K/4), 2, M/16}
static CUtensorMap map_mc(const double* p, int64_t M, int64_t K, int64_t ld) {
  CUtensorMap m;
  const int64_t kq = (K + 3) / 4;
  cuuint64_t dims[5] = {16, 2, static_cast<cuuint64_t>(kq), 2, static_cast<cuuint64_t>(M / 16)};
  cuuint64_t strides[4] = {static_cast<cuuint64_t>(ld * 8), static_cast<cuuint64_t>(ld * 32),
                           static_cast<cuuint64_t>(ld * 16), 128};
  cuuint32_t box[5] = {16, 2, 4, 2, 8}, es[5] = {1, 1, 1, 1, 1};
  CUresult r = encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double*>(p), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode mc failed %d\n", r); exit(1); }
  return m;
}

static CUtensorMap map_mc3(const double* p, int64_t M, int64_t K, int64_t ld) {
  CUtensorMap m;
  cuuint64_t dims[3] = {16, static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(M / 16)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld * 8), 128};
  cuuint32_t box[3] = {16, 16, 8}, es[3] = {1, 1, 1};
  CUresult r = encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(p), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode mc3 failed %d\n", r); exit(1); }
  return m;
}

template <class F> float best_ms(F f, int reps = 8) {
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

static double maxdiff(const double* a, const double* b, size_t n) {
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
  const int d = 64, D = d * d, NB = 4095, NC = 8192, LDB = 4096;
  std::mt19937_64 rng(3);
  std::normal_distribution<double> nd;
  std::vector<double> hv(static_cast<size_t>(NB + 1) * D, 0.0), hx(static_cast<size_t>(NC) * D);
  for (size_t i = 0; i < static_cast<size_t>(NB) * D; ++i) hv[i] = nd(rng) / 64;
  for (auto& v : hx) v = nd(rng) / 64;
  double *V, *X, *beta1, *beta2, *R1, *R2, *p1, *p2;
  CK(cudaMalloc(&V, hv.size() * 8));
  CK(cudaMalloc(&X, hx.size() * 8));
  CK(cudaMalloc(&beta1, static_cast<size_t>(NC) * LDB * 8));
  CK(cudaMalloc(&beta2, static_cast<size_t>(NC) * LDB * 8));
  CK(cudaMalloc(&R1, hx.size() * 8));
  CK(cudaMalloc(&R2, hx.size() * 8));
  CK(cudaMalloc(&p1, 64 * NC * 8));
  CK(cudaMalloc(&p2, 64 * NC * 8));
  CK(cudaMemcpy(V, hv.data(), hv.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(X, hx.data(), hx.size() * 8, cudaMemcpyHostToDevice));
  const double flops = 2.0 * NB * D * NC;

  // K2a: beta = (1/d) V^T X  (A K-contiguous: rows of V)
  {
    const int sm = rg::smem_bytes<true>();
    auto k = dgemm_dmma_kernel<true, REpi::kStoreScaled>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    dim3 grid((NB + rg::BM - 1) / rg::BM, (NC + rg::BN - 1) / rg::BN);
    float ms = best_ms([&] { k<<<grid, rg::THREADS, sm>>>(NB, NC, D, V, D, X, D, beta1, LDB, 1.0 / d, nullptr, 0, nullptr, d, 0, 0); });
    printf("{\"gemm\": \"K2a\", \"kernel\": \"cp.async\", \"ms\": %.4f, \"tflops\": %.2f}\n", ms, flops / ms / 1e9);
    auto kt = dgemm_tma_kernel<true, REpi::kStoreScaled>;
    CK(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, tg::SMEM));
    CUtensorMap ma = map_kc(V, D, NB, D, tg::BM), mb = map_kc(X, D, NC, D, tg::BN);
    float ms2 = best_ms([&] { kt<<<grid, tg::THREADS, tg::SMEM>>>(ma, mb, NB, NC, D, beta2, LDB, 1.0 / d, nullptr, 0, nullptr, d); });
    printf("{\"gemm\": \"K2a\", \"kernel\": \"tma\", \"ms\": %.4f, \"tflops\": %.2f, \"rel_diff\": %.3e}\n", ms2,
           flops / ms2 / 1e9, maxdiff(beta2, beta1, static_cast<size_t>(NC) * LDB));
  }
  // K2b: R = X - V beta (A M-contiguous: A(m, k) = V[k*D + m]; B(k, n) = beta[n*LDB + k])
  {
    const int sm = rg::smem_bytes<false>();
    auto k = dgemm_dmma_kernel<false, REpi::kSubtractNorm>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    dim3 grid((D + rg::BM - 1) / rg::BM, (NC + rg::BN - 1) / rg::BN);
    float ms = best_ms([&] { k<<<grid, rg::THREADS, sm>>>(D, NC, NB, V, D, beta1, LDB, R1, D, 1.0, X, D, p1, d, 0, 0); });
    printf("{\"gemm\": \"K2b\", \"kernel\": \"cp.async\", \"ms\": %.4f, \"tflops\": %.2f}\n", ms, flops / ms / 1e9);
    auto kt = dgemm_tma_kernel<false, REpi::kSubtractNorm>;
    CK(cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, tg::SMEM));
    CUtensorMap ma = map_mc(V, D, NB, D), mb = map_kc(beta1, NB, NC, LDB, tg::BN);
    auto kt3 = dgemm_tma_kernel<false, REpi::kSubtractNorm, 3>;
    CK(cudaFuncSetAttribute(kt3, cudaFuncAttributeMaxDynamicSharedMemorySize, tg::SMEM));
    CUtensorMap ma3 = map_mc3(V, D, NB, D);
    for (int rep = 0; rep < 2; ++rep) {
      float ms2 = best_ms([&] { kt<<<grid, tg::THREADS, tg::SMEM>>>(ma, mb, D, NC, NB, R2, D, 1.0, X, D, p2, d); });
      printf("{\"gemm\": \"K2b\", \"kernel\": \"tma_5d\", \"ms\": %.4f, \"tflops\": %.2f, \"rel_diff\": %.3e, \"partial_rel_diff\": %.3e}\n",
             ms2, flops / ms2 / 1e9, maxdiff(R2, R1, hx.size()), maxdiff(p2, p1, static_cast<size_t>(32) * NC));
      float ms3 = best_ms([&] { kt3<<<grid, tg::THREADS, tg::SMEM>>>(ma3, mb, D, NC, NB, R2, D, 1.0, X, D, p2, d); });
      printf("{\"gemm\": \"K2b\", \"kernel\": \"tma_3d\", \"ms\": %.4f, \"tflops\": %.2f, \"rel_diff\": %.3e}\n", ms3,
             flops / ms3 / 1e9, maxdiff(R2, R1, hx.size()));
    }
  }
  return 0;
}
