// Probe: raster group of the TMA projection GEMMs (M-tiles per group sweeping
// all candidate tiles) against time; run under
//   ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:dgemm_tma
// for the DRAM bytes per launch. K2a (A = Vw, K-contiguous) and K2b (A = VT,
// K-contiguous) on the headline shapes.
#include <cudaTypedefs.h>
#include <cstdio>
#include <random>
#include <vector>
#include "../../paper_2506_01120_b200/csrc/dgemm_tma.cuh"
using namespace liecl_b200;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)
static CUtensorMap map_kc(const double* p, int64_t len, int64_t rows, int64_t ld, int box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&fn), cudaEnableDefault, &q));
  }
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(len), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 8)};
  cuuint32_t box[2] = {16, static_cast<cuuint32_t>(box_rows)}, es[2] = {1, 1};
  if (fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(p), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode\n");
    exit(1);
  }
  return m;
}
template <int G> void run(const CUtensorMap& va, const CUtensorMap& xb, const CUtensorMap& vt, const CUtensorMap& pb,
                          int NB, int D, int NC, double* beta, double* R, const double* X, double* part, int d) {
  auto ka = dgemm_tma_kernel<true, REpi::kStoreScaled, 5, G>;
  auto kb = dgemm_tma_kernel<true, REpi::kSubtractNorm, 5, G>;
  CK(cudaFuncSetAttribute(ka, cudaFuncAttributeMaxDynamicSharedMemorySize, tg::SMEM));
  CK(cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, tg::SMEM));
  dim3 ga((NB + 127) / 128, (NC + 63) / 64), gb((D + 127) / 128, (NC + 63) / 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ta = 1e30f, tb = 1e30f;
  for (int it = 0; it < 5; ++it) {
    float ms;
    cudaEventRecord(e0);
    ka<<<ga, tg::THREADS, tg::SMEM>>>(va, xb, NB, NC, D, beta, 4096, 1.0 / d, nullptr, 0, nullptr, d);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    if (it) ta = std::min(ta, ms);
    cudaEventRecord(e0);
    kb<<<gb, tg::THREADS, tg::SMEM>>>(vt, pb, D, NC, NB, R, D, 1.0, X, D, part, d);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    if (it) tb = std::min(tb, ms);
  }
  printf("{\"group\": %d, \"k2a_ms\": %.4f, \"k2b_ms\": %.4f}\n", G, ta, tb);
}
int main() {
  const int d = 64, D = d * d, NB = 4095, NC = 8192, LDB = 4096;
  std::mt19937_64 rng(3);
  std::normal_distribution<double> nd;
  std::vector<double> hv(static_cast<size_t>(NB + 1) * D, 0.0), hx(static_cast<size_t>(NC) * D), ht(static_cast<size_t>(D) * 4096, 0.0);
  for (size_t i = 0; i < static_cast<size_t>(NB) * D; ++i) hv[i] = nd(rng) / 64;
  for (auto& v : hx) v = nd(rng) / 64;
  for (int k = 0; k < NB; ++k)
    for (int m = 0; m < D; ++m) ht[static_cast<size_t>(m) * 4096 + k] = hv[static_cast<size_t>(k) * D + m];
  double *V, *VT, *X, *beta, *R, *part;
  CK(cudaMalloc(&V, hv.size() * 8));
  CK(cudaMalloc(&VT, ht.size() * 8));
  CK(cudaMalloc(&X, hx.size() * 8));
  CK(cudaMalloc(&beta, static_cast<size_t>(NC) * LDB * 8));
  CK(cudaMalloc(&R, hx.size() * 8));
  CK(cudaMalloc(&part, 64 * NC * 8));
  CK(cudaMemcpy(V, hv.data(), hv.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(VT, ht.data(), ht.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(X, hx.data(), hx.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemset(beta, 0, static_cast<size_t>(NC) * LDB * 8));
  CUtensorMap va = map_kc(V, D, NB, D, 128), xb = map_kc(X, D, NC, D, 64), vt = map_kc(VT, NB, D, 4096, 128),
              pb = map_kc(beta, NB, NC, LDB, 64);
  run<4>(va, xb, vt, pb, NB, D, NC, beta, R, X, part, d);
  run<8>(va, xb, vt, pb, NB, D, NC, beta, R, X, part, d);
  run<12>(va, xb, vt, pb, NB, D, NC, beta, R, X, part, d);
  run<16>(va, xb, vt, pb, NB, D, NC, beta, R, X, part, d);
  run<24>(va, xb, vt, pb, NB, D, NC, beta, R, X, part, d);
  run<32>(va, xb, vt, pb, NB, D, NC, beta, R, X, part, d);
  return 0;
}
