// Probe: sort.cuh (the PauliSum engine's stable pair sorts) against
// std::stable_sort on the masked keys: one-CTA sizes, radix sizes across tile
// and scan-level edges, few distinct keys (long equal runs test stability),
// every end_bit class, and timing at 1M / 8M pairs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o sort_test sort_test.cu
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#include "../../paper_2506_01120_b200/csrc/sort.cuh"

using namespace liecl_b200;
using u64 = unsigned long long;

static bool check(int64_t n, int end_bit, int distinct_bits, std::mt19937_64& rng, bool time_it = false) {
  std::vector<u64> h(n), gk(n);
  std::vector<unsigned> v(n), gv(n);
  for (auto& k : h) {
    k = rng();
    if (distinct_bits < 64) k &= (1ull << distinct_bits) - 1;
    if (rng() % 97 == 0) k = ~0ull;  // the engine's marker
  }
  for (int64_t i = 0; i < n; ++i) v[i] = static_cast<unsigned>(rng());
  const u64 mask = end_bit >= 64 ? ~0ull : (1ull << end_bit) - 1;
  std::vector<int64_t> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return (h[a] & mask) < (h[b] & mask); });
  u64 *kin, *kout;
  unsigned *vin, *vout;
  void* ws;
  cudaMalloc(&kin, n * 8);
  cudaMalloc(&kout, n * 8);
  cudaMalloc(&vin, n * 4);
  cudaMalloc(&vout, n * 4);
  cudaMalloc(&ws, sort::workspace_bytes(n));
  cudaMemcpy(kin, h.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(vin, v.data(), n * 4, cudaMemcpyHostToDevice);
  int k = 0;
  sort::pairs(kin, kout, vin, vout, n, end_bit, ws, 0, k);
  float ms = 0;
  if (time_it) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) sort::pairs(kin, kout, vin, vout, n, end_bit, ws, 0, k);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
  }
  cudaMemcpy(gk.data(), kout, n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(gv.data(), vout, n * 4, cudaMemcpyDeviceToHost);
  std::vector<u64> back(n);
  cudaMemcpy(back.data(), kin, n * 8, cudaMemcpyDeviceToHost);
  bool ok = cudaGetLastError() == cudaSuccess && back == h;  // input untouched
  for (int64_t i = 0; ok && i < n; ++i) ok = gk[i] == h[ord[i]] && gv[i] == v[ord[i]];
  printf("n=%lld end_bit=%d distinct_bits=%d %s", static_cast<long long>(n), end_bit, distinct_bits, ok ? "ok" : "FAIL");
  if (time_it) printf("  %.3f ms (%.2f Gpairs/s)", ms, n / ms / 1e6);
  printf("\n");
  cudaFree(kin), cudaFree(kout), cudaFree(vin), cudaFree(vout), cudaFree(ws);
  return ok;
}

int main() {
  std::mt19937_64 rng(5);
  bool ok = true;
  if (std::getenv("SORT_ONLY_LARGE")) {  // for an ncu capture of the 8M-pair passes
    ok &= check(1 << 23, 40, 64, rng, true);
    printf(ok ? "all ok\n" : "FAILED\n");
    return ok ? 0 : 1;
  }
  for (int64_t n : {1, 2, 3, 31, 1000, 2047, 2048, 2049, 4096, 4097, 8191, 65537, 1048576, 1048577, 3000001})
    for (int eb : {1, 7, 8, 9, 20, 41, 63, 64}) {
      ok &= check(n, eb, 64, rng);
      ok &= check(n, eb, 3, rng);
    }
  ok &= check(5000, 0, 64, rng);
  ok &= check(1 << 20, 40, 64, rng, true);
  ok &= check(1 << 23, 40, 64, rng, true);
  ok &= check(1 << 23, 64, 64, rng, true);
  ok &= check(1 << 14, 40, 64, rng, true);
  ok &= check(2048, 40, 64, rng, true);
  printf(ok ? "all ok\n" : "FAILED\n");
  return ok ? 0 : 1;
}
