// Probe: scan.cuh (the PauliSum engine's exclusive scans) against a host scan,
// int and long long, n across one, two and three levels (1 .. 3M).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scan_test scan_test.cu
#include <cstdio>
#include <random>
#include <vector>

#include "../../paper_2506_01120_b200/csrc/scan.cuh"

using namespace liecl_b200;

template <class T> bool check(int64_t n, std::mt19937_64& rng) {
  std::vector<T> h(n), ref(n), got(n);
  for (auto& v : h) v = static_cast<T>(rng() % (sizeof(T) == 4 ? 3 : 1000000));
  T run = 0;
  for (int64_t i = 0; i < n; ++i) { ref[i] = run; run += h[i]; }
  T *in, *out, *ws;
  cudaMalloc(&in, n * sizeof(T));
  cudaMalloc(&out, n * sizeof(T));
  cudaMalloc(&ws, scan::workspace(n) * sizeof(T));
  cudaMemcpy(in, h.data(), n * sizeof(T), cudaMemcpyHostToDevice);
  int k = 0;
  T* total = scan::exclusive<T>(in, out, n, ws, 0, k);
  T tot = 0;
  cudaMemcpy(got.data(), out, n * sizeof(T), cudaMemcpyDeviceToHost);
  cudaMemcpy(&tot, total, sizeof(T), cudaMemcpyDeviceToHost);
  const bool ok = got == ref && tot == run && cudaGetLastError() == cudaSuccess;
  printf("%s n=%lld launches=%d %s\n", sizeof(T) == 4 ? "int" : "i64", static_cast<long long>(n), k, ok ? "ok" : "FAIL");
  cudaFree(in);
  cudaFree(out);
  cudaFree(ws);
  return ok;
}

int main() {
  std::mt19937_64 rng(3);
  bool ok = true;
  for (int64_t n : {1, 31, 1024, 1025, 4097, 1048576, 1048577, 3000001}) {
    ok &= check<int>(n, rng);
    ok &= check<long long>(n, rng);
  }
  printf(ok ? "all ok\n" : "FAILED\n");
  return ok ? 0 : 1;
}
