// standalone check of the block_chol.cuh kernels (Cholesky) on small SPD matrices; chol_dbg
// (DBG=1) keeps the 2-D array-pointer form that nvcc 12.9 miscompiled for sm_100a: its SASS
// reads the loop's shared-memory row address before the first write on loop entry, so
// Rs[0][0] lands elsewhere (printed R00 = 0 / stale)
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../../paper_2506_01120_b200/csrc/block_chol.cuh"
using namespace liecl_b200;
__global__ void chol_dbg(const double* G, int ldg, int a, double* R, double* diag) {
  extern __shared__ __align__(16) unsigned char sm2[];
  double(*Rs)[kBcMax] = reinterpret_cast<double(*)[kBcMax]>(sm2);
  const int t = threadIdx.x;
  for (int i = 0; i < a; ++i) {
    if (t == 0) {
      double s = G[i + i * ldg];
      for (int k = 0; k < i; ++k) s -= Rs[k][i] * Rs[k][i];
      Rs[i][i] = sqrt(fmax(s, 0.0));
      diag[i] = Rs[i][i];
    }
    __syncthreads();
    if (t > i && t < a) {
      double z = G[i + t * ldg];
      for (int k = 0; k < i; ++k) z -= Rs[k][i] * Rs[k][t];
      Rs[i][t] = z / Rs[i][i];
    }
    __syncthreads();
  }
  if (t == 0) printf("dbg a=%d Rs00=%f\n", a, Rs[0][0]);
  for (int e = t; e < a * a; e += blockDim.x) {
    const int i = e % a, j = e / a;
    R[i + j * kBcMax] = i <= j ? Rs[i][j] : 0.0;
  }
}
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
int main() {
  for (int a : {1, 2, 3, 5, 17, 64}) {
    std::vector<double> B(a * a), G(64 * 64, 0.0);
    srand(a);
    for (auto& v : B) v = rand() / double(RAND_MAX) - 0.5;
    for (int i = 0; i < a; ++i) for (int j = 0; j < a; ++j) {
      double s = (i == j) ? 1.0 : 0.0;
      for (int k = 0; k < a; ++k) s += B[k + i * a] * B[k + j * a];
      G[i + j * a] = s;
    }
    double *dG, *dR, *dd;
    CK(cudaMalloc(&dG, 64 * 64 * 8)); CK(cudaMalloc(&dR, 64 * 64 * 8)); CK(cudaMalloc(&dd, 64 * 8));
    CK(cudaMemcpy(dG, G.data(), 64 * 64 * 8, cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(bc_cholesky_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, bc_smem_bytes<double>()));
    if (getenv("DBG")) chol_dbg<<<1, kBcMax, 32768>>>(dG, a, a, dR, dd);
    else bc_cholesky_kernel<double><<<1, kBcThreads, bc_smem_bytes<double>()>>>(dG, a, a, dR, dd);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<double> R(64 * 64);
    CK(cudaMemcpy(R.data(), dR, 64 * 64 * 8, cudaMemcpyDeviceToHost));
    double err = 0;
    for (int i = 0; i < a; ++i) for (int j = 0; j < a; ++j) {
      double s = 0; for (int k = 0; k < a; ++k) s += R[k + i * 64] * R[k + j * 64];
      err = fmax(err, fabs(s - G[i + j * a]));
    }
    std::vector<double> dg(64);
    CK(cudaMemcpy(dg.data(), dd, 64 * 8, cudaMemcpyDeviceToHost));
    printf("a=%d chol err %.3g  G00 %.6f R00 %.6f diag0 %.6f R01 %.6f\n", a, err, G[0], R[0], dg[0], R[64]);
  }
  return 0;
}
