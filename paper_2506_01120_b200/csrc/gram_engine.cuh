// GramEngine -- the matrix-inversion strategy (Alg. 2) on the B200: SURVEY §8
// row f1. Replaces MatrixInversionStrategy + GramState
// (R:src/closure.cpp:44-140, 214-265) inside the same batched cursor loop as
// DenseEngine. Included by engine.cu inside its anonymous namespace.
//
// Check (matrix_inversion_residual, R:src/closure.cpp:110-131), batched:
//   beta = (1/d) B^H C        K2a (B = the accepted unit candidates, not orthonormal)
//   x    = A^{-1} beta        complex DMMA GEMM against the maintained inverse
//   R    = C - B x, ||R||     K2b with the fused norm
// one pass (the reference does not re-orthogonalise); independent iff ||R|| > tol.
// Accept (R:src/closure.cpp:238-249): Schur complement s = Re(1 - beta^H u),
// u = A^{-1} beta (= x); degeneracy below the conditioning floor; bordered
// inverse update (GramState::expand, :55-87); full refresh from A (blocked
// Cholesky on the DMMA GEMMs, pivoted fallback; HermInverse) when s < 1e-4 or
// every `gram_refresh_interval` accepts (:89-95).
// The speculative rule of :440-444 is kept: a "dependent" verdict against the
// batch-start state stands; an "independent" one after an in-batch accept is
// recomputed against the current state.

__global__ void schur_kernel(const double2* __restrict__ beta, const double2* __restrict__ u, int64_t n,
                             double* __restrict__ s_out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t l = threadIdx.x; l < n; l += blockDim.x) acc += beta[l].x * u[l].x + beta[l].y * u[l].y;
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) t += red[w];
    *s_out = 1.0 - t;  // Re(1 - sum conj(beta) u)
  }
}

// Bordered inverse (GramState::expand): with u = A^{-1} beta and s the Schur
// complement, [A b; b* 1]^{-1} = [A^{-1} + u u^H/s, -u/s; -u^H/s, 1/s].
__global__ void bordered_update_kernel(double2* __restrict__ Ainv, double2* __restrict__ A, int64_t ld, int64_t n,
                                       const double2* __restrict__ u, const double2* __restrict__ beta, double s) {
  const int64_t total = (n + 1) * (n + 1);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e % (n + 1), k = e / (n + 1);
    const int64_t idx = i + k * ld;
    if (i < n && k < n) {
      const double2 ui = u[i], uk = u[k];
      const double2 p = make_double2(ui.x * uk.x + ui.y * uk.y, ui.y * uk.x - ui.x * uk.y);  // u_i conj(u_k)
      Ainv[idx] = make_double2(Ainv[idx].x + p.x / s, Ainv[idx].y + p.y / s);
    } else if (i < n) {  // column n
      Ainv[idx] = make_double2(-u[i].x / s, -u[i].y / s);
      A[idx] = beta[i];
    } else if (k < n) {  // row n = conj(column n)
      Ainv[idx] = make_double2(-u[k].x / s, u[k].y / s);
      A[idx] = make_double2(beta[k].x, -beta[k].y);
    } else {
      Ainv[idx] = make_double2(n == 0 ? 1.0 : 1.0 / s, 0.0);
      A[idx] = make_double2(1.0, 0.0);
    }
  }
}

__global__ void identity_kernel(double2* __restrict__ M, int64_t ld, int64_t n) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n * n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e % n, k = e / n;
    M[i + k * ld] = make_double2(i == k ? 1.0 : 0.0, 0.0);
  }
}

// ---- GramState::refresh's inverse (R:src/closure.cpp:89-95: A.ldlt().solve(I))
// Hand-written, Cholesky based (a Hermitian positive definite Gram matrix),
// i.e. zpotrf + zpotrs(I) in 64-wide blocks:
//  1. right-looking Cholesky A = L L^H: per panel one CTA factors the diagonal
//     block (gj_chol_block_kernel), L21 = A21 L11^-H by row-wise substitution
//     (gj_trsm_rows_kernel), the trailing A22 -= L21 L21^H is a complex DMMA
//     GEMM (gemm_subtract);
//  2. L Y = I, block rows top-down: Z = E_K - L[K,:k0] Y[:k0,:] (gemm_mc_store),
//     Y[K,:] = L_KK^-1 Z (column-wise substitution, gj_solve_cols_kernel);
//  3. L^H X = Y, block rows bottom-up: Z = Y[K,:] - L[I,K]^H X[I,:]
//     (gemm_project), X[K,:] = L_KK^-H Z.
// Triangular blocks are solved with, never multiplied by their inverses: a
// blocked Gauss-Jordan with explicit 64 x 64 pivot inverses measured a 3 %
// error at cond 3e9 (this scheme: 1.6e-7, like LAPACK's potrf/potrs).
// A diagonal that is not a finite positive number (not numerically positive
// definite) sends the whole inverse to an unblocked Gauss-Jordan with partial
// pivoting (Numerical-Recipes style row interchanges, columns unscrambled at
// the end): like the reference's LDL^T it still returns an inverse; an
// exactly singular matrix raises DegeneracyError.

__device__ __forceinline__ double2 gj_mul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 gj_mulc(double2 a, double2 b) {  // a conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ double2 gj_inv(double2 p) {
  const double q = p.x * p.x + p.y * p.y;
  return make_double2(p.x / q, -p.y / q);
}

// One CTA: the diagonal block W[K,K] (b <= 64, lower part) -> L11 (Cholesky,
// right-looking in shared memory), written to L (ld b, upper part zero).
// *bad = 1 on a diagonal that is not a finite positive number.
__global__ void __launch_bounds__(256) gj_chol_block_kernel(const double2* __restrict__ W, int64_t ldw, int64_t k0,
                                                           int b, double2* __restrict__ Lout, int* __restrict__ bad) {
  extern __shared__ double2 gm[];  // b x b
  double2* L = gm;
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int i = e % b, c = e / b;
    L[e] = i >= c ? W[(k0 + i) + (k0 + c) * ldw] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int j = 0; j < b; ++j) {
    const double dj = L[j + j * b].x;
    if (threadIdx.x == 0 && !(dj > 0.0 && dj < INFINITY)) *bad = 1;
    const double l = sqrt(dj), il = 1.0 / l;
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < b; i += blockDim.x)
      L[i + j * b] = make_double2(L[i + j * b].x * il, L[i + j * b].y * il);
    if (threadIdx.x == 0) L[j + j * b] = make_double2(l, 0.0);
    __syncthreads();
    // trailing lower part: L[i,c] -= L[i,j] conj(L[c,j]), j < c <= i
    const int m = b - j - 1;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      const int i = j + 1 + e % m, c = j + 1 + e / m;
      if (c <= i) {
        const double2 f = gj_mulc(L[i + j * b], L[c + j * b]);
        L[i + c * b] = make_double2(L[i + c * b].x - f.x, L[i + c * b].y - f.y);
      }
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) Lout[e] = L[e];
}

// L21 = A21 L11^-H in place: rows [r0, r0 + m) of W, columns [c0, c0 + b); one
// thread per row: x_i = (a_i - sum_{k<i} x_k conj(L[i,k])) / L[i,i]
__global__ void __launch_bounds__(128) gj_trsm_rows_kernel(double2* __restrict__ W, int64_t ldw, int64_t r0, int64_t m,
                                                          int64_t c0, int b, const double2* __restrict__ Lg) {
  extern __shared__ double2 gl[];
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) gl[e] = Lg[e];
  __syncthreads();
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= m) return;
  double2* row = W + r0 + r + c0 * ldw;
  for (int i = 0; i < b; ++i) {
    double2 acc = row[i * ldw];
    for (int k = 0; k < i; ++k) {
      const double2 f = gj_mulc(row[k * ldw], gl[i + k * b]);
      acc.x -= f.x;
      acc.y -= f.y;
    }
    const double il = 1.0 / gl[i + i * b].x;
    row[i * ldw] = make_double2(acc.x * il, acc.y * il);
  }
}

// Z (b x cols, ld b) <- L^-1 Z (FWD) or L^-H Z (backward), one thread per column
template <bool FWD>
__global__ void __launch_bounds__(128) gj_solve_cols_kernel(double2* __restrict__ Z, int b, int64_t cols,
                                                           const double2* __restrict__ Lg) {
  extern __shared__ double2 gl[];
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) gl[e] = Lg[e];
  __syncthreads();
  const int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j >= cols) return;
  double2* z = Z + j * b;
  if constexpr (FWD) {
    for (int i = 0; i < b; ++i) {  // y_i = (z_i - sum_{k<i} L[i,k] y_k) / L[i,i]
      double2 acc = z[i];
      for (int k = 0; k < i; ++k) {
        const double2 f = gj_mul(gl[i + k * b], z[k]);
        acc.x -= f.x;
        acc.y -= f.y;
      }
      const double il = 1.0 / gl[i + i * b].x;
      z[i] = make_double2(acc.x * il, acc.y * il);
    }
  } else {
    for (int i = b - 1; i >= 0; --i) {  // x_i = (z_i - sum_{k>i} conj(L[k,i]) x_k) / L[i,i]
      double2 acc = z[i];
      for (int k = i + 1; k < b; ++k) {
        const double2 f = gj_mulc(z[k], gl[k + i * b]);
        acc.x -= f.x;
        acc.y -= f.y;
      }
      const double il = 1.0 / gl[i + i * b].x;
      z[i] = make_double2(acc.x * il, acc.y * il);
    }
  }
}

// out (c x r, ld c) = in^H for in (r x c, ld r)
__global__ void gj_conj_transpose_kernel(const double2* __restrict__ in, int64_t r, int c, double2* __restrict__ out) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < r * c;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e % r, j = e / r;
    const double2 v = in[e];
    out[j + i * c] = make_double2(v.x, -v.y);
  }
}

// Z[:, c0 : c0 + b] = I (Z: b x *, ld b)
__global__ void gj_identity_cols_kernel(double2* __restrict__ Z, int b, int64_t c0) {
  for (int e = threadIdx.x; e < b * b; e += blockDim.x)
    Z[(e % b) + (c0 + e / b) * b] = make_double2((e % b) == (e / b) ? 1.0 : 0.0, 0.0);
}

// Z[i + j b] += Y[(k0 + i) + j ldy], j < cols
__global__ void gj_add_rows_kernel(double2* __restrict__ Z, int b, int64_t cols, const double2* __restrict__ Y,
                                   int64_t ldy, int64_t k0) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < b * cols;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e % b, j = e / b;
    const double2 y = Y[(k0 + i) + j * ldy];
    Z[e] = make_double2(Z[e].x + y.x, Z[e].y + y.y);
  }
}

// ---- fallback: unblocked Gauss-Jordan with partial pivoting (column k) ----
// pivot = argmax_{i >= k} |W[i,k]| (ties: smallest i), rows k and pivot swapped,
// row k scaled by 1/pivot (W[k,k] keeps the pivot until gjp_column_kernel)
__global__ void __launch_bounds__(1024) gjp_pivot_kernel(double2* __restrict__ W, int64_t ldw, int64_t n, int64_t k,
                                                        int* __restrict__ piv, double2* __restrict__ ipiv,
                                                        int* __restrict__ bad) {
  __shared__ double sv[32];
  __shared__ int64_t si[32];
  __shared__ int64_t sp;
  double best = -1.0;
  int64_t bi = n;
  for (int64_t i = k + threadIdx.x; i < n; i += blockDim.x) {
    const double2 v = W[i + k * ldw];
    const double m = v.x * v.x + v.y * v.y;
    if (m > best) { best = m; bi = i; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_down_sync(0xffffffffu, best, o);
    const int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = best; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
      if (sv[w] > best || (sv[w] == best && si[w] < bi)) { best = sv[w]; bi = si[w]; }
    if (!(best > 0.0)) { *bad = 2; bi = k; }
    piv[k] = static_cast<int>(bi);
    sp = bi;
  }
  __syncthreads();
  const int64_t p = sp;
  const double2 pv = W[p + k * ldw];
  const double2 ip = gj_inv(pv);
  __syncthreads();  // every thread read the pivot before the swap moves it
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    double2 vk = W[k + j * ldw];
    const double2 vp = W[p + j * ldw];
    if (p != k) W[p + j * ldw] = vk;
    vk = vp;
    W[k + j * ldw] = j == k ? vk : gj_mul(vk, ip);
  }
  if (threadIdx.x == 0) *ipiv = ip;
}
// W[i,j] -= W[i,k] W[k,j] for i, j != k (row k already scaled)
__global__ void gjp_eliminate_kernel(double2* __restrict__ W, int64_t ldw, int64_t n, int64_t k) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n * n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e % n, j = e / n;
    if (i == k || j == k) continue;
    const double2 f = gj_mul(W[i + k * ldw], W[k + j * ldw]);
    W[i + j * ldw] = make_double2(W[i + j * ldw].x - f.x, W[i + j * ldw].y - f.y);
  }
}
// column k: W[i,k] = -W[i,k] / pivot, W[k,k] = 1 / pivot
__global__ void gjp_column_kernel(double2* __restrict__ W, int64_t ldw, int64_t n, int64_t k,
                                  const double2* __restrict__ ipiv) {
  const double2 ip = *ipiv;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (i == k) W[k + k * ldw] = ip;
    else {
      const double2 f = gj_mul(W[i + k * ldw], ip);
      W[i + k * ldw] = make_double2(-f.x, -f.y);
    }
  }
}
// undo the row interchanges: columns k and piv[k] swapped, k = n-1 .. 0 (one thread per row)
__global__ void gjp_unscramble_kernel(double2* __restrict__ W, int64_t ldw, int64_t n, const int* __restrict__ piv) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    for (int64_t k = n - 1; k >= 0; --k) {
      const int64_t p = piv[k];
      if (p != k) {
        const double2 t = W[i + k * ldw];
        W[i + k * ldw] = W[i + p * ldw];
        W[i + p * ldw] = t;
      }
    }
}

// A (lda) is read only; Ainv (ldi) receives A^{-1}.
struct HermInverse {
  static constexpr int NB = 64;
  DevBuf<double2> w, y, lall, lp, lh, z, ipiv;
  DevBuf<double> partial;
  DevBuf<int> bad, piv;
  HostBuf<int> h_bad;
  void operator()(liecl_b200_ctx* ctx, const double2* A, int64_t lda, int64_t n, double2* Ainv, int64_t ldi) {
    if (n == 0) return;
    cudaStream_t st = ctx->stream;
    const int64_t nblk = (n + NB - 1) / NB;
    w.ensure(static_cast<size_t>(n * n));
    y.ensure(static_cast<size_t>(n * n));
    lall.ensure(static_cast<size_t>(nblk * NB * NB));
    lp.ensure(static_cast<size_t>(n * NB));
    lh.ensure(static_cast<size_t>(n * NB));
    z.ensure(static_cast<size_t>(n * NB));
    partial.ensure(static_cast<size_t>(((n + zg::BM - 1) / zg::BM) * n));
    bad.ensure(1);
    h_bad.ensure(1);
    constexpr int kL = NB * NB * 16;  // one 64 x 64 complex block in shared memory
    func_attr_once(gj_chol_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kL);
    func_attr_once(gj_trsm_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kL);
    func_attr_once(gj_solve_cols_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kL);
    func_attr_once(gj_solve_cols_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kL);
    auto read_bad = [&] {
      CU(cudaMemcpyAsync(h_bad.p, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
      return h_bad.p[0];
    };
    const auto grid = [](int64_t e) { return static_cast<unsigned>(std::min<int64_t>((e + 255) / 256, 4096)); };
    const auto blocks128 = [](int64_t e) { return static_cast<unsigned>((e + 127) / 128); };
    CU(cudaMemcpy2DAsync(w.p, n * sizeof(double2), A, lda * sizeof(double2), n * sizeof(double2), n,
                         cudaMemcpyDeviceToDevice, st));
    CU(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    // 1. Cholesky: W's strictly-lower blocks become L's, the diagonal blocks go to lall
    for (int64_t kb = 0; kb < nblk; ++kb) {
      const int64_t k0 = kb * NB;
      const int b = static_cast<int>(std::min<int64_t>(NB, n - k0));
      const int64_t m = n - k0 - b;
      double2* L = lall.p + kb * NB * NB;
      gj_chol_block_kernel<<<1, 256, b * b * 16, st>>>(w.p, n, k0, b, L, bad.p);
      launched(ctx);
      if (m == 0) break;
      gj_trsm_rows_kernel<<<blocks128(m), 128, b * b * 16, st>>>(w.p, n, k0 + b, m, k0, b, L);  // L21 in place
      launched(ctx);
      double2* l21 = w.p + (k0 + b) + k0 * n;
      CU(cudaMemcpy2DAsync(lp.p, m * sizeof(double2), l21, n * sizeof(double2), m * sizeof(double2), b,
                           cudaMemcpyDeviceToDevice, st));
      gj_conj_transpose_kernel<<<grid(m * b), 256, 0, st>>>(lp.p, m, b, lh.p);  // L21^H (b x m)
      launched(ctx);
      double2* a22 = w.p + (k0 + b) + (k0 + b) * n;
      gemm_subtract(ctx, lp.p, b, m, lh.p, a22, static_cast<int>(m), a22, partial.p, m, n);  // A22 -= L21 L21^H
    }
    if (read_bad() == 0) {
      // 2. L Y = I (Y lower triangular: block row K spans columns [0, k0 + b))
      for (int64_t kb = 0; kb < nblk; ++kb) {
        const int64_t k0 = kb * NB;
        const int b = static_cast<int>(std::min<int64_t>(NB, n - k0));
        const int64_t cols = k0 + b;
        if (k0 > 0) gemm_mc_store(ctx, w.p + k0, n, b, k0, y.p, n, static_cast<int>(k0), z.p, b, -1.0);
        gj_identity_cols_kernel<<<1, 256, 0, st>>>(z.p, b, k0);
        launched(ctx);
        gj_solve_cols_kernel<true><<<blocks128(cols), 128, b * b * 16, st>>>(z.p, b, cols, lall.p + kb * NB * NB);
        launched(ctx);
        CU(cudaMemcpy2DAsync(y.p + k0, n * sizeof(double2), z.p, b * sizeof(double2), b * sizeof(double2), cols,
                             cudaMemcpyDeviceToDevice, st));
        if (cols < n)
          CU(cudaMemset2DAsync(y.p + k0 + cols * n, n * sizeof(double2), 0, b * sizeof(double2), n - cols, st));
      }
      // 3. L^H X = Y, bottom-up, X = Ainv
      for (int64_t kb = nblk - 1; kb >= 0; --kb) {
        const int64_t k0 = kb * NB;
        const int b = static_cast<int>(std::min<int64_t>(NB, n - k0));
        const int64_t m = n - k0 - b;
        if (m > 0)  // Z = -L[I,K]^H X[I,:]
          gemm_project(ctx, w.p + (k0 + b) + k0 * n, b, m, Ainv + (k0 + b), static_cast<int>(n), z.p, -1.0, n, ldi);
        else
          CU(cudaMemsetAsync(z.p, 0, static_cast<size_t>(b * n) * sizeof(double2), st));
        gj_add_rows_kernel<<<grid(b * n), 256, 0, st>>>(z.p, b, n, y.p, n, k0);
        launched(ctx);
        gj_solve_cols_kernel<false><<<blocks128(n), 128, b * b * 16, st>>>(z.p, b, n, lall.p + kb * NB * NB);
        launched(ctx);
        CU(cudaMemcpy2DAsync(Ainv + k0, ldi * sizeof(double2), z.p, b * sizeof(double2), b * sizeof(double2), n,
                             cudaMemcpyDeviceToDevice, st));
      }
      return;
    }
    // not numerically positive definite: pivoted Gauss-Jordan on a fresh copy
    CU(cudaMemcpy2DAsync(Ainv, ldi * sizeof(double2), A, lda * sizeof(double2), n * sizeof(double2), n,
                         cudaMemcpyDeviceToDevice, st));
    CU(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    piv.ensure(static_cast<size_t>(n));
    ipiv.ensure(1);
    const unsigned g_el = static_cast<unsigned>(std::min<int64_t>((n * n + 255) / 256, 8192));
    const unsigned g_n = grid(n);
    for (int64_t k = 0; k < n; ++k) {
      gjp_pivot_kernel<<<1, 1024, 0, st>>>(Ainv, ldi, n, k, piv.p, ipiv.p, bad.p);
      launched(ctx);
      gjp_eliminate_kernel<<<g_el, 256, 0, st>>>(Ainv, ldi, n, k);
      launched(ctx);
      gjp_column_kernel<<<g_n, 256, 0, st>>>(Ainv, ldi, n, k, ipiv.p);
      launched(ctx);
    }
    gjp_unscramble_kernel<<<g_n, 256, 0, st>>>(Ainv, ldi, n, piv.p);
    launched(ctx);
    if (read_bad() == 2) throw Error(LIECL_B200_DEGENERACY, "Gram matrix is singular: no inverse to refresh");
  }
};

class GramEngine {
public:
  GramEngine(liecl_b200_ctx* ctx, int d, const liecl_b200_config& cfg)
      : ctx_(ctx), d_(d), D_(static_cast<int64_t>(d) * d), tol_(cfg.tolerance), floor_(cfg.conditioning_floor),
        interval_(cfg.gram_refresh_interval), record_(cfg.record_log != 0) {
    if (d < 1 || d > 4096)  // 12 qubits: the reference's dense expansion limit (R:include/liecl/dense.hpp:45)
      throw Error(LIECL_B200_INVALID_INPUT, "dense dimension must be in [1, 4096]");
    if (!(tol_ >= 0.0)) throw Error(LIECL_B200_INVALID_INPUT, "tolerance must be non-negative");
    cap_ = cfg.max_dim ? static_cast<int64_t>(cfg.max_dim) : D_;
    bmax_ = cfg.batch_max > 0 ? cfg.batch_max
                              : std::clamp<int64_t>((int64_t(8) << 30) / (2 * D_ * 16), D_ > (int64_t(1) << 20) ? 8 : 64,
                                                    4096);
    if (cfg.deadline_seconds > 0) {
      has_deadline_ = true;
      deadline_ = Clock::now() + std::chrono::duration_cast<Clock::duration>(
                                     std::chrono::duration<double>(cfg.deadline_seconds));
    }
    sqrt_d_ = std::sqrt(static_cast<double>(d));
    C_.ensure(static_cast<size_t>(bmax_ * D_));
    R_.ensure(static_cast<size_t>(bmax_ * D_));
    Y_.ensure(static_cast<size_t>(D_));
    reserve(std::min<int64_t>(cap_ + 1, D_ > (int64_t(1) << 20) ? 8 : 64));  // basis slabs grow with the closure
    partial_.ensure(static_cast<size_t>(((D_ + zg::BM - 1) / zg::BM) * bmax_));
    rn_.ensure(bmax_); hn_.ensure(bmax_); nul_.ensure(bmax_); yn_.ensure(1); s_.ensure(1);
    h_rn_.ensure(bmax_); h_hn_.ensure(bmax_); h_nul_.ensure(bmax_); h_one_.ensure(2);
  }

  int64_t size() const { return n_; }
  liecl_b200_stats stats() {
    liecl_b200_stats s = st_;
    s.dimension = static_cast<uint64_t>(n_);
    s.warnings = warns_.size();
    s.kernels = ctx_->kernels - kernels0_;
    return s;
  }
  const std::vector<Warning>& warnings() const { return warns_; }
  const std::vector<liecl_b200_decision>& log() const { return log_; }

  void run_generators(const double2* gens, int ngens) {
    kernels0_ = ctx_->kernels;
    for (int64_t c0 = 0; c0 < ngens; c0 += bmax_) {
      const int cnt = static_cast<int>(std::min<int64_t>(bmax_, ngens - c0));
      CU(cudaMemcpyAsync(R_.p, gens + c0 * D_, static_cast<size_t>(cnt * D_) * sizeof(double2),
                         cudaMemcpyHostToDevice, ctx_->stream));
      column_norm_kernel<<<cnt, 256, 0, ctx_->stream>>>(R_.p, D_, sqrt_d_, hn_.p);
      launched(ctx_);
      dim3 g2(static_cast<unsigned>(std::min<int64_t>((D_ + 255) / 256, 64)), cnt);
      scale_columns_kernel<<<g2, 256, 0, ctx_->stream>>>(R_.p, hn_.p, tol_, D_, C_.p);
      launched(ctx_);
      check(C_.p, cnt, beta_.p, x_.p, R_.p, rn_.p);
      CU(cudaMemcpyAsync(h_hn_.p, hn_.p, cnt * sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream));
      CU(cudaMemcpyAsync(h_rn_.p, rn_.p, cnt * sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream));
      CU(cudaStreamSynchronize(ctx_->stream));
      for (int j = 0; j < cnt; ++j) h_nul_.p[j] = !(h_hn_.p[j] > tol_);
      ++st_.batches;
      apply(cnt, -1, c0, true);
    }
  }

  void run_closure_pairs() {
    int64_t g = 0;
    int64_t B = std::min<int64_t>(bmax_, 512);
    for (;;) {
      const int64_t avail = n_ * (n_ - 1) / 2;
      if (g >= avail) break;
      if (has_deadline_ && Clock::now() > deadline_)
        throw Error(LIECL_B200_TIMEOUT, "closure computation exceeded its deadline");
      const int cnt = static_cast<int>(std::min(B, avail - g));
      launch_commutator_complex(ctx_, B_.p, d_, g, cnt, tol_, C_.p, hn_.p, nul_.p);
      check(C_.p, cnt, beta_.p, x_.p, R_.p, rn_.p);
      CU(cudaMemcpyAsync(h_nul_.p, nul_.p, cnt * sizeof(int), cudaMemcpyDeviceToHost, ctx_->stream));
      CU(cudaMemcpyAsync(h_rn_.p, rn_.p, cnt * sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream));
      CU(cudaStreamSynchronize(ctx_->stream));
      st_.commutators_evaluated += static_cast<uint64_t>(cnt);
      ++st_.batches;
      const uint64_t before = st_.accepted;
      apply(cnt, g, 0, false);
      g += cnt;
      const uint64_t acc = st_.accepted - before;
      if (acc == 0) B = std::min<int64_t>(2 * B, bmax_);
      else if (acc * 4 > static_cast<uint64_t>(cnt)) B = std::max<int64_t>(std::min<int64_t>(64, bmax_), B / 2);
    }
  }

  void download_basis(double* out) { copy_basis(0, n_, out); }
  // basis elements [first, first+count) -> host
  void copy_basis(int64_t first, int64_t count, double* out) {
    if (first < 0 || count < 0 || first + count > n_) throw Error(LIECL_B200_INVALID_INPUT, "vector range out of bounds");
    if (count == 0) return;
    CU(cudaMemcpyAsync(out, B_.p + first * D_, static_cast<size_t>(count * D_) * sizeof(double2),
                       cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
  }
  // A and A^{-1} as n x n column-major (ld n)
  void download_gram(double* a_out, double* ainv_out) {
    if (n_ == 0) return;
    const size_t pitch = static_cast<size_t>(ld()) * sizeof(double2), w = static_cast<size_t>(n_) * sizeof(double2);
    if (a_out)
      CU(cudaMemcpy2DAsync(a_out, w, A_.p, pitch, w, n_, cudaMemcpyDeviceToHost, ctx_->stream));
    if (ainv_out)
      CU(cudaMemcpy2DAsync(ainv_out, w, Ainv_.p, pitch, w, n_, cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
  }

private:
  int64_t ld() const { return vcap_; }

  // Slots for `need` basis elements: B, A, A^{-1} and the per-batch beta / x
  // scratch grow geometrically up to cap + 1 (a closure of dimension 64 at
  // d = 256 must not allocate d^2 slots). Contents are kept: the batch's beta
  // and x (computed before apply) and A, A^{-1} re-pitched to the new ld.
  void reserve(int64_t need) {
    if (need <= vcap_) return;
    const int64_t nc = std::min<int64_t>(cap_ + 1, std::max<int64_t>(need, 2 * vcap_));
    auto grow1 = [&](DevBuf<double2>& buf, size_t n, size_t live) {
      DevBuf<double2> nb;
      nb.ensure(n);
      if (live > 0) CU(cudaMemcpyAsync(nb.p, buf.p, live * sizeof(double2), cudaMemcpyDeviceToDevice, ctx_->stream));
      CU(cudaStreamSynchronize(ctx_->stream));
      std::swap(buf.p, nb.p);
      std::swap(buf.n, nb.n);
    };
    auto grow2 = [&](DevBuf<double2>& buf) {
      DevBuf<double2> nb;
      nb.ensure(static_cast<size_t>(nc * nc));
      if (n_ > 0)
        CU(cudaMemcpy2DAsync(nb.p, nc * sizeof(double2), buf.p, vcap_ * sizeof(double2), n_ * sizeof(double2), n_,
                             cudaMemcpyDeviceToDevice, ctx_->stream));
      CU(cudaStreamSynchronize(ctx_->stream));
      std::swap(buf.p, nb.p);
      std::swap(buf.n, nb.n);
    };
    grow1(B_, static_cast<size_t>(nc * D_), static_cast<size_t>(n_ * D_));
    grow2(A_);
    grow2(Ainv_);
    grow1(beta_, static_cast<size_t>(nc * bmax_), beta_.n);
    grow1(x_, static_cast<size_t>(nc * bmax_), x_.n);
    grow1(bre_, static_cast<size_t>(nc), bre_.n);
    grow1(xre_, static_cast<size_t>(nc), xre_.n);
    vcap_ = nc;
  }

  // beta = B^H C / d, x = A^{-1} beta, R = C - B x, rn = ||R||
  void check(const double2* Cc, int cnt, double2* beta, double2* x, double2* R, double* rn) {
    if (n_ == 0) {
      column_norm_kernel<<<cnt, 256, 0, ctx_->stream>>>(Cc, D_, sqrt_d_, rn);
      launched(ctx_);
      return;
    }
    gemm_project(ctx_, B_.p, n_, D_, Cc, cnt, beta, 1.0 / d_);
    gemm_mc_store(ctx_, Ainv_.p, ld(), n_, n_, beta, n_, cnt, x, n_, 1.0);
    gemm_subtract(ctx_, B_.p, n_, D_, x, Cc, cnt, R, partial_.p);
    const int mtiles = static_cast<int>((D_ + zg::BM - 1) / zg::BM);
    norm_finalize_kernel<<<(cnt + 255) / 256, 256, 0, ctx_->stream>>>(partial_.p, mtiles, cnt, sqrt_d_, rn);
    launched(ctx_);
  }

  std::string where_str(int64_t l, int64_t m) const {
    return m < 0 ? "generator " + std::to_string(l) : "pair (" + std::to_string(l) + "," + std::to_string(m) + ")";
  }

  void apply(int cnt, int64_t pair_g0, int64_t cand0, bool generators) {
    reserve(std::min<int64_t>(cap_ + 1, n_ + cnt + 1));  // before any pointer into the slabs
    const int64_t n_bs = n_;
    const int64_t ldb = n_bs;  // column stride of the batch's beta / x
    for (int j = 0; j < cnt; ++j) {
      int64_t l, m;
      if (pair_g0 >= 0) pair_from_index(pair_g0 + j, l, m);
      else { l = cand0 + j; m = -1; }
      if (h_nul_.p[j]) {
        if (generators)
          warns_.push_back({"null_generator",
                            "generator " + std::to_string(l) + " has norm " + fmt_double(h_hn_.p[j]) +
                                " and was skipped",
                            h_hn_.p[j]});
        if (record_) log_.push_back({l, m, 1, 0, 0, 0, generators ? h_hn_.p[j] : 0.0});
        continue;
      }
      ++st_.independence_checks;
      const double2* h = C_.p + static_cast<int64_t>(j) * D_;
      double rn = h_rn_.p[j];
      const double2* beta = beta_.p + j * ldb;
      const double2* u = x_.p + j * ldb;
      int rc = 0;
      if (n_ != n_bs && rn > tol_) {  // stale "independent": recompute against the current state
        check(h, 1, bre_.p, xre_.p, Y_.p, yn_.p);
        CU(cudaMemcpyAsync(h_one_.p, yn_.p, sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream));
        CU(cudaStreamSynchronize(ctx_->stream));
        rn = h_one_.p[0];
        beta = bre_.p;
        u = xre_.p;
        rc = 1;
        ++st_.rechecks;
      }
      const bool ind = rn > tol_;
      if (borderline(rn, tol_))
        warns_.push_back({"borderline_residual",
                          where_str(l, m) + ": residual " + fmt_double(rn) + " within 10x of tolerance " +
                              fmt_double(tol_) + (ind ? " (accepted)" : " (rejected)"),
                          rn});
      if (record_) log_.push_back({l, m, 0, ind ? 1 : 0, rc, 0, rn});
      if (!ind) continue;
      if (n_ >= cap_)
        throw Error(LIECL_B200_CAPACITY,
                    "basis size cap of " + std::to_string(cap_) + " exceeded; raise the cap to continue");
      accept(h, beta, u);
      if (rn * rn <= 1e4 * floor_)  // R:src/closure.cpp:451-457
        warns_.push_back({"schur_conditioning", where_str(l, m) + " accepted with near-degenerate Schur complement",
                          rn * rn});
    }
  }

  // MatrixInversionStrategy::accept (R:src/closure.cpp:238-249)
  void accept(const double2* h, const double2* beta, const double2* u) {
    double s = 1.0;  // schur_complement of an empty basis (:48-50)
    if (n_ > 0) {
      schur_kernel<<<1, 256, 0, ctx_->stream>>>(beta, u, n_, s_.p);
      launched(ctx_);
      CU(cudaMemcpyAsync(h_one_.p, s_.p, sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream));
      CU(cudaStreamSynchronize(ctx_->stream));
      s = h_one_.p[0];
    }
    if (s <= floor_)
      throw Error(LIECL_B200_DEGENERACY, "Gram expansion is numerically degenerate for element " + std::to_string(n_) +
                                             " (Schur complement " + std::to_string(s) +
                                             "); the element should have been rejected as dependent");
    CU(cudaMemcpyAsync(B_.p + n_ * D_, h, D_ * sizeof(double2), cudaMemcpyDeviceToDevice, ctx_->stream));
    const int64_t total = (n_ + 1) * (n_ + 1);
    bordered_update_kernel<<<static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 4096)), 256, 0,
                             ctx_->stream>>>(Ainv_.p, A_.p, ld(), n_, u, beta, s);
    launched(ctx_);
    ++n_;
    ++st_.accepted;
    ++since_refresh_;
    if (s < 1e-4 || (interval_ > 0 && since_refresh_ >= interval_)) {
      refresh();
      since_refresh_ = 0;
    }
  }

  // GramState::refresh (R:src/closure.cpp:89-95): A^{-1} recomputed from A
  // (HermInverse; A is Hermitian positive definite while the basis is independent)
  void refresh() { inverse_(ctx_, A_.p, ld(), n_, Ainv_.p, ld()); }

  liecl_b200_ctx* ctx_;
  int d_;
  int64_t D_;
  double tol_, floor_;
  uint64_t interval_;
  bool record_;
  int64_t cap_ = 0, bmax_ = 0, n_ = 0;
  uint64_t since_refresh_ = 0, kernels0_ = 0;
  double sqrt_d_ = 1.0;
  bool has_deadline_ = false;
  Clock::time_point deadline_{};
  liecl_b200_stats st_{};
  std::vector<Warning> warns_;
  std::vector<liecl_b200_decision> log_;
  HermInverse inverse_;
  DevBuf<double2> B_, A_, Ainv_, C_, R_, beta_, x_, Y_, bre_, xre_;
  int64_t vcap_ = 0;  // basis slots allocated (ld of A and A^{-1})
  DevBuf<double> partial_, rn_, hn_, yn_, s_;
  DevBuf<int> nul_;
  HostBuf<double> h_rn_, h_hn_, h_one_;
  HostBuf<int> h_nul_;
};
