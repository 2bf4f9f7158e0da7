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
// inverse update (GramState::expand, :55-87); full refresh from A (Cholesky,
// LU when A is not numerically positive definite; cuSOLVER) when s < 1e-4 or
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

// GramState::refresh's inverse (R:src/closure.cpp:89-95: A.ldlt().solve(I)) on
// the device: Cholesky (zpotrf / zpotrs) for the Hermitian positive definite
// Gram matrix of an independent basis; a matrix that is not numerically
// positive definite takes LU with partial pivoting (zgetrf / zgetrs) and, like
// the reference's LDL^T, still returns an inverse instead of failing.
// A (lda) is read only; Ainv (ldi) receives A^{-1}.
struct HermInverse {
  cusolverDnHandle_t solver = nullptr;
  DevBuf<double2> tmp, work;
  DevBuf<int> info, piv;
  HermInverse() = default;
  HermInverse(const HermInverse&) = delete;
  HermInverse& operator=(const HermInverse&) = delete;
  ~HermInverse() {
    if (solver) cusolverDnDestroy(solver);
  }
  void operator()(liecl_b200_ctx* ctx, const double2* A, int64_t lda, int64_t n, double2* Ainv, int64_t ldi) {
    if (n == 0) return;
    if (!solver && cusolverDnCreate(&solver) != CUSOLVER_STATUS_SUCCESS) throw Error(LIECL_B200_CUDA, "cusolverDnCreate");
    cusolverDnSetStream(solver, ctx->stream);
    const int N = static_cast<int>(n);
    tmp.ensure(static_cast<size_t>(n * n));
    info.ensure(1);
    auto* a = reinterpret_cast<cuDoubleComplex*>(tmp.p);
    auto* b = reinterpret_cast<cuDoubleComplex*>(Ainv);
    auto load = [&] {
      CU(cudaMemcpy2DAsync(tmp.p, n * sizeof(double2), A, lda * sizeof(double2), n * sizeof(double2), n,
                           cudaMemcpyDeviceToDevice, ctx->stream));
      identity_kernel<<<static_cast<unsigned>(std::min<int64_t>((n * n + 255) / 256, 4096)), 256, 0, ctx->stream>>>(
          Ainv, ldi, n);
      launched(ctx);
    };
    auto read_info = [&] {
      int v = 0;
      CU(cudaMemcpyAsync(&v, info.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
      return v;
    };
    load();
    int lwork = 0;
    if (cusolverDnZpotrf_bufferSize(solver, CUBLAS_FILL_MODE_LOWER, N, a, N, &lwork) != CUSOLVER_STATUS_SUCCESS)
      throw Error(LIECL_B200_CUDA, "cusolverDnZpotrf_bufferSize");
    work.ensure(static_cast<size_t>(std::max(lwork, 1)));
    if (cusolverDnZpotrf(solver, CUBLAS_FILL_MODE_LOWER, N, a, N, reinterpret_cast<cuDoubleComplex*>(work.p), lwork,
                         info.p) != CUSOLVER_STATUS_SUCCESS)
      throw Error(LIECL_B200_CUDA, "cusolverDnZpotrf");
    ctx->kernels += 1;
    if (read_info() == 0) {
      if (cusolverDnZpotrs(solver, CUBLAS_FILL_MODE_LOWER, N, N, a, N, b, static_cast<int>(ldi), info.p) !=
          CUSOLVER_STATUS_SUCCESS)
        throw Error(LIECL_B200_CUDA, "cusolverDnZpotrs");
      ctx->kernels += 1;
      return;
    }
    load();  // not positive definite: LU
    if (cusolverDnZgetrf_bufferSize(solver, N, N, a, N, &lwork) != CUSOLVER_STATUS_SUCCESS)
      throw Error(LIECL_B200_CUDA, "cusolverDnZgetrf_bufferSize");
    work.ensure(static_cast<size_t>(std::max(lwork, 1)));
    piv.ensure(static_cast<size_t>(n));
    if (cusolverDnZgetrf(solver, N, N, a, N, reinterpret_cast<cuDoubleComplex*>(work.p), piv.p, info.p) !=
            CUSOLVER_STATUS_SUCCESS ||
        cusolverDnZgetrs(solver, CUBLAS_OP_N, N, N, a, N, piv.p, b, static_cast<int>(ldi), info.p) !=
            CUSOLVER_STATUS_SUCCESS)
      throw Error(LIECL_B200_CUDA, "cuSOLVER LU refresh failed");
    ctx->kernels += 2;
    CU(cudaStreamSynchronize(ctx->stream));
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
  // (Cholesky; A is Hermitian positive definite while the basis is independent)
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
