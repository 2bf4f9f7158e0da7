// RankEngine -- the rank strategy (Alg. 1) on the B200:
// RankStrategy + rank_independence_check (R:src/closure.cpp:185-212, 500-517;
// R:src/dense.cpp:119-147) inside the same batched cursor loop as the other
// engines. Included by engine.cu inside its anonymous namespace.
//
// The reference stacks vec(B_1..B_n, h) into a d^2 x (n+1) matrix S, takes
// its singular values (BDCSVD) and calls h independent iff all n+1 exceed
// thr * sigma_max, thr = rank_tolerance or eps * max(d^2, n+1). Here S is
// never formed: the engine keeps an orthonormal tuple V and the triangular
// factor R with B = V R (the accepted columns' CGS2 coefficients), so
//   S = [B | h] = [V | r/rho] * T,   T = [[R, beta], [0, rho]],
// beta = beta_1 + beta_2 (both projection passes), rho = ||h - V beta||.
// S and T share their singular values (the left factor has orthonormal
// columns); T is (n+1) x (n+1). One CTA per candidate runs a one-sided
// (Hestenes) Jacobi SVD on T -- high relative accuracy -- and counts. The
// relative threshold is invariant under the 1/sqrt(d) scaling of the
// reference inner product that V and R use.
//
// Certified screen (most candidates never need the SVD). Every column of T
// is the coordinate vector of a unit operator, so 1 <= sigma_max(T) <=
// sqrt(n+1); the last row of T is rho e_n, so sigma_min(T) <= rho; and with
// T^{-1} = [[R^{-1}, -R^{-1} beta / rho], [0, 1/rho]] and |beta| <= 1,
//   sigma_min(T) >= 1 / sqrt(F + (F + 1) / rho^2),   F = ||R^{-1}||_F^2,
// where F is kept exactly up to rounding (an O(n^2) back-substitution per
// accept, rank_backsolve_kernel). A candidate is dependent if rho < thr / 8,
// independent if that lower bound >= 8 thr sqrt(n+1) -- both a factor 8
// clear of the threshold, where the Jacobi SVD's rounding (~m eps sigma_max)
// cannot reach -- and otherwise goes to the Jacobi kernel as before.
// LIECL_B200_RANK_SCREEN=0 sends every candidate to the SVD.

// T of candidate j (m = n + 1 columns, m_pad even, column-major in W_j):
// columns < n from R (upper triangle, ld ldr), column n = (beta_j, rho_j),
// padding column zero.
// sel (optional): slot blockIdx.y builds the T of candidate sel[slot].
__global__ void rank_build_t_kernel(const double2* __restrict__ R, int64_t ldr, int n, const double2* __restrict__ beta,
                                    int64_t ldb, const double* __restrict__ rho, int m_pad, double2* __restrict__ W,
                                    const int* __restrict__ sel) {
  const int slot = blockIdx.y;
  const int j = sel ? sel[slot] : slot;
  double2* T = W + static_cast<int64_t>(slot) * m_pad * m_pad;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < static_cast<int64_t>(m_pad) * m_pad;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e % m_pad), k = static_cast<int>(e / m_pad);
    double2 v = make_double2(0.0, 0.0);
    if (k < n) {
      if (i <= k) v = R[i + k * ldr];
    } else if (k == n) {
      if (i < n) v = beta[i + j * ldb];
      else if (i == n) v = make_double2(rho[j], 0.0);
    }
    T[e] = v;
  }
}

// One-sided Jacobi on the m_pad columns of T_j (one CTA, round-robin
// tournament: the m_pad/2 disjoint pairs of a step go to the warps in
// parallel). Writes indep[j] = (#sigma > thr * sigma_max == m) and the
// extreme singular values.
// T lives in shared memory when it fits (in_smem; every step is then a
// shared-memory round trip instead of an L2 one), else in its global slot.
__global__ void rank_jacobi_kernel(double2* __restrict__ W, int m, int m_pad, double thr, int max_sweeps,
                                   int in_smem, int* __restrict__ indep, double* __restrict__ smin,
                                   double* __restrict__ smax) {
  extern __shared__ double2 s_dyn[];  // [T (m_pad^2) if in_smem] [m_pad column norms^2]
  __shared__ int s_rot;
  const int j = blockIdx.x;
  double2* T = W + static_cast<int64_t>(j) * m_pad * m_pad;
  double* s_norm2 = reinterpret_cast<double*>(s_dyn + (in_smem ? static_cast<int64_t>(m_pad) * m_pad : 0));
  if (in_smem) {
    for (int e = threadIdx.x; e < m_pad * m_pad; e += blockDim.x) s_dyn[e] = T[e];
    T = s_dyn;
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const double eps = 2.220446049250313e-16;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) s_rot = 0;
    __syncthreads();
    for (int step = 0; step < m_pad - 1; ++step) {
      for (int pr = warp; pr < m_pad / 2; pr += nwarps) {
        // round-robin: position 0 fixed, the others rotate
        const int a = pr == 0 ? 0 : 1 + (pr - 1 + step) % (m_pad - 1);
        const int b = 1 + (m_pad - 2 - pr + step) % (m_pad - 1);
        const int p = min(a, b), q = max(a, b);
        double2* tp = T + static_cast<int64_t>(p) * m_pad;
        double2* tq = T + static_cast<int64_t>(q) * m_pad;
        double al = 0.0, be = 0.0, gr = 0.0, gi = 0.0;
        for (int i = lane; i < m_pad; i += 32) {
          const double2 u = tp[i], v = tq[i];
          al += u.x * u.x + u.y * u.y;
          be += v.x * v.x + v.y * v.y;
          gr += u.x * v.x + u.y * v.y;  // conj(u) * v
          gi += u.x * v.y - u.y * v.x;
        }
        al = warp_sum(al), be = warp_sum(be), gr = warp_sum(gr), gi = warp_sum(gi);
        const double g = sqrt(gr * gr + gi * gi);
        // orthogonal to working accuracy (the one-sided Jacobi SVD test
        // |a^H b| <= m eps ||a|| ||b||; tighter never settles under roundoff)
        if (g == 0.0 || g <= m_pad * eps * sqrt(al * be)) continue;
        if (lane == 0) s_rot = 1;
        const double cph = gr / g, sph = gi / g;  // e^{i phi} = gamma / |gamma|
        const double zeta = (be - al) / (2.0 * g);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int i = lane; i < m_pad; i += 32) {
          const double2 u = tp[i], v0 = tq[i];
          const double2 v = make_double2(cph * v0.x + sph * v0.y, cph * v0.y - sph * v0.x);  // e^{-i phi} v
          tp[i] = make_double2(c * u.x - s * v.x, c * u.y - s * v.y);
          tq[i] = make_double2(s * u.x + c * v.x, s * u.y + c * v.y);
        }
      }
      __syncthreads();
    }
    const int rotated = s_rot;
    __syncthreads();
    if (!rotated) break;
  }
  for (int k = warp; k < m_pad; k += nwarps) {
    const double2* tk = T + static_cast<int64_t>(k) * m_pad;
    double a = 0.0;
    for (int i = lane; i < m_pad; i += 32) a += tk[i].x * tk[i].x + tk[i].y * tk[i].y;
    a = warp_sum(a);
    if (lane == 0) s_norm2[k] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double mx = 0.0;
    for (int k = 0; k < m_pad; ++k) mx = fmax(mx, sqrt(s_norm2[k]));
    int rank = 0;
    double mn = mx;
    for (int k = 0; k < m_pad; ++k) {
      const double sv = sqrt(s_norm2[k]);
      if (sv > thr * mx) ++rank;
      if (k < m) mn = fmin(mn, sv);
    }
    indep[j] = rank == m;
    smin[j] = mn;
    smax[j] = mx;
  }
}

__global__ void add_columns_kernel(double2* __restrict__ acc, const double2* __restrict__ add, int64_t n) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    acc[e] = make_double2(acc[e].x + add[e].x, acc[e].y + add[e].y);
}

// R column n = (beta, rho)
__global__ void rank_append_r_kernel(double2* __restrict__ R, int64_t ldr, int n, const double2* __restrict__ beta,
                                     const double* __restrict__ rho) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x)
    R[i + static_cast<int64_t>(n) * ldr] = i < n ? beta[i] : make_double2(*rho, 0.0);
}

// xx[slot] = ||R^{-1} beta_j||^2, j = sel ? sel[slot] : slot: back-substitution
// on the upper-triangular R (column-major, ld ldr), one CTA per column of
// beta, x in xs (n per slot). Block rows of 32 from the bottom: the diagonal
// block is solved by one warp out of shared memory (one shuffle per step),
// the rows above take x_k -= sum_c R[k, i0 + c] x_c with R read down its
// columns (coalesced).
__global__ void __launch_bounds__(256)
rank_backsolve_kernel(const double2* __restrict__ R, int64_t ldr, int n, const double2* __restrict__ beta, int64_t ldb,
                      const int* __restrict__ sel, double2* __restrict__ xs, double* __restrict__ xx) {
  __shared__ double2 s_blk[32][33];
  __shared__ double2 s_x[32];
  __shared__ double s_red[8];
  const int slot = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int j = sel ? sel[slot] : slot;
  double2* x = xs + static_cast<int64_t>(slot) * n;
  for (int i = tid; i < n; i += blockDim.x) x[i] = beta[static_cast<int64_t>(j) * ldb + i];
  __syncthreads();
  for (int i1 = n; i1 > 0; i1 -= 32) {
    const int i0 = i1 > 32 ? i1 - 32 : 0, w = i1 - i0;
    for (int e = tid; e < w * w; e += blockDim.x) {
      const int r = e % w, c = e / w;
      s_blk[r][c] = R[(i0 + r) + static_cast<int64_t>(i0 + c) * ldr];
    }
    __syncthreads();
    if (warp == 0) {
      double2 v = lane < w ? x[i0 + lane] : make_double2(0.0, 0.0);
      for (int c = w - 1; c >= 0; --c) {
        if (lane == c) {  // v / R[c, c]
          const double2 dg = s_blk[c][c];
          const double den = dg.x * dg.x + dg.y * dg.y;
          v = make_double2((v.x * dg.x + v.y * dg.y) / den, (v.y * dg.x - v.x * dg.y) / den);
        }
        const double xr = __shfl_sync(0xffffffffu, v.x, c), xi = __shfl_sync(0xffffffffu, v.y, c);
        if (lane < c) {
          const double2 a = s_blk[lane][c];
          v.x -= a.x * xr - a.y * xi;
          v.y -= a.x * xi + a.y * xr;
        }
      }
      if (lane < w) {
        x[i0 + lane] = v;
        s_x[lane] = v;
      }
    }
    __syncthreads();
    for (int k = tid; k < i0; k += blockDim.x) {
      double2 acc = x[k];
      for (int c = 0; c < w; ++c) {
        const double2 a = R[k + static_cast<int64_t>(i0 + c) * ldr], b = s_x[c];
        acc.x -= a.x * b.x - a.y * b.y;
        acc.y -= a.x * b.y + a.y * b.x;
      }
      x[k] = acc;
    }
    __syncthreads();
  }
  double part = 0.0;
  for (int i = tid; i < n; i += blockDim.x) part += x[i].x * x[i].x + x[i].y * x[i].y;
  part = warp_sum(part);
  if (lane == 0) s_red[warp] = part;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) t += s_red[q];
    xx[slot] = t;
  }
}

// squared row norms of R after the column (beta, rho) joins: rows2[i] +=
// |beta_i|^2, rows2[n] = rho^2; *rmax2 = the largest so far (non-negative
// doubles order like their bit patterns)
__global__ void rank_rows2_kernel(const double2* __restrict__ beta, const double* __restrict__ rho, int n,
                                  double* __restrict__ rows2, unsigned long long* __restrict__ rmax2) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) {
    const double v = i < n ? rows2[i] + beta[i].x * beta[i].x + beta[i].y * beta[i].y : rho[0] * rho[0];
    rows2[i] = v;
    atomicMax(rmax2, static_cast<unsigned long long>(__double_as_longlong(v)));
  }
}

class RankEngine {
public:
  RankEngine(liecl_b200_ctx* ctx, int d, const liecl_b200_config& cfg)
      : ctx_(ctx), d_(d), D_(static_cast<int64_t>(d) * d), tol_(cfg.tolerance), rank_tol_(cfg.rank_tolerance),
        record_(cfg.record_log != 0) {
    if (d < 1 || d > 4096)  // 12 qubits: the reference's dense expansion limit (R:include/liecl/dense.hpp:45)
      throw Error(LIECL_B200_INVALID_INPUT, "dense dimension must be in [1, 4096]");
    if (!(tol_ >= 0.0)) throw Error(LIECL_B200_INVALID_INPUT, "tolerance must be non-negative");
    cap_ = cfg.max_dim ? static_cast<int64_t>(cfg.max_dim) : D_;
    bmax_ = cfg.batch_max > 0 ? cfg.batch_max
                              : std::clamp<int64_t>((int64_t(4) << 30) / (3 * D_ * 16), D_ > (int64_t(1) << 20) ? 4 : 16,
                                                    1024);
    if (cfg.deadline_seconds > 0) {
      has_deadline_ = true;
      deadline_ = Clock::now() + std::chrono::duration_cast<Clock::duration>(
                                     std::chrono::duration<double>(cfg.deadline_seconds));
    }
    sqrt_d_ = std::sqrt(static_cast<double>(d));
    C_.ensure(static_cast<size_t>(bmax_ * D_));
    X_.ensure(static_cast<size_t>(bmax_ * D_));
    reserve(std::min<int64_t>(cap_ + 1, D_ > (int64_t(1) << 20) ? 8 : 64));  // basis slabs grow with the closure
    partial_.ensure(static_cast<size_t>(((D_ + zg::BM - 1) / zg::BM) * bmax_));
    rn_.ensure(bmax_); hn_.ensure(bmax_); nul_.ensure(bmax_); ind_.ensure(bmax_); smin_.ensure(bmax_);
    smax_.ensure(bmax_);
    h_hn_.ensure(bmax_); h_nul_.ensure(bmax_); h_ind_.ensure(bmax_); h_one_.ensure(4);
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
      CU(cudaMemcpyAsync(X_.p, gens + c0 * D_, static_cast<size_t>(cnt * D_) * sizeof(double2),
                         cudaMemcpyHostToDevice, ctx_->stream));
      column_norm_kernel<<<cnt, 256, 0, ctx_->stream>>>(X_.p, D_, sqrt_d_, hn_.p);
      launched(ctx_);
      dim3 g2(static_cast<unsigned>(std::min<int64_t>((D_ + 255) / 256, 64)), cnt);
      scale_columns_kernel<<<g2, 256, 0, ctx_->stream>>>(X_.p, hn_.p, tol_, D_, C_.p);
      launched(ctx_);
      check(C_.p, cnt, X_.p, P1_.p, rn_.p, ind_.p);
      CU(cudaMemcpyAsync(h_hn_.p, hn_.p, cnt * sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream));
      CU(cudaStreamSynchronize(ctx_->stream));
      for (int j = 0; j < cnt; ++j) h_nul_.p[j] = !(h_hn_.p[j] > tol_);
      ++st_.batches;
      apply(cnt, -1, c0, true);
    }
  }

  void run_closure_pairs() {
    int64_t g = 0;
    for (;;) {
      const int64_t avail = n_ * (n_ - 1) / 2;
      if (g >= avail) break;
      if (has_deadline_ && Clock::now() > deadline_)
        throw Error(LIECL_B200_TIMEOUT, "closure computation exceeded its deadline");
      const int cnt = static_cast<int>(std::min<int64_t>(batch_limit(), avail - g));
      launch_commutator_complex(ctx_, B_.p, d_, g, cnt, tol_, C_.p, hn_.p, nul_.p);
      check(C_.p, cnt, X_.p, P1_.p, rn_.p, ind_.p);
      CU(cudaMemcpyAsync(h_nul_.p, nul_.p, cnt * sizeof(int), cudaMemcpyDeviceToHost, ctx_->stream));
      CU(cudaStreamSynchronize(ctx_->stream));
      st_.commutators_evaluated += static_cast<uint64_t>(cnt);
      ++st_.batches;
      apply(cnt, g, 0, false);
      g += cnt;
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

private:
  static constexpr size_t kJacobiSmem = 200 * 1024;
  bool jacobi_attr_ = false;
  int64_t ldr() const { return vcap_; }

  // Slots for `need` basis elements: B, V, R (re-pitched to the new ld) and
  // the batch's projection coefficients P1 (computed before apply, kept)
  // grow geometrically up to cap + 1.
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
    grow1(B_, static_cast<size_t>(nc * D_), static_cast<size_t>(n_ * D_));
    grow1(V_, static_cast<size_t>(nc * D_), static_cast<size_t>(n_ * D_));
    {
      DevBuf<double2> nb;
      nb.ensure(static_cast<size_t>(nc * nc));
      CU(cudaMemsetAsync(nb.p, 0, nb.n * sizeof(double2), ctx_->stream));
      if (n_ > 0)
        CU(cudaMemcpy2DAsync(nb.p, nc * sizeof(double2), R_.p, vcap_ * sizeof(double2), n_ * sizeof(double2), n_,
                             cudaMemcpyDeviceToDevice, ctx_->stream));
      CU(cudaStreamSynchronize(ctx_->stream));
      std::swap(R_.p, nb.p);
      std::swap(R_.n, nb.n);
    }
    {  // squared row norms of R: n_ live entries
      DevBuf<double> nb;
      nb.ensure(static_cast<size_t>(nc + 1));
      if (n_ > 0) CU(cudaMemcpyAsync(nb.p, rows2_.p, n_ * sizeof(double), cudaMemcpyDeviceToDevice, ctx_->stream));
      CU(cudaStreamSynchronize(ctx_->stream));
      std::swap(rows2_.p, nb.p);
      std::swap(rows2_.n, nb.n);
    }
    grow1(P1_, static_cast<size_t>(nc * bmax_), P1_.n);
    grow1(P2_, static_cast<size_t>(nc * bmax_), 0);
    vcap_ = nc;
  }
  int m_pad() const { return static_cast<int>((n_ + 2) & ~int64_t(1)); }
  // candidates per batch: the T matrices (m_pad^2 complex each) within 1 GB
  int64_t batch_limit() const {
    const int64_t m = m_pad();
    return std::clamp<int64_t>((int64_t(1) << 30) / (m * m * 16), 1, bmax_);
  }
  double threshold() const {  // R:src/dense.cpp:133-137
    return rank_tol_ > 0.0 ? rank_tol_ : 2.220446049250313e-16 * static_cast<double>(std::max<int64_t>(D_, n_ + 1));
  }

  // rank verdicts of cnt unit candidates (columns of Cc) against the current
  // state -> ind (device) and h_ind_; residuals -> Xo, beta_1 + beta_2 ->
  // Pacc (ld n), their norms -> rho
  void check(const double2* Cc, int cnt, double2* Xo, double2* Pacc, double* rho, int* ind) {
    const int m = static_cast<int>(n_ + 1), mp = m_pad();
    W_.ensure(static_cast<size_t>(cnt) * mp * mp);
    if (n_ == 0) {
      column_norm_kernel<<<cnt, 256, 0, ctx_->stream>>>(Cc, D_, sqrt_d_, rho);
      launched(ctx_);
      CU(cudaMemcpyAsync(Xo, Cc, static_cast<size_t>(cnt * D_) * sizeof(double2), cudaMemcpyDeviceToDevice,
                         ctx_->stream));
    } else {
      // two CGS passes; T's last column collects both passes' coefficients
      P2_.ensure(static_cast<size_t>(n_) * cnt);
      gemm_project(ctx_, V_.p, n_, D_, Cc, cnt, Pacc, 1.0 / d_);
      gemm_subtract(ctx_, V_.p, n_, D_, Pacc, Cc, cnt, Xo, partial_.p);
      gemm_project(ctx_, V_.p, n_, D_, Xo, cnt, P2_.p, 1.0 / d_);
      gemm_subtract(ctx_, V_.p, n_, D_, P2_.p, Xo, cnt, Xo, partial_.p);
      const int mtiles = static_cast<int>((D_ + zg::BM - 1) / zg::BM);
      norm_finalize_kernel<<<(cnt + 255) / 256, 256, 0, ctx_->stream>>>(partial_.p, mtiles, cnt, sqrt_d_, rho);
      add_columns_kernel<<<grid_for(n_ * cnt), 256, 0, ctx_->stream>>>(Pacc, P2_.p, n_ * cnt);
      launched(ctx_), launched(ctx_);
    }
    // certified screen on the host (see the header); the rest -> Jacobi SVD
    h_rho_.ensure(cnt);
    CU(cudaMemcpyAsync(h_rho_.p, rho, cnt * sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
    const double thr = threshold();
    const double smax_hi = std::sqrt(static_cast<double>(n_ + 1)) * (1.0 + 1e-12);
    // sigma_max(T) >= sigma_max(R) >= its largest row norm, and >= 1 (a unit column)
    const double smax_lo = std::max(1.0, smax_row_) * (1.0 - 1e-12);
    std::vector<int> amb;
    amb.reserve(static_cast<size_t>(cnt));
    for (int j = 0; j < cnt; ++j) {
      const double r = h_rho_.p[j];
      if (screen_ && r < thr * smax_lo / 8.0) {
        h_ind_.p[j] = 0;
      } else if (screen_ && r > 0.0 && 1.0 / std::sqrt(finv_ + (finv_ + 1.0) / (r * r)) >= 8.0 * thr * smax_hi) {
        h_ind_.p[j] = 1;
      } else {
        amb.push_back(j);
      }
    }
    // second stage for the few left: x = R^{-1} beta exactly (back-substitution
    // on the device, rank_backsolve_kernel, one CTA per candidate) gives ||T^{-1}||_F^2 = F + (|x|^2 + 1) / rho^2
    // and ||T^{-1} e_n|| = sqrt(|x|^2 + 1) / rho, i.e.
    //   1 / sqrt(F + (|x|^2 + 1) / rho^2) <= sigma_min(T) <= rho / sqrt(|x|^2 + 1)
    if (screen_ && !amb.empty() && n_ > 0) {
      h_xx_.ensure(amb.size());
      solve_norm2(Pacc, n_, amb.data(), static_cast<int>(amb.size()), h_xx_.p);
      std::vector<int> rest;
      for (size_t q = 0; q < amb.size(); ++q) {
        const int j = amb[q];
        const double r = h_rho_.p[j];
        const double xx = h_xx_.p[q];
        if (r / std::sqrt(xx + 1.0) < thr * smax_lo / 8.0) h_ind_.p[j] = 0;
        else if (r > 0.0 && 1.0 / std::sqrt(finv_ + (xx + 1.0) / (r * r)) >= 8.0 * thr * smax_hi) h_ind_.p[j] = 1;
        else rest.push_back(j);
      }
      amb.swap(rest);
    }
    st_.survivors += amb.size();  // candidates that needed the SVD
    if (trace_ && !amb.empty()) {
      int small = 0;
      double lo = 1e300, hi = 0.0;
      for (int j : amb) {
        small += h_rho_.p[j] < 1e-6;
        lo = std::min(lo, h_rho_.p[j]);
        hi = std::max(hi, h_rho_.p[j]);
      }
      std::fprintf(stderr, "[rank] n=%lld cnt=%d svd=%zu (rho<1e-6: %d) rho in [%.3g, %.3g] F=%.3g thr=%.3g smax_row=%.3g\n",
                   static_cast<long long>(n_), cnt, amb.size(), small, lo, hi, finv_, thr, smax_row_);
    }
    if (amb.empty()) return;
    const int na = static_cast<int>(amb.size());
    W_.ensure(static_cast<size_t>(na) * mp * mp);
    sel_.ensure(na);
    jind_.ensure(na);
    CU(cudaMemcpyAsync(sel_.p, amb.data(), na * sizeof(int), cudaMemcpyHostToDevice, ctx_->stream));
    dim3 gb(static_cast<unsigned>(std::min<int64_t>((static_cast<int64_t>(mp) * mp + 255) / 256, 256)), na);
    rank_build_t_kernel<<<gb, 256, 0, ctx_->stream>>>(R_.p, ldr(), static_cast<int>(n_), Pacc, n_, rho, mp, W_.p,
                                                      sel_.p);
    const size_t t_bytes = static_cast<size_t>(mp) * mp * sizeof(double2);
    const bool in_smem = t_bytes + mp * sizeof(double) <= kJacobiSmem;
    if (!jacobi_attr_) {
      CU(cudaFuncSetAttribute(rank_jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(kJacobiSmem)));
      jacobi_attr_ = true;
    }
    rank_jacobi_kernel<<<na, 256, (in_smem ? t_bytes : 0) + mp * sizeof(double), ctx_->stream>>>(
        W_.p, m, mp, threshold(), 30, in_smem ? 1 : 0, jind_.p, smin_.p, smax_.p);
    launched(ctx_), launched(ctx_);
    h_jind_.ensure(na);
    CU(cudaMemcpyAsync(h_jind_.p, jind_.p, na * sizeof(int), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
    for (int q = 0; q < na; ++q) h_ind_.p[amb[q]] = h_jind_.p[q];
  }
  static unsigned grid_for(int64_t n) { return static_cast<unsigned>(std::clamp<int64_t>((n + 255) / 256, 1, 4096)); }

  std::string where_str(int64_t l, int64_t m) const {
    return m < 0 ? "generator " + std::to_string(l) : "pair (" + std::to_string(l) + "," + std::to_string(m) + ")";
  }

  // verdicts in cursor order (R:src/closure.cpp:440-444): a stale
  // "independent" after an in-batch accept is re-run against the current
  // state; "dependent" stands. The rank check has no residual scale: the log
  // carries 0 like the reference's outcome.
  void apply(int cnt, int64_t pair_g0, int64_t cand0, bool generators) {
    reserve(std::min<int64_t>(cap_ + 1, n_ + cnt + 1));  // before any pointer into the slabs
    const int64_t n_bs = n_;
    std::vector<int> ind(h_ind_.p, h_ind_.p + cnt);
    // re-checks are batched: every stale "independent" left in the batch is
    // re-run at once against the current state; those results hold until the
    // next accept (then the rest is re-run again) -- the same verdicts as
    // re-checking one at a time, with one SVD launch per accept instead of one
    // per candidate
    std::vector<int> rslot(static_cast<size_t>(cnt), -1), rind;
    int64_t r_state = -1;  // basis size the re-check results refer to
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
      bool indep = ind[j] != 0;
      int rc = 0;
      const double2* resid = X_.p + static_cast<int64_t>(j) * D_;
      const double2* beta = P1_.p + j * n_bs;
      const double* rho = rn_.p + j;
      if (n_ != n_bs && indep) {  // stale "independent": recompute against the current state
        if (r_state != n_) {
          std::vector<int> todo;
          for (int k = j; k < cnt; ++k)
            if (!h_nul_.p[k] && ind[k]) todo.push_back(k);
          rind = recheck(todo);
          std::fill(rslot.begin(), rslot.end(), -1);
          for (size_t q = 0; q < todo.size(); ++q) rslot[todo[q]] = static_cast<int>(q);
          r_state = n_;
        }
        const int q = rslot[j];
        indep = rind[q] != 0;
        resid = Xr_.p + static_cast<int64_t>(q) * D_;
        beta = Pr_.p + static_cast<int64_t>(q) * n_;
        rho = rnr_.p + q;
        rc = 1;
        ++st_.rechecks;
      }
      if (record_) log_.push_back({l, m, 0, indep ? 1 : 0, rc, 0, 0.0});
      if (!indep) continue;
      if (n_ >= cap_)
        throw Error(LIECL_B200_CAPACITY,
                    "basis size cap of " + std::to_string(cap_) + " exceeded; raise the cap to continue");
      accept(h, resid, beta, rho);
    }
  }

  // batch candidates `todo` (columns of C_) checked against the current state
  // into the re-check buffers; returns their verdicts (slot q = todo[q])
  std::vector<int> recheck(const std::vector<int>& todo) {
    const int k = static_cast<int>(todo.size());
    Yb_.ensure(static_cast<size_t>(k) * D_);
    Xr_.ensure(static_cast<size_t>(k) * D_);
    Pr_.ensure(static_cast<size_t>(std::max<int64_t>(n_, 1)) * k);
    rnr_.ensure(k);
    indr_.ensure(k);
    idx_.ensure(k);
    CU(cudaMemcpyAsync(idx_.p, todo.data(), k * sizeof(int), cudaMemcpyHostToDevice, ctx_->stream));
    dim3 gg(static_cast<unsigned>(std::min<int64_t>((D_ + 255) / 256, 64)), k);
    gather_columns_kernel<<<gg, 256, 0, ctx_->stream>>>(C_.p, idx_.p, D_, Yb_.p);
    launched(ctx_);
    check(Yb_.p, k, Xr_.p, Pr_.p, rnr_.p, indr_.p);
    return std::vector<int>(h_ind_.p, h_ind_.p + k);
  }

  // RankStrategy::accept (R:src/closure.cpp:200-203): B gets h; V and R grow
  // with the CGS2 residual (rho = 0 cannot be accepted: sigma_min <= rho)
  void accept(const double2* h, const double2* resid, const double2* beta, const double* rho) {
    CU(cudaMemcpyAsync(B_.p + n_ * D_, h, D_ * sizeof(double2), cudaMemcpyDeviceToDevice, ctx_->stream));
    // F = ||R^{-1}||_F^2 after the column (beta, rho) joins R:
    // F += (||R^{-1} beta||^2 + 1) / rho^2; the largest row norm of R bounds
    // sigma_max(R) from below. Both on the device; three doubles come back.
    acc_.ensure(4);
    if (n_ == 0) CU(cudaMemsetAsync(acc_.p, 0, 4 * sizeof(double), ctx_->stream));
    if (n_ > 0) {
      xs_.ensure(static_cast<size_t>(n_));
      rank_backsolve_kernel<<<1, 256, 0, ctx_->stream>>>(R_.p, ldr(), static_cast<int>(n_), beta, n_, nullptr, xs_.p,
                                                         acc_.p);
      launched(ctx_);
    }
    rank_rows2_kernel<<<grid_for(n_ + 1), 256, 0, ctx_->stream>>>(
        beta, rho, static_cast<int>(n_), rows2_.p, reinterpret_cast<unsigned long long*>(acc_.p + 1));
    launched(ctx_);
    CU(cudaMemcpyAsync(acc_.p + 2, rho, sizeof(double), cudaMemcpyDeviceToDevice, ctx_->stream));
    CU(cudaMemcpyAsync(h_one_.p, acc_.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
    const double r = h_one_.p[2];
    finv_ += ((n_ > 0 ? h_one_.p[0] : 0.0) + 1.0) / (r * r);
    smax_row_ = std::sqrt(h_one_.p[1]);
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((D_ + 255) / 256, 256));
    append_scaled_kernel<<<blocks, 256, 0, ctx_->stream>>>(resid, 1.0 / r, D_, V_.p + n_ * D_, nullptr, nullptr);
    rank_append_r_kernel<<<grid_for(n_ + 1), 256, 0, ctx_->stream>>>(R_.p, ldr(), static_cast<int>(n_), beta, rho);
    launched(ctx_), launched(ctx_);
    ++n_;
    ++st_.accepted;
  }

  // ||R^{-1} beta_j||^2 for the columns j = sel[0..count) of beta (ld ldb) -> out (host)
  void solve_norm2(const double2* beta, int64_t ldb, const int* sel, int count, double* out) {
    constexpr int kChunk = 256;  // columns per launch: bounds the x scratch
    xs_.ensure(static_cast<size_t>(std::min(count, kChunk)) * n_);
    sel_.ensure(kChunk);
    xx_.ensure(kChunk);
    for (int c0 = 0; c0 < count; c0 += kChunk) {
      const int c = std::min(kChunk, count - c0);
      CU(cudaMemcpyAsync(sel_.p, sel + c0, c * sizeof(int), cudaMemcpyHostToDevice, ctx_->stream));
      rank_backsolve_kernel<<<c, 256, 0, ctx_->stream>>>(R_.p, ldr(), static_cast<int>(n_), beta, ldb, sel_.p, xs_.p,
                                                         xx_.p);
      launched(ctx_);
      CU(cudaMemcpyAsync(out + c0, xx_.p, c * sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream));
      CU(cudaStreamSynchronize(ctx_->stream));  // sel (pageable) and out are reused per chunk
    }
  }

  liecl_b200_ctx* ctx_;
  int d_;
  int64_t D_;
  double tol_, rank_tol_;
  bool screen_ = [] {
    const char* e = std::getenv("LIECL_B200_RANK_SCREEN");
    return !(e && e[0] == '0');
  }();
  double finv_ = 0.0;  // ||R^{-1}||_F^2
  double smax_row_ = 0.0;  // largest row norm of R
  bool trace_ = std::getenv("LIECL_B200_TRACE") != nullptr;
  int64_t vcap_ = 0;  // basis slots allocated (ld of R)
  bool record_;
  int64_t cap_ = 0, bmax_ = 0, n_ = 0;
  uint64_t kernels0_ = 0;
  double sqrt_d_ = 1.0;
  bool has_deadline_ = false;
  Clock::time_point deadline_{};
  liecl_b200_stats st_{};
  std::vector<Warning> warns_;
  std::vector<liecl_b200_decision> log_;
  DevBuf<double2> B_, V_, R_, C_, X_, Y_, Yb_, P1_, P2_, W_, Xr_, Pr_;
  DevBuf<double> partial_, rn_, hn_, smin_, smax_, rnr_, rows2_, acc_, xx_;
  DevBuf<double2> xs_;
  DevBuf<int> nul_, ind_, indr_, idx_, sel_, jind_;
  HostBuf<double> h_hn_, h_one_, h_rho_, h_xx_;
  HostBuf<int> h_nul_, h_ind_, h_jind_;
};
