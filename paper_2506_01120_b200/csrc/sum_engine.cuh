// SumEngine -- the closure loop over multi-term PauliSums on the B200 (SURVEY
// §8 row f2). Replaces run_engine + OrthonormStrategy on the Pauli backend
// (R:src/closure.cpp:142-162, 267-310, 356-473 over R:src/pauli.cpp:78-228,
// R:src/operator.cpp:137-182) bit for bit. Included by engine.cu inside its
// anonymous namespace (Error, CU, DevBuf, HostBuf, launched, Warning, Clock,
// fmt_double, borderline, pair_from_index).
//
// Verdict order is the reference's exactly:
//   * generators are checked one by one against the then-current basis; a
//     batch of generators is checked against the batch-start basis and cut
//     after its first accept (later ones are re-run);
//   * cursor rows are speculative like run_engine: every pair of row l is
//     checked against the row-start basis (basis elements l' < n_limit), then
//     applied in cursor order -- after an accept in the row, a "dependent"
//     speculation stands and an "independent" one is recomputed against the
//     current basis (R:src/closure.cpp:412-460). A device batch spans whole or
//     partial rows; it stops at the end of the first row in which the basis
//     grew, so every row is speculated against its own row-start basis.
// Basis elements live in one append-only term pool (keys + coefficients,
// element l = [off[l], off[l+1])); a key -> (l, coefficient) index with
// per-key lists in ascending l serves sum_inner_product's merge join.

template <class K> class SumEngineT {
public:
  // 1..31 qubits with narrow keys (x | z << 32), 32..64 with WKey {x, z}
  // (pauli_sum.cuh). All ones is the key arrays' marker: on 64 qubits that is
  // the string Y^64, so a 64-qubit closure runs unless Y^64 itself turns up
  // (in an input term or as a bracket's product), which raises
  // InvalidInputError instead of a wrong answer
  static constexpr unsigned kMaxQubits = std::is_same_v<K, psum::WKey> ? 64 : 31;
  // gram = true: Alg. 2 (matrix inversion, R:src/closure.cpp:214-265) -- the
  // pool holds the accepted unit brackets B, a check is beta = <B_l, h>,
  // x = A^{-1} beta (device GEMM against the maintained inverse), residual
  // from_terms(h ++ -x_l B_l) (R:src/closure.cpp:107-131) in one pass, and an
  // accept expands A and A^{-1} (bordered update, refresh as GramEngine)
  SumEngineT(liecl_b200_ctx* ctx, unsigned qubits, bool keep_original, const liecl_b200_config& cfg, bool gram = false)
      : ctx_(ctx), q_(qubits), keep_(keep_original && !gram), gram_(gram), tol_(cfg.tolerance),
        floor_(cfg.conditioning_floor), interval_(cfg.gram_refresh_interval), record_(cfg.record_log != 0) {
    if (qubits < 1 || qubits > kMaxQubits)
      throw Error(LIECL_B200_INVALID_INPUT, "the multi-term PauliSum path supports 1..64 qubits");
    if (!(tol_ >= 0.0)) throw Error(LIECL_B200_INVALID_INPUT, "tolerance must be non-negative");
    const uint64_t full = qubits >= 31 ? static_cast<uint64_t>(INT64_MAX) : (1ull << (2 * qubits));
    cap_ = cfg.max_dim ? static_cast<int64_t>(std::min<uint64_t>(cfg.max_dim, full)) : static_cast<int64_t>(full);
    budget_ = cfg.batch_max > 0 ? cfg.batch_max : (int64_t(1) << 24);
    if (cfg.deadline_seconds > 0) {
      has_deadline_ = true;
      deadline_ = Clock::now() + std::chrono::duration_cast<Clock::duration>(
                                     std::chrono::duration<double>(cfg.deadline_seconds));
    }
    voff_.assign(1, 0);
    ooff_.assign(1, 0);
    need(dvoff_, 1024);
    CU(cudaMemsetAsync(dvoff_.p, 0, sizeof(int64_t), ctx_->stream));
    if (keep_) {
      need(dooff_, 1024);
      CU(cudaMemsetAsync(dooff_.p, 0, sizeof(int64_t), ctx_->stream));
    }
    grow_index(1 << 12);
    need(small_, 4);
    need(marker_flag_, 1);
    CU(cudaMemsetAsync(marker_flag_.p, 0, sizeof(int), ctx_->stream));
  }

  void print_trace() const {
    if (trace_) {
      std::fprintf(stderr,
                   "[sum_engine] n=%lld basis_terms=%lld brackets=%llu batches=%llu rechecks=%llu accepts=%llu "
                   "fused=%llu fallbacks=%llu\n",
                   (long long)n_, (long long)(voff_.empty() ? 0 : voff_.back()),
                   (unsigned long long)st_.commutators_evaluated, (unsigned long long)st_.batches,
                   (unsigned long long)st_.rechecks,
                   (unsigned long long)st_.accepted, (unsigned long long)fused_batches_,
                   (unsigned long long)fused_fallbacks_);
      for (const auto& kv : tsum_)
        std::fprintf(stderr, "[sum_engine] %-10s %9.3f ms  %8llu calls\n", kv.first.c_str(), kv.second.first,
                     (unsigned long long)kv.second.second);
    }
  }

  int64_t size() const { return n_; }
  int64_t terms(bool ortho) const { return (ortho || !keep_) ? voff_.back() : ooff_.back(); }
  liecl_b200_stats stats() const {
    liecl_b200_stats s = st_;
    s.dimension = static_cast<uint64_t>(n_);
    s.warnings = warns_.size();
    return s;
  }
  const std::vector<Warning>& warnings() const { return warns_; }
  const std::vector<liecl_b200_decision>& log() const { return log_; }

  // generators: ngens sums, terms [goff[i], goff[i+1]) of (x, z, coef re/im)
  void run(const int64_t* goff, const uint64_t* gx, const uint64_t* gz, const double* gc, int ngens) {
    try {
      run_impl(goff, gx, gz, gc, ngens);
    } catch (...) {
      print_trace();  // a deadline or capacity stop still reports where the time went
      throw;
    }
  }

  void run_impl(const int64_t* goff, const uint64_t* gx, const uint64_t* gz, const double* gc, int ngens) {
    Stage st_run(this, "run");
    const uint64_t kmask = (q_ >= 64) ? ~0ull : ((1ull << q_) - 1);
    const int64_t nt = ngens > 0 ? goff[ngens] : 0;
    if (nt > (int64_t(1) << 30)) throw Error(LIECL_B200_CAPACITY, "generator terms exceed 2^30");
    std::vector<int> hoff(static_cast<size_t>(ngens) + 1);
    std::vector<K> hkey(static_cast<size_t>(std::max<int64_t>(nt, 1)));
    for (int i = 0; i <= ngens; ++i) hoff[i] = static_cast<int>(goff[i]);
    for (int64_t t = 0; t < nt; ++t) {
      if ((gx[t] & ~kmask) || (gz[t] & ~kmask)) throw Error(LIECL_B200_INVALID_INPUT, "string mask exceeds qubits");
      hkey[t] = psum::kpack<K>(gx[t], gz[t]);
      refuse_marker(hkey[t]);
    }
    Segs g;
    g.shape(ngens, static_cast<int>(nt));
    CU(cudaMemcpyAsync(g.off.p, hoff.data(), hoff.size() * sizeof(int), cudaMemcpyHostToDevice, ctx_->stream));
    if (nt > 0) {
      CU(cudaMemcpyAsync(g.key.p, hkey.data(), nt * sizeof(K), cudaMemcpyHostToDevice,
                         ctx_->stream));
      CU(cudaMemcpyAsync(g.val.p, gc, nt * sizeof(psum::C2), cudaMemcpyHostToDevice, ctx_->stream));
    }
    // generator loop (R:src/closure.cpp:378-403): norms, units, then checks
    DevBuf<double> gn;
    gn.ensure(std::max(ngens, 1));
    std::vector<double> h_gn(static_cast<size_t>(std::max(ngens, 1)));
    if (ngens > 0) {
      psum::seg_norm_kernel<<<grid(ngens), 256, 0, ctx_->stream>>>(g.off.p, ngens, g.val.p, gn.p);
      launched(ctx_);
      psum::seg_scale_kernel<<<std::min(ngens, 4096), 256, 0, ctx_->stream>>>(g.off.p, ngens, gn.p, tol_, g.val.p);
      launched(ctx_);
      CU(cudaMemcpyAsync(h_gn.data(), gn.p, ngens * sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream));
      CU(cudaStreamSynchronize(ctx_->stream));
    }
    int i = 0;
    while (i < ngens) {
      check_deadline();
      Segs sub;
      subrange(g, i, ngens, sub);
      std::vector<double> rn;
      Segs res;
      check(sub, static_cast<int>(n_), res, rn);
      int next = ngens;
      for (int k = 0; i + k < ngens; ++k) {
        const int gi = i + k;
        if (!(h_gn[gi] > tol_)) {
          warns_.push_back({"null_generator",
                            "generator " + std::to_string(gi) + " has norm " + fmt_double(h_gn[gi]) +
                                " and was skipped",
                            h_gn[gi]});
          log_decision(gi, -1, 1, 0, 0, h_gn[gi]);
          continue;
        }
        ++st_.independence_checks;
        const bool ind = rn[k] > tol_;
        note(gi, -1, rn[k], ind);
        log_decision(gi, -1, 0, ind ? 1 : 0, 0, rn[k]);
        if (ind) {
          accept(res, k, rn[k], sub, k);
          if (gram_) gram_note(gi, -1, rn[k]);
          next = gi + 1;  // later generators see the new basis
          break;
        }
      }
      i = next;
    }
    ++st_.batches;
    {
      Stage st_cur(this, "cursor");
      cursor_loop();
    }
    print_trace();
  }

  // basis (or orthonormal tuple) -> host arrays: offsets (n+1), x, z, coef
  void download(bool ortho, int64_t* off, uint64_t* x, uint64_t* z, double* coef) {
    const bool v = ortho || !keep_;
    const std::vector<int64_t>& o = v ? voff_ : ooff_;
    const int64_t nt = o.back();
    for (int64_t l = 0; l <= n_; ++l) off[l] = o[l];
    if (nt == 0) return;
    std::vector<K> k(static_cast<size_t>(nt));
    CU(cudaMemcpyAsync(k.data(), (v ? vkey_ : okey_).p, nt * sizeof(K), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaMemcpyAsync(coef, (v ? vval_ : oval_).p, nt * sizeof(psum::C2), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
    for (int64_t t = 0; t < nt; ++t) {
      x[t] = psum::kx(k[t]);
      z[t] = psum::kz(k[t]);
    }
  }

private:
  using C2 = psum::C2;
  // LIECL_B200_TRACE=1: synchronised per-stage wall times (diagnostics)
  bool trace_ = std::getenv("LIECL_B200_TRACE") != nullptr;
  std::map<std::string, std::pair<double, uint64_t>> tsum_;
  struct Stage {
    SumEngineT* e;
    const char* name;
    Clock::time_point t0;
    Stage(SumEngineT* eng, const char* n) : e(eng), name(n) {
      if (e->trace_) {
        cudaStreamSynchronize(e->ctx_->stream);
        t0 = Clock::now();
      }
    }
    ~Stage() {
      if (e->trace_) {
        cudaStreamSynchronize(e->ctx_->stream);
        auto& v = e->tsum_[name];
        v.first += std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
        ++v.second;
      }
    }
  };
  // scratch grows geometrically: batch sizes vary call to call, and every
  // exact-size reallocation would be a device-synchronising cudaFree
  template <class T> static void need(DevBuf<T>& b, size_t n) {
    if (n > b.n) b.ensure(std::max(n, b.n + b.n / 2));
  }
public:
  struct Segs {  // nseg sums on the device: terms [off[p], off[p+1])
    int nseg = 0, total = 0;
    DevBuf<int> off;
    DevBuf<K> key;
    DevBuf<C2> val;
    void shape(int ns, int tot) {
      nseg = ns;
      total = tot;
      need(off, static_cast<size_t>(ns) + 1);
      need(key, static_cast<size_t>(std::max(tot, 1)));
      need(val, static_cast<size_t>(std::max(tot, 1)));
    }
    void swap(Segs& o) {
      std::swap(nseg, o.nseg);
      std::swap(total, o.total);
      std::swap(off.p, o.off.p), std::swap(off.n, o.off.n);
      std::swap(key.p, o.key.p), std::swap(key.n, o.key.n);
      std::swap(val.p, o.val.p), std::swap(val.n, o.val.n);
    }
  };

private:
  static unsigned grid(int64_t n) { return static_cast<unsigned>(std::clamp<int64_t>((n + 255) / 256, 1, 8192)); }
  static constexpr int64_t kMaxItems = int64_t(1) << 30;

  void check_deadline() {
    if (has_deadline_ && Clock::now() > deadline_)
      throw Error(LIECL_B200_TIMEOUT, "closure computation exceeded its deadline");
  }
  void log_decision(int64_t l, int64_t m, int nul, int ind, int rc, double rn) {
    if (record_) log_.push_back({l, m, nul, ind, rc, 0, rn});
  }
  std::string where_str(int64_t l, int64_t m) const {
    return m < 0 ? "generator " + std::to_string(l) : "pair (" + std::to_string(l) + "," + std::to_string(m) + ")";
  }
  void note(int64_t l, int64_t m, double rn, bool ind) {  // R:src/closure.cpp:324-337
    if (borderline(rn, tol_))
      warns_.push_back({"borderline_residual",
                        where_str(l, m) + ": residual " + fmt_double(rn) + " within 10x of tolerance " +
                            fmt_double(tol_) + (ind ? " (accepted)" : " (rejected)"),
                        rn});
  }
  int read_int(const int* dev) {
    int v = 0;
    CU(cudaMemcpyAsync(&v, dev, sizeof v, cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
    return v;
  }
  long long read_ll(const long long* dev) {
    long long v = 0;
    CU(cudaMemcpyAsync(&v, dev, sizeof v, cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
    return v;
  }
  template <class T> void grow_keep(DevBuf<T>& b, size_t used, size_t need) {
    Stage st_g(this, "grow_keep");
    if (need <= b.n) return;
    DevBuf<T> nb;
    nb.ensure(std::max(need, 2 * b.n));
    if (used) CU(cudaMemcpyAsync(nb.p, b.p, used * sizeof(T), cudaMemcpyDeviceToDevice, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
    std::swap(b.p, nb.p);
    std::swap(b.n, nb.n);
  }
  // 64 qubits: Y^64 (x = z = all ones) is the key arrays' marker
  static void refuse_marker(const K& k) {
    if (psum::kmarked(k))
      throw Error(LIECL_B200_INVALID_INPUT,
                  "the 64-qubit string Y^64 cannot be a term of the multi-term PauliSum path (it is the key marker)");
  }
  // a bracket's product was Y^64 (products_kernel raised the flag)
  void check_marker_flag() {
    if (q_ < 64) return;
    if (read_int(marker_flag_.p))
      throw Error(LIECL_B200_INVALID_INPUT,
                  "a bracket produced the 64-qubit string Y^64, which the multi-term PauliSum path cannot hold "
                  "(it is the key marker)");
  }
  void ensure_temp(size_t bytes) {
    Stage st_t(this, "temp");
    need(temp_, bytes);
  }

  // (kout, vout) = (kin, vin) stably sorted on the keys' low end_bit bits (sort.cuh)
  void sort_pairs(const unsigned long long* kin, unsigned long long* kout, const unsigned* vin, unsigned* vout, int n,
                  int end_bit) {
    ensure_temp(sort::workspace_bytes(n));
    Stage st_s(this, "sort");
    int k = 0;
    sort::pairs(kin, kout, vin, vout, n, end_bit, temp_.p, ctx_->stream, k);
    ctx_->kernels += k;
    CU(cudaGetLastError());
  }

  // int exclusive sum of n flags -> pos (hand-written scan, scan.cuh); returns the total
  int scan_flags(const int* flag, int* pos, int n) {
    Stage st_sc(this, "scan");
    if (n <= 0) return 0;
    need(scan_ws_, static_cast<size_t>(scan::workspace(n)));
    int k = 0;
    const int* total = scan::exclusive<int>(flag, pos, n, scan_ws_.p, ctx_->stream, k);
    ctx_->kernels += k;
    CU(cudaGetLastError());
    return read_int(total);
  }
  // 64-bit exclusive sum of n counts -> pos; returns the total
  long long scan_counts(const long long* cnt, long long* pos, int n) {
    if (n <= 0) return 0;
    need(scan_ws_ll_, static_cast<size_t>(scan::workspace(n)));
    int k = 0;
    const long long* total = scan::exclusive<long long>(cnt, pos, n, scan_ws_ll_.p, ctx_->stream, k);
    ctx_->kernels += k;
    CU(cudaGetLastError());
    return read_ll(total);
  }

  // PauliSum::from_terms on every segment of (off, key, val), n items:
  // out = the merged sums (drop = true) or the raw runs (drop = false, with
  // run_seg_ = each run's segment)
  // pauli_q > 0: keys are packed Pauli strings (kbits = 2q); 0: basis indices
  // below 2^kbits
  void merge(int nseg, const int* off, const K* key, const C2* val, int n, bool drop, Segs& out, int pauli_q,
             int kbits) {
    Stage st_merge(this, drop ? "merge" : "merge_beta");
    if (n == 0) {
      out.shape(nseg, 0);
      CU(cudaMemsetAsync(out.off.p, 0, (nseg + 1) * sizeof(int), ctx_->stream));
      return;
    }
    need(ks_, n);
    need(idx_, n);
    need(is_, n);
    need(seg_, n);
    need(flag_, n);
    need(pos_, n);
    psum::iota_kernel<<<grid(n), 256, 0, ctx_->stream>>>(idx_.p, n);
    launched(ctx_);
    int segbits = 1;
    while ((1ll << segbits) < nseg) ++segbits;
    const int end_bit = segbits + kbits + 1;
    if (end_bit <= 64) {
      // one stable radix sort of (segment | invalid | key) over end_bit bits
      need(ck_, n);
      need(cks_, n);
      psum::combine_kernel<<<grid(n), 256, 0, ctx_->stream>>>(off, nseg, n, key, pauli_q, kbits, ck_.p);
      launched(ctx_);
      sort_pairs(ck_.p, cks_.p, idx_.p, is_.p, n, end_bit);
      psum::split_kernel<<<grid(n), 256, 0, ctx_->stream>>>(cks_.p, n, pauli_q, kbits, ks_.p, seg_.p);
      launched(ctx_), launched(ctx_);
    } else {
      // the key does not fit one 64-bit composite: stable passes from the
      // least significant word up (wide keys: x, then z; narrow: the key),
      // then one over the segment of each term's input position. Unmarked
      // words stay below 2^q, the marker is all ones: q + 1 bits order them.
      need(ck_, n);
      need(cks_, n);
      need(is1_, n);
      constexpr bool wide = std::is_same_v<K, psum::WKey>;
      const int words = (wide && pauli_q > 0) ? 2 : 1;
      const int wbits = !wide ? 64 : std::min(64, (pauli_q > 0 ? pauli_q : kbits) + 1);
      const unsigned* perm = nullptr;  // identity
      unsigned* pp[2] = {is_.p, is1_.p};
      int cur = (words & 1) ? 1 : 0;   // words + 1 sorts in all: the last one writes is_
      for (int w = 0; w < words; ++w) {
        psum::key_words_kernel<K><<<grid(n), 256, 0, ctx_->stream>>>(key, perm, n, w, ck_.p);
        launched(ctx_);
        sort_pairs(ck_.p, cks_.p, perm ? perm : idx_.p, pp[cur], n, wbits);
        perm = pp[cur];
        cur ^= 1;
      }
      psum::seg_words_kernel<<<grid(n), 256, 0, ctx_->stream>>>(off, nseg, perm, n, ck_.p);
      launched(ctx_);
      sort_pairs(ck_.p, cks_.p, perm, pp[cur], n, segbits);
      psum::gather_keys_kernel<<<grid(n), 256, 0, ctx_->stream>>>(key, is_.p, n, ks_.p);
      psum::seg_of_kernel<<<grid(n), 256, 0, ctx_->stream>>>(off, nseg, n, seg_.p);
      launched(ctx_), launched(ctx_);
    }
    psum::heads_kernel<<<grid(n), 256, 0, ctx_->stream>>>(ks_.p, seg_.p, n, flag_.p);
    launched(ctx_);
    const int nruns = scan_flags(flag_.p, pos_.p, n);
    need(rkey_, std::max(nruns, 1));
    need(rval_, std::max(nruns, 1));
    need(rmag_, std::max(nruns, 1));
    need(run_seg_, std::max(nruns, 1));
    need(roff_, nseg + 1);
    psum::run_sum_kernel<<<grid(n), 256, 0, ctx_->stream>>>(ks_.p, is_.p, val, seg_.p, flag_.p, pos_.p, n, rkey_.p,
                                                             rval_.p, rmag_.p, run_seg_.p);
    psum::seg_positions_kernel<<<grid(nseg + 1), 256, 0, ctx_->stream>>>(off, nseg, n, pos_.p, nruns, roff_.p);
    launched(ctx_), launched(ctx_);
    if (!drop) {
      out.shape(nseg, nruns);
      std::swap(out.key.p, rkey_.p), std::swap(out.key.n, rkey_.n);
      std::swap(out.val.p, rval_.p), std::swap(out.val.n, rval_.n);
      std::swap(out.off.p, roff_.p), std::swap(out.off.n, roff_.n);
      return;
    }
    need(keep_flag_, std::max(nruns, 1));
    need(kpos_, std::max(nruns, 1));
    psum::floor_keep_kernel<<<static_cast<unsigned>((nseg + 7) / 8), 256, 0, ctx_->stream>>>(roff_.p, nseg, rmag_.p,
                                                                                        keep_flag_.p);
    launched(ctx_);
    const int nk = nruns > 0 ? scan_flags(keep_flag_.p, kpos_.p, nruns) : 0;
    out.shape(nseg, nk);
    if (nruns > 0) {
      psum::compact_kernel<<<grid(nruns), 256, 0, ctx_->stream>>>(keep_flag_.p, kpos_.p, nruns, rkey_.p, rval_.p,
                                                                  out.key.p, out.val.p);
      launched(ctx_);
    }
    psum::seg_positions_kernel<<<grid(nseg + 1), 256, 0, ctx_->stream>>>(roff_.p, nseg, nruns, kpos_.p, nk,
                                                                         out.off.p);
    launched(ctx_);
  }

  // nseg host sums (terms [off[p], off[p+1]) relative to off[0]) -> device
  void upload(const int64_t* off, const uint64_t* x, const uint64_t* z, const double* coef, int nseg, Segs& out) {
    const int64_t t0 = off[0], nt = off[nseg] - off[0];
    if (nt > kMaxItems) throw Error(LIECL_B200_CAPACITY, "sums exceed 2^30 terms");
    const uint64_t kmask = (q_ >= 64) ? ~0ull : ((1ull << q_) - 1);
    std::vector<int> ho(static_cast<size_t>(nseg) + 1);
    for (int p = 0; p <= nseg; ++p) ho[p] = static_cast<int>(off[p] - t0);
    std::vector<K> hk(static_cast<size_t>(std::max<int64_t>(nt, 1)));
    for (int p = 0; p < nseg; ++p)
      for (int64_t t = off[p]; t < off[p + 1]; ++t) {
        if ((x[t] & ~kmask) || (z[t] & ~kmask)) throw Error(LIECL_B200_INVALID_INPUT, "string mask exceeds qubits");
        hk[t - t0] = psum::kpack<K>(x[t], z[t]);
        refuse_marker(hk[t - t0]);
        if (t > off[p] && !psum::kless(hk[t - 1 - t0], hk[t - t0]))
          throw Error(LIECL_B200_INVALID_INPUT, "sum terms must be unique and sorted by (z, x)");
      }
    out.shape(nseg, static_cast<int>(nt));
    CU(cudaMemcpyAsync(out.off.p, ho.data(), ho.size() * sizeof(int), cudaMemcpyHostToDevice, ctx_->stream));
    if (nt > 0) {
      CU(cudaMemcpyAsync(out.key.p, hk.data(), nt * sizeof(K), cudaMemcpyHostToDevice, ctx_->stream));
      CU(cudaMemcpyAsync(out.val.p, coef + 2 * t0, nt * sizeof(C2), cudaMemcpyHostToDevice, ctx_->stream));
    }
    CU(cudaStreamSynchronize(ctx_->stream));  // host staging vectors
  }
  // the beta runs of the last pass over ONE segment -> dense host vector (n_ complex)
  void beta_to_host(double* beta) {
    const int nr = beta_.total;
    if (nr == 0) return;
    std::vector<K> l(static_cast<size_t>(nr));
    std::vector<C2> v(static_cast<size_t>(nr));
    CU(cudaMemcpyAsync(l.data(), beta_.key.p, nr * sizeof(K), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaMemcpyAsync(v.data(), beta_.val.p, nr * sizeof(C2), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
    for (int r = 0; r < nr; ++r) {
      const int64_t li = psum::kindex(l[r]);
      beta[2 * li] = v[r].re;
      beta[2 * li + 1] = v[r].im;
    }
  }

  // One linear_combination pass (project_residual, R:src/closure.cpp:142-162):
  // out = from_terms(in * (1,0) ++ V_l * (-beta_l)), beta_l = <V_l, in>, for
  // basis elements l < n_limit. Returns false when the batch is too large
  // (the caller splits it).
  bool pass(const Segs& in, int n_limit, Segs& out) {
    Stage st_pass(this, "pass");
    if (!overlap_runs(in, n_limit)) return false;
    return combine(in, C2{1.0, 0.0}, true, out);
  }

  // beta runs of every segment of `in` against V_0..V_{n_limit-1}: beta_
  // (per segment, ascending l; run_seg_ = each run's segment). False when too large.
  bool overlap_runs(const Segs& in, int n_limit) {
    const int n = in.total, nseg = in.nseg;
    need(cnt_, std::max(n, 1));
    need(cpos_, std::max(n, 1));
    if (n > 0) {
      psum::beta_count_kernel<<<grid(n), 256, 0, ctx_->stream>>>(ix_, in.key.p, n, n_limit, cnt_.p);
      launched(ctx_);
    }
    const long long nb = n > 0 ? scan_counts(cnt_.p, cpos_.p, n) : 0;
    if (nb > kMaxItems) return false;
    need(bl_, std::max<long long>(nb, 1));
    need(bv_, std::max<long long>(nb, 1));
    need(boff_, nseg + 1);
    if (n > 0) {
      psum::beta_fill_kernel<<<grid(n), 256, 0, ctx_->stream>>>(ix_, in.key.p, in.val.p, n, n_limit, cpos_.p, bl_.p,
                                                                bv_.p);
      launched(ctx_);
    }
    psum::seg_offsets64_kernel<<<grid(nseg + 1), 256, 0, ctx_->stream>>>(in.off.p, nullptr, nseg, n, cpos_.p, nb,
                                                                         boff_.p);
    launched(ctx_);
    int lbits = 1;
    while ((1ll << lbits) < n_limit) ++lbits;
    merge(nseg, boff_.p, bl_.p, bv_.p, static_cast<int>(nb), false, beta_, 0, lbits);  // beta runs, ascending l
    return true;
  }

  // out = from_terms(base * in ++ coefficient_r * V_l(r) over the runs r of
  // beta_ (per segment, ascending l; run_seg_ = each run's segment)), with
  // coefficient_r = -beta_r (negate: a projection pass) or beta_r as given
  bool combine(const Segs& in, C2 base, bool negate, Segs& out) {
    const int nseg = in.nseg;
    const int nruns = beta_.total;
    const int nch = nseg + nruns;
    need(chunks_, std::max(nch, 1));
    need(clen_, std::max(nch, 1));
    need(chpos_, std::max(nch, 1));
    psum::chunk_base_kernel<<<grid(nseg), 256, 0, ctx_->stream>>>(in.off.p, beta_.off.p, nseg, base, chunks_.p,
                                                                 clen_.p);
    launched(ctx_);
    if (nruns > 0) {
      psum::chunk_basis_kernel<<<grid(nruns), 256, 0, ctx_->stream>>>(beta_.key.p, beta_.val.p, run_seg_.p, nruns,
                                                                      dvoff_.p, negate, chunks_.p, clen_.p);
      launched(ctx_);
    }
    const long long nt = scan_counts(clen_.p, chpos_.p, nch);
    if (nt > kMaxItems) return false;
    lc_.shape(nseg, static_cast<int>(nt));
    psum::seg_offsets64_kernel<<<grid(nseg + 1), 256, 0, ctx_->stream>>>(nullptr, beta_.off.p, nseg, nch, chpos_.p,
                                                                         nt, lc_.off.p);
    launched(ctx_);
    if (nt > 0) {
      psum::chunk_fill_kernel<<<static_cast<unsigned>(std::min(nch, 65535)), 256, 0, ctx_->stream>>>(
          chunks_.p, chpos_.p, nch, in.key.p, in.val.p, vkey_.p, vval_.p, lc_.key.p, lc_.val.p);
      launched(ctx_);
    }
    merge(nseg, lc_.off.p, lc_.key.p, lc_.val.p, static_cast<int>(nt), true, out, static_cast<int>(q_),
          2 * static_cast<int>(q_));
    return true;
  }

  // OrthonormStrategy::check for every segment of h (unit candidates):
  // residual sums and their norms, against basis elements l < n_limit
  // The fused single-CTA check (pauli_sum.cuh) for batches whose sums fit in
  // shared memory: one launch and one synchronisation instead of two merge
  // pipelines; false (nothing changed) when some candidate outgrows it.
  bool fused_check(const Segs& h, int n_limit, Segs& res, std::vector<double>& rn) {
    // latency path: re-checks and short batches (large batches run faster
    // through the throughput-oriented merges); it switches itself off once
    // candidates keep outgrowing it
    if (!fused_ || h.nseg > kFusedMaxBatch || fused_fallbacks_ > fused_batches_ + 8) return false;
    const int hc = n_limit <= 4096 ? 2048 : (n_limit <= 8192 ? 1024 : 0);
    if (hc == 0) return false;
    const size_t smem = psum::fused_smem_bytes<K>(hc, n_limit);
    if (smem > kFusedSmemMax) return false;
    if (!fused_attr_) {
      CU(cudaFuncSetAttribute(psum::fused_check_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(kFusedSmemMax)));
      fused_attr_ = true;
    }
    const int ns = h.nseg;
    need(fk_, static_cast<size_t>(ns) * hc);
    need(fv_, static_cast<size_t>(ns) * hc);
    need(flen_, ns);
    need(fst_, ns);
    need(frn_, ns);
    psum::fused_check_kernel<<<static_cast<unsigned>(std::min(ns, 65535)), psum::kFusedThreads, smem, ctx_->stream>>>(
        h.off.p, ns, h.key.p, h.val.p, ix_, n_limit, dvoff_.p, vkey_.p, vval_.p, hc, fk_.p, fv_.p, flen_.p, frn_.p,
        fst_.p);
    launched(ctx_);
    std::vector<int> st(static_cast<size_t>(ns)), len(static_cast<size_t>(ns));
    CU(cudaMemcpyAsync(st.data(), fst_.p, ns * sizeof(int), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaMemcpyAsync(len.data(), flen_.p, ns * sizeof(int), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaMemcpyAsync(rn.data(), frn_.p, ns * sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
    for (int p = 0; p < ns; ++p)
      if (st[p] != 0) {
        ++fused_fallbacks_;
        return false;
      }
    std::vector<int> off(static_cast<size_t>(ns) + 1, 0);
    for (int p = 0; p < ns; ++p) off[p + 1] = off[p] + len[p];
    res.shape(ns, off[ns]);
    CU(cudaMemcpyAsync(res.off.p, off.data(), off.size() * sizeof(int), cudaMemcpyHostToDevice, ctx_->stream));
    psum::strided_to_segs_kernel<<<static_cast<unsigned>(std::min(ns, 65535)), 256, 0, ctx_->stream>>>(
        fk_.p, fv_.p, hc, res.off.p, ns, res.key.p, res.val.p);
    launched(ctx_);
    CU(cudaStreamSynchronize(ctx_->stream));  // `off` is a stack buffer
    ++fused_batches_;
    return true;
  }

  // check() with the certified-reject screen (as DenseEngine::apply): after
  // pass 1, a candidate with rn1 <= tol/20 cannot come out independent of
  // pass 2 (||r2|| <= ||r1|| up to rounding; the drop rule only removes
  // terms), nor borderline (tol/20 < tol/10), so pass 2 runs on the others
  // only. Basis, statistics and warnings are the reference's bits either way;
  // only a rejected candidate's log entry would carry rn1, so with the
  // decision log on every candidate takes both passes. index[p] = segment of
  // `res` holding candidate p's residual (-1: certified reject).
  void check_screened(const Segs& h, int n_limit, Segs& res, std::vector<double>& rn, std::vector<int>& index) {
    index.resize(static_cast<size_t>(h.nseg));
    for (int p = 0; p < h.nseg; ++p) index[p] = p;
    if (gram_ || record_ || n_limit == 0 || h.nseg <= kFusedMaxBatch) {
      check(h, n_limit, res, rn);
      return;
    }
    rn.assign(static_cast<size_t>(h.nseg), 0.0);
    Segs& r1 = r1_;
    if (!pass(h, n_limit, r1)) {  // too large for one batch: the splitting path
      check(h, n_limit, res, rn);
      return;
    }
    std::vector<double> rn1(static_cast<size_t>(h.nseg));
    need(rn_dev_, h.nseg);
    psum::seg_norm_kernel<<<grid(h.nseg), 256, 0, ctx_->stream>>>(r1.off.p, r1.nseg, r1.val.p, rn_dev_.p);
    launched(ctx_);
    std::vector<int> off1(static_cast<size_t>(h.nseg) + 1);
    CU(cudaMemcpyAsync(rn1.data(), rn_dev_.p, h.nseg * sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaMemcpyAsync(off1.data(), r1.off.p, off1.size() * sizeof(int), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
    const double screen = tol_ / 20.0;
    std::vector<int> surv;
    for (int p = 0; p < h.nseg; ++p)
      if (rn1[p] > screen) surv.push_back(p);
    st_.survivors += surv.size();
    const int ns = static_cast<int>(surv.size());
    if (ns == h.nseg) {
      if (!pass(r1, n_limit, res)) {
        check(h, n_limit, res, rn);
        return;
      }
    } else {
      // survivors' pass-1 residuals as a batch of their own
      std::vector<int> goff(static_cast<size_t>(ns) + 1, 0), gsrc(static_cast<size_t>(std::max(ns, 1)));
      for (int q = 0; q < ns; ++q) {
        gsrc[q] = off1[surv[q]];
        goff[q + 1] = goff[q] + off1[surv[q] + 1] - off1[surv[q]];
      }
      Segs& sv = rs_;
      sv.shape(ns, goff[ns]);
      need(gsrc_, std::max(ns, 1));
      CU(cudaMemcpyAsync(sv.off.p, goff.data(), goff.size() * sizeof(int), cudaMemcpyHostToDevice, ctx_->stream));
      CU(cudaMemcpyAsync(gsrc_.p, gsrc.data(), std::max(ns, 1) * sizeof(int), cudaMemcpyHostToDevice, ctx_->stream));
      if (ns > 0) {
        psum::gather_segs_kernel<<<static_cast<unsigned>(std::min(ns, 65535)), 256, 0, ctx_->stream>>>(
            r1.key.p, r1.val.p, gsrc_.p, sv.off.p, ns, sv.key.p, sv.val.p);
        launched(ctx_);
      }
      CU(cudaStreamSynchronize(ctx_->stream));  // goff / gsrc are host vectors
      if (ns > 0 && !pass(sv, n_limit, res)) {
        check(h, n_limit, res, rn);
        for (int p = 0; p < h.nseg; ++p) index[p] = p;
        return;
      }
      if (ns == 0) res.shape(0, 0);
      std::fill(index.begin(), index.end(), -1);
      for (int q = 0; q < ns; ++q) index[surv[q]] = q;
    }
    std::vector<double> rn2(static_cast<size_t>(std::max(ns, 1)));
    if (ns > 0) {
      psum::seg_norm_kernel<<<grid(ns), 256, 0, ctx_->stream>>>(res.off.p, ns, res.val.p, rn_dev_.p);
      launched(ctx_);
      CU(cudaMemcpyAsync(rn2.data(), rn_dev_.p, ns * sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream));
      CU(cudaStreamSynchronize(ctx_->stream));
    }
    for (int p = 0; p < h.nseg; ++p) rn[p] = index[p] >= 0 ? rn2[index[p]] : rn1[p];
  }

  void check(const Segs& h, int n_limit, Segs& res, std::vector<double>& rn) {
    rn.assign(static_cast<size_t>(h.nseg), 0.0);
    if (h.nseg == 0) return;
    if (gram_) {
      gram_check(h, n_limit, res, rn);
      return;
    }
    if (fused_check(h, n_limit, res, rn)) return;
    if (n_limit == 0) {  // project_residual of an empty tuple returns h itself
      copy_segs(h, res);
    } else {
      Segs& r1 = depth_ == 0 ? r1_ : *new_scratch();
      ++depth_;
      const bool ok = pass(h, n_limit, r1) && pass(r1, n_limit, res);
      --depth_;
      if (!ok) {
        if (h.nseg == 1) throw Error(LIECL_B200_CAPACITY, "one projection exceeds 2^30 terms");
        // split the batch: segments are independent
        const int half = h.nseg / 2;
        Segs a, b, ra, rb;
        subrange(h, 0, half, a);
        subrange(h, half, h.nseg, b);
        std::vector<double> na, nb;
        check(a, n_limit, ra, na);
        check(b, n_limit, rb, nb);
        concat(ra, rb, res);
        std::copy(na.begin(), na.end(), rn.begin());
        std::copy(nb.begin(), nb.end(), rn.begin() + half);
        return;
      }
    }
    need(rn_dev_, h.nseg);
    psum::seg_norm_kernel<<<grid(h.nseg), 256, 0, ctx_->stream>>>(res.off.p, res.nseg, res.val.p, rn_dev_.p);
    launched(ctx_);
    CU(cudaMemcpyAsync(rn.data(), rn_dev_.p, h.nseg * sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
  }

  // ---- Alg. 2 (gram_) ----------------------------------------------------
  // matrix_inversion_residual (R:src/closure.cpp:107-131) for every segment of
  // h against B_0..B_{n_limit-1}: beta and x kept in gb_ / gx_ (column p =
  // segment p) for the accept that may follow
  void gram_check(const Segs& h, int n_limit, Segs& res, std::vector<double>& rn) {
    Stage st_g(this, "gram_check");
    const int nseg = h.nseg;
    if (n_limit == 0) {  // empty basis: residual norm = ||h|| (R:src/closure.cpp:121-123)
      copy_segs(h, res);
    } else {
      const int64_t pool_terms = voff_[n_limit];
      if (static_cast<int64_t>(nseg) * pool_terms + h.total > kMaxItems)
        throw Error(LIECL_B200_CAPACITY, "one Alg. 2 batch exceeds 2^30 terms");
      // beta runs (the first half of a projection pass)
      Segs r1;
      overlap_runs(h, n_limit);
      const int64_t ld = n_limit;
      gld_ = ld;
      need(gb_, static_cast<size_t>(ld * nseg));
      need(gx_, static_cast<size_t>(ld * nseg));
      CU(cudaMemsetAsync(gb_.p, 0, static_cast<size_t>(ld * nseg) * sizeof(double2), ctx_->stream));
      if (beta_.total > 0) {
        psum::scatter_runs_kernel<<<grid(beta_.total), 256, 0, ctx_->stream>>>(
            beta_.key.p, beta_.val.p, run_seg_.p, beta_.total, ld, reinterpret_cast<C2*>(gb_.p));
        launched(ctx_);
      }
      // x = A^{-1} beta
      gemm_mc_store(ctx_, Ainv_.p, gcap_, n_limit, n_limit, gb_.p, ld, nseg, gx_.p, ld, 1.0);
      // runs (l, x_l) for every l, then h - sum_l x_l B_l
      const int64_t nr = ld * nseg;
      beta_.shape(nseg, static_cast<int>(nr));
      need(run_seg_, static_cast<size_t>(nr));
      psum::dense_runs_kernel<<<grid(nr), 256, 0, ctx_->stream>>>(reinterpret_cast<const C2*>(gx_.p), n_limit, nseg,
                                                                   beta_.key.p, beta_.val.p, run_seg_.p, beta_.off.p);
      launched(ctx_);
      if (!combine(h, C2{1.0, 0.0}, true, res)) throw Error(LIECL_B200_CAPACITY, "one Alg. 2 batch exceeds 2^30 terms");
    }
    need(rn_dev_, nseg);
    psum::seg_norm_kernel<<<grid(nseg), 256, 0, ctx_->stream>>>(res.off.p, nseg, res.val.p, rn_dev_.p);
    launched(ctx_);
    CU(cudaMemcpyAsync(rn.data(), rn_dev_.p, nseg * sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
  }

  // MatrixInversionStrategy::accept (R:src/closure.cpp:238-249) of segment hk of
  // h, whose beta / x are column hk of gb_ / gx_ (from the gram_check that
  // produced the verdict)
  void gram_accept(const Segs& h, int hk) {
    const int64_t n = n_;
    double s = 1.0;  // schur_complement of an empty basis
    if (n > 0) {
      if (gld_ != n) throw Error(LIECL_B200_INTERNAL, "Alg. 2 accept without a current check");
      need(gs_, 1);
      schur_kernel<<<1, 256, 0, ctx_->stream>>>(gb_.p + hk * gld_, gx_.p + hk * gld_, n, gs_.p);
      launched(ctx_);
      CU(cudaMemcpyAsync(&s, gs_.p, sizeof s, cudaMemcpyDeviceToHost, ctx_->stream));
      CU(cudaStreamSynchronize(ctx_->stream));
    }
    if (s <= floor_)
      throw Error(LIECL_B200_DEGENERACY, "Gram expansion is numerically degenerate for element " + std::to_string(n) +
                                             " (Schur complement " + std::to_string(s) +
                                             "); the element should have been rejected as dependent");
    if (n + 1 > gcap_) {  // A, A^{-1} grow geometrically, re-pitched
      const int64_t nc = std::max<int64_t>(n + 1, std::max<int64_t>(64, 2 * gcap_));
      auto grow = [&](DevBuf<double2>& b) {
        DevBuf<double2> nb;
        nb.ensure(static_cast<size_t>(nc * nc));
        if (n > 0)
          CU(cudaMemcpy2DAsync(nb.p, nc * sizeof(double2), b.p, gcap_ * sizeof(double2), n * sizeof(double2), n,
                               cudaMemcpyDeviceToDevice, ctx_->stream));
        CU(cudaStreamSynchronize(ctx_->stream));
        std::swap(b.p, nb.p);
        std::swap(b.n, nb.n);
      };
      grow(A_);
      grow(Ainv_);
      gcap_ = nc;
    }
    const int64_t total = (n + 1) * (n + 1);
    bordered_update_kernel<<<static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 4096)), 256, 0,
                             ctx_->stream>>>(Ainv_.p, A_.p, gcap_, n, n > 0 ? gx_.p + hk * gld_ : nullptr,
                                             n > 0 ? gb_.p + hk * gld_ : nullptr, s);
    launched(ctx_);
    int h0 = 0, h1 = 0;
    CU(cudaMemcpyAsync(&h0, h.off.p + hk, sizeof(int), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaMemcpyAsync(&h1, h.off.p + hk + 1, sizeof(int), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
    append_pool(h.key.p + h0, h.val.p + h0, h1 - h0, 0.0);  // B gains the unit bracket itself
    ++n_;
    ++st_.accepted;
    gld_ = -1;  // the kept beta / x no longer match the basis
    if (++since_refresh_, s < 1e-4 || (interval_ > 0 && since_refresh_ >= interval_)) {
      inverse_(ctx_, A_.p, gcap_, n_, Ainv_.p, gcap_);  // GramState::refresh (R:src/closure.cpp:89-95)
      since_refresh_ = 0;
    }
  }
  void gram_note(int64_t l, int64_t m, double rn) {  // R:src/closure.cpp:451-457
    if (rn * rn <= 1e4 * floor_)
      warns_.push_back({"schur_conditioning", where_str(l, m) + " accepted with near-degenerate Schur complement",
                        rn * rn});
  }

  void copy_segs(const Segs& a, Segs& b) {
    b.shape(a.nseg, a.total);
    CU(cudaMemcpyAsync(b.off.p, a.off.p, (a.nseg + 1) * sizeof(int), cudaMemcpyDeviceToDevice, ctx_->stream));
    if (a.total > 0) {
      CU(cudaMemcpyAsync(b.key.p, a.key.p, a.total * sizeof(K), cudaMemcpyDeviceToDevice,
                         ctx_->stream));
      CU(cudaMemcpyAsync(b.val.p, a.val.p, a.total * sizeof(C2), cudaMemcpyDeviceToDevice, ctx_->stream));
    }
  }
  // segments [a, b) of src as a batch of their own
  void subrange(const Segs& src, int a, int b, Segs& dst) {
    int lo = 0, hi = 0;
    CU(cudaMemcpyAsync(&lo, src.off.p + a, sizeof(int), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaMemcpyAsync(&hi, src.off.p + b, sizeof(int), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
    dst.shape(b - a, hi - lo);
    psum::rebase_kernel<<<grid(b - a + 1), 256, 0, ctx_->stream>>>(src.off.p, a, b - a, dst.off.p);
    launched(ctx_);
    if (hi > lo) {
      CU(cudaMemcpyAsync(dst.key.p, src.key.p + lo, (hi - lo) * sizeof(K), cudaMemcpyDeviceToDevice,
                         ctx_->stream));
      CU(cudaMemcpyAsync(dst.val.p, src.val.p + lo, (hi - lo) * sizeof(C2), cudaMemcpyDeviceToDevice, ctx_->stream));
    }
  }
  void concat(const Segs& a, const Segs& b, Segs& out) {
    out.shape(a.nseg + b.nseg, a.total + b.total);
    std::vector<int> ho(static_cast<size_t>(a.nseg + b.nseg) + 1);
    CU(cudaMemcpyAsync(ho.data(), a.off.p, (a.nseg + 1) * sizeof(int), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaMemcpyAsync(ho.data() + a.nseg, b.off.p, (b.nseg + 1) * sizeof(int), cudaMemcpyDeviceToHost,
                       ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
    for (int p = a.nseg; p <= a.nseg + b.nseg; ++p) ho[p] += a.total;
    CU(cudaMemcpyAsync(out.off.p, ho.data(), ho.size() * sizeof(int), cudaMemcpyHostToDevice, ctx_->stream));
    if (a.total) {
      CU(cudaMemcpyAsync(out.key.p, a.key.p, a.total * sizeof(K), cudaMemcpyDeviceToDevice,
                         ctx_->stream));
      CU(cudaMemcpyAsync(out.val.p, a.val.p, a.total * sizeof(C2), cudaMemcpyDeviceToDevice, ctx_->stream));
    }
    if (b.total) {
      CU(cudaMemcpyAsync(out.key.p + a.total, b.key.p, b.total * sizeof(K), cudaMemcpyDeviceToDevice,
                         ctx_->stream));
      CU(cudaMemcpyAsync(out.val.p + a.total, b.val.p, b.total * sizeof(C2), cudaMemcpyDeviceToDevice,
                         ctx_->stream));
    }
    CU(cudaStreamSynchronize(ctx_->stream));  // ho is a stack buffer
  }

  // ---- basis pools + index ----------------------------------------------
  void grow_index(uint64_t slots) {
    DevBuf<K> k;
    DevBuf<int> h, t, c;
    k.ensure(slots);
    h.ensure(slots);
    t.ensure(slots);
    c.ensure(slots);
    psum::Index<K> nx = ix_;
    nx.key = k.p, nx.head = h.p, nx.tail = t.p, nx.count = c.p, nx.mask = slots - 1;
    psum::index_reset_kernel<<<grid(static_cast<int64_t>(slots)), 256, 0, ctx_->stream>>>(nx, slots);
    launched(ctx_);
    if (slots_ > 0) {
      psum::index_rehash_kernel<<<grid(static_cast<int64_t>(slots_)), 256, 0, ctx_->stream>>>(ix_, slots_, nx);
      launched(ctx_);
    }
    CU(cudaStreamSynchronize(ctx_->stream));
    std::swap(skey_.p, k.p), std::swap(skey_.n, k.n);
    std::swap(shead_.p, h.p), std::swap(shead_.n, h.n);
    std::swap(stail_.p, t.p), std::swap(stail_.n, t.n);
    std::swap(scount_.p, c.p), std::swap(scount_.n, c.n);
    slots_ = slots;
    sync_index();
  }
  void sync_index() {
    ix_.key = skey_.p, ix_.head = shead_.p, ix_.tail = stail_.p, ix_.count = scount_.p, ix_.mask = slots_ - 1;
    ix_.e_l = el_.p, ix_.e_v = ev_.p, ix_.e_next = enext_.p;
  }

  // V pool + index: append one element (device terms), scaled by 1/rn (rn = 0: as given)
  void append_pool(const K* key, const C2* val, int T, double rn) {
    const int64_t vt = voff_.back();
    grow_keep(vkey_, static_cast<size_t>(vt), static_cast<size_t>(vt + T));
    grow_keep(vval_, static_cast<size_t>(vt), static_cast<size_t>(vt + T));
    if (T > 0) {
      if (rn > 0.0) {
        psum::append_scaled_kernel<<<grid(T), 256, 0, ctx_->stream>>>(key, val, T, rn, vkey_.p + vt, vval_.p + vt);
        launched(ctx_);
      } else {
        CU(cudaMemcpyAsync(vkey_.p + vt, key, T * sizeof(K), cudaMemcpyDeviceToDevice, ctx_->stream));
        CU(cudaMemcpyAsync(vval_.p + vt, val, T * sizeof(C2), cudaMemcpyDeviceToDevice, ctx_->stream));
      }
    }
    // index: keys of one element are distinct; keep the load factor <= 1/2
    keys_upper_ += static_cast<uint64_t>(T);
    if (2 * keys_upper_ > slots_) {
      uint64_t s = slots_;
      while (2 * keys_upper_ > s) s *= 2;
      grow_index(s);
    }
    grow_keep(el_, static_cast<size_t>(entries_), static_cast<size_t>(entries_ + T));
    grow_keep(ev_, static_cast<size_t>(entries_), static_cast<size_t>(entries_ + T));
    grow_keep(enext_, static_cast<size_t>(entries_), static_cast<size_t>(entries_ + T));
    sync_index();
    if (T > 0) {
      psum::index_insert_kernel<<<grid(T), 256, 0, ctx_->stream>>>(ix_, vkey_.p + vt, vval_.p + vt, T,
                                                                   static_cast<int>(n_), static_cast<int>(entries_));
      launched(ctx_);
    }
    entries_ += T;
    voff_.push_back(vt + T);
    grow_keep(dvoff_, voff_.size() - 1, voff_.size());
    CU(cudaMemcpyAsync(dvoff_.p + n_ + 1, &voff_.back(), sizeof(int64_t), cudaMemcpyHostToDevice, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));  // voff_.back() is a vector slot
  }

  // accept residual segment k (norm rn) of res; the candidate h_unit is
  // segment hk of h (the original kept by Alg. 3)
  void accept(const Segs& res, int k, double rn, const Segs& h, int hk) {
    Stage st_acc(this, "accept");
    if (n_ >= cap_)
      throw Error(LIECL_B200_CAPACITY,
                  "basis size cap of " + std::to_string(cap_) + " exceeded; raise the cap to continue");
    if (gram_) {
      gram_accept(h, hk);
      return;
    }
    int r0 = 0, r1 = 0;
    CU(cudaMemcpyAsync(&r0, res.off.p + k, sizeof(int), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaMemcpyAsync(&r1, res.off.p + k + 1, sizeof(int), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
    append_pool(res.key.p + r0, res.val.p + r0, r1 - r0, rn);
    if (keep_) {
      int h0 = 0, h1 = 0;
      CU(cudaMemcpyAsync(&h0, h.off.p + hk, sizeof(int), cudaMemcpyDeviceToHost, ctx_->stream));
      CU(cudaMemcpyAsync(&h1, h.off.p + hk + 1, sizeof(int), cudaMemcpyDeviceToHost, ctx_->stream));
      CU(cudaStreamSynchronize(ctx_->stream));
      const int64_t ot = ooff_.back();
      grow_keep(okey_, static_cast<size_t>(ot), static_cast<size_t>(ot + h1 - h0));
      grow_keep(oval_, static_cast<size_t>(ot), static_cast<size_t>(ot + h1 - h0));
      if (h1 > h0) {
        CU(cudaMemcpyAsync(okey_.p + ot, h.key.p + h0, (h1 - h0) * sizeof(K),
                           cudaMemcpyDeviceToDevice, ctx_->stream));
        CU(cudaMemcpyAsync(oval_.p + ot, h.val.p + h0, (h1 - h0) * sizeof(C2), cudaMemcpyDeviceToDevice,
                           ctx_->stream));
      }
      ooff_.push_back(ot + h1 - h0);
      grow_keep(dooff_, ooff_.size() - 1, ooff_.size());
      CU(cudaMemcpyAsync(dooff_.p + n_ + 1, &ooff_.back(), sizeof(int64_t), cudaMemcpyHostToDevice, ctx_->stream));
    }
    CU(cudaStreamSynchronize(ctx_->stream));  // the host offset sources above are vector slots
    ++n_;
    ++st_.accepted;
  }

  // ---- the cursor loop (R:src/closure.cpp:412-460) -----------------------
  void cursor_loop() {
    int64_t l = 1, m = 0;
    int64_t row_start_n = n_;
    while (l < n_) {
      check_deadline();
      if (m == 0) row_start_n = n_;
      const int n_limit = static_cast<int>(row_start_n);
      // pairs from (l, m) in cursor order, whole rows while the basis has not
      // grown in this row, within the product budget (at least one pair)
      const std::vector<int64_t>& bo = keep_ ? ooff_ : voff_;
      const int64_t g0 = pair_index(l, m);
      std::vector<int> poff(1, 0);
      int64_t prods = 0, ll = l, mm = m;
      for (;;) {
        const int64_t c = (bo[ll + 1] - bo[ll]) * (bo[mm + 1] - bo[mm]);
        if (poff.size() > 1 && prods + c > budget_) break;
        if (prods + c > kMaxItems) throw Error(LIECL_B200_CAPACITY, "one bracket exceeds 2^30 term products");
        prods += c;
        poff.push_back(static_cast<int>(prods));
        if (++mm == ll) {
          ++ll;
          mm = 0;
          if (ll >= n_ || n_ != row_start_n) break;  // next row: only if it exists and nothing grew
        }
        if (static_cast<int64_t>(poff.size()) > (int64_t(1) << 20)) break;
        // Alg. 2 combines every basis element into every candidate: bound the batch's chunk terms
        if (gram_ && static_cast<int64_t>(poff.size()) * voff_[n_] > (int64_t(1) << 28)) break;
      }
      const int cnt = static_cast<int>(poff.size()) - 1;
      // commutators -> merged sums -> norms -> units (K1, R:src/closure.cpp:419-423)
      need(poff_, cnt + 1);
      CU(cudaMemcpyAsync(poff_.p, poff.data(), poff.size() * sizeof(int), cudaMemcpyHostToDevice, ctx_->stream));
      need(pk_, std::max<int64_t>(prods, 1));
      need(pv_, std::max<int64_t>(prods, 1));
      const int64_t* bdoff = keep_ ? dooff_.p : dvoff_.p;
      const K* bkey = keep_ ? okey_.p : vkey_.p;
      const C2* bval = keep_ ? oval_.p : vval_.p;
      Stage st_p(this, "products");
      psum::products_kernel<<<cnt, 256, 0, ctx_->stream>>>(g0, cnt, poff_.p, bdoff, bkey, bval, pk_.p, pv_.p,
                                                           q_ >= 64 ? marker_flag_.p : nullptr);
      launched(ctx_);
      check_marker_flag();
      Segs& h = h_;
      {
        Stage st_c(this, "commutator");
        merge(cnt, poff_.p, pk_.p, pv_.p, static_cast<int>(prods), true, h, static_cast<int>(q_),
              2 * static_cast<int>(q_));
      }
      need(hn_, cnt);
      psum::seg_norm_kernel<<<grid(cnt), 256, 0, ctx_->stream>>>(h.off.p, cnt, h.val.p, hn_.p);
      psum::seg_scale_kernel<<<std::min(cnt, 4096), 256, 0, ctx_->stream>>>(h.off.p, cnt, hn_.p, tol_, h.val.p);
      launched(ctx_), launched(ctx_);
      std::vector<double> hn(static_cast<size_t>(cnt));
      CU(cudaMemcpyAsync(hn.data(), hn_.p, cnt * sizeof(double), cudaMemcpyDeviceToHost, ctx_->stream));
      CU(cudaStreamSynchronize(ctx_->stream));
      // speculative checks against the row-start basis
      Segs& res = res_;
      std::vector<double> rn;
      {
        Stage st_k(this, "check");
        check_screened(h, n_limit, res, rn, res_index_);
      }
      ++st_.batches;
      // ordered apply
      Stage st_apply(this, "apply");
      int j = 0;
      for (; j < cnt; ++j) {
        int64_t pl, pm;
        pair_from_index(g0 + j, pl, pm);
        if (pm == 0 && j > 0 && n_ != row_start_n) break;  // row after growth: speculate again
        if (pm == 0) row_start_n = n_;
        ++st_.commutators_evaluated;
        if (!(hn[j] > tol_)) {
          log_decision(pl, pm, 1, 0, 0, 0.0);
          continue;
        }
        ++st_.independence_checks;
        double r = rn[j];
        int rc = 0;
        if (n_ != row_start_n && r > tol_) {  // stale "independent": recompute (R:src/closure.cpp:440-444)
          Stage st_rc(this, "recheck");
          Segs &one = one_, &rres = rres_;
          std::vector<double> rr;
          subrange(h, j, j + 1, one);
          check(one, static_cast<int>(n_), rres, rr);
          r = rr[0];
          rc = 1;
          ++st_.rechecks;
          const bool ind = r > tol_;
          note(pl, pm, r, ind);
          log_decision(pl, pm, 0, ind ? 1 : 0, rc, r);
          if (ind) accept(rres, 0, r, one, 0);
          if (ind && gram_) gram_note(pl, pm, r);
          continue;
        }
        const bool ind = r > tol_;
        note(pl, pm, r, ind);
        log_decision(pl, pm, 0, ind ? 1 : 0, rc, r);
        if (ind) accept(res, res_index_[j], r, h, j);  // independent => a pass-2 survivor
        if (ind && gram_) gram_note(pl, pm, r);
      }
      const int64_t g_next = g0 + j;
      pair_from_index(g_next, l, m);
    }
  }

  liecl_b200_ctx* ctx_;
  unsigned q_;
  bool keep_;
  bool gram_;
  double tol_;
  double floor_;
  uint64_t interval_;
  bool record_;
  // Alg. 2 state: A and A^{-1} (ld gcap_), the last check's dense beta / x
  // (n_limit x nseg, ld gld_)
  DevBuf<double2> A_, Ainv_, gb_, gx_;
  DevBuf<double> gs_;
  int64_t gcap_ = 0, gld_ = 0;
  uint64_t since_refresh_ = 0;
  HermInverse inverse_;
  int64_t cap_ = 0, budget_ = 0;
  bool has_deadline_ = false;
  Clock::time_point deadline_{};
  int64_t n_ = 0;
  liecl_b200_stats st_{};
  std::vector<Warning> warns_;
  std::vector<liecl_b200_decision> log_;
  // basis pools: orthonormal tuple V; originals O (Alg. 3, commutator basis)
  std::vector<int64_t> voff_, ooff_;
  DevBuf<int64_t> dvoff_, dooff_;
  DevBuf<K> vkey_, okey_;
  DevBuf<C2> vval_, oval_;
  // index
  psum::Index<K> ix_{};
  uint64_t slots_ = 0, keys_upper_ = 0;
  int64_t entries_ = 0;
  DevBuf<K> skey_;
  DevBuf<int> shead_, stail_, scount_, el_, enext_;
  DevBuf<C2> ev_;
  // batch scratch
  DevBuf<unsigned char> temp_;
  DevBuf<int> marker_flag_, small_, poff_, seg_, flag_, pos_, run_seg_, roff_, keep_flag_, kpos_, boff_;
  DevBuf<long long> cnt_, cpos_, clen_, chpos_, scan_ws_ll_;
  DevBuf<int> scan_ws_;
  DevBuf<unsigned> idx_, is_, is1_;
  DevBuf<K> ks_, rkey_, pk_, bl_;
  DevBuf<unsigned long long> ck_, cks_;  // composite sort keys
  DevBuf<C2> rval_, pv_, bv_;
  DevBuf<double> rmag_, hn_, rn_dev_;
  DevBuf<psum::Chunk> chunks_;
  Segs beta_, lc_, h_, res_, r1_, one_, rres_, rs_;
  std::vector<int> res_index_;
  DevBuf<int> gsrc_;
  // fused check (LIECL_B200_SUMS_FUSED=0 disables it, e.g. to exercise the
  // general merges)
  static constexpr size_t kFusedSmemMax = 220 * 1024;
  // batches of at most this many candidates take the fused single-CTA check
  // (LIECL_B200_SUMS_FUSED_BATCH overrides; larger batches run the merges)
  const int kFusedMaxBatch = [] {
    const char* e = std::getenv("LIECL_B200_SUMS_FUSED_BATCH");
    return e ? std::max(1, std::atoi(e)) : 16;
  }();
  bool fused_ = [] {
    const char* e = std::getenv("LIECL_B200_SUMS_FUSED");
    return !(e && e[0] == '0');
  }();
  bool fused_attr_ = false;
  uint64_t fused_batches_ = 0, fused_fallbacks_ = 0;
  DevBuf<K> fk_;
  DevBuf<C2> fv_;
  DevBuf<int> flen_, fst_;
  DevBuf<double> frn_;
  int depth_ = 0;  // check() recursion (batch splits) takes fresh scratch
  std::vector<std::unique_ptr<Segs>> spill_;
  Segs* new_scratch() {
    spill_.push_back(std::make_unique<Segs>());
    return spill_.back().get();
  }
public:
  // ---- single queries over Pauli sums (the drop-in's project_residual /
  // check_matrix_inversion / linear_combination on the Pauli backend) --------
  // The tuple is loaded into the basis pool + index with its coefficients as
  // given; h is one sum (PauliSum form: unique terms sorted by (z, x)).

  // n sums, terms [off[l], off[l+1]) of (x, z, coef re/im)
  void load_basis(const int64_t* off, const uint64_t* x, const uint64_t* z, const double* coef, int64_t n) {
    if (n_ != 0) throw Error(LIECL_B200_INTERNAL, "load_basis needs an empty engine");
    if (n > cap_) throw Error(LIECL_B200_CAPACITY, "basis larger than the engine capacity");
    Segs all;
    upload(off, x, z, coef, static_cast<int>(n), all);
    std::vector<int> ho(static_cast<size_t>(n) + 1);
    for (int64_t l = 0; l <= n; ++l) ho[l] = static_cast<int>(off[l] - off[0]);
    for (int64_t l = 0; l < n; ++l) {
      append_pool(all.key.p + ho[l], all.val.p + ho[l], ho[l + 1] - ho[l], 0.0);
      ++n_;  // element l of the pool (index entries carry l)
    }
  }

  // project_residual (R:src/closure.cpp:142-162) of h against the loaded
  // tuple: residual after two passes -> out, first-pass coefficients
  // beta_l = <V_l, h> -> coeffs (n complex; 0 where no string is shared)
  void project_one(const int64_t nterms, const uint64_t* x, const uint64_t* z, const double* coef, Segs& out,
                   double* coeffs) {
    Segs h;
    const int64_t off[2] = {0, nterms};
    upload(off, x, z, coef, 1, h);
    std::fill(coeffs, coeffs + 2 * n_, 0.0);
    if (n_ == 0) {
      copy_segs(h, out);
      return;
    }
    Segs r1;
    if (!pass(h, static_cast<int>(n_), r1)) throw Error(LIECL_B200_CAPACITY, "one projection exceeds 2^30 terms");
    beta_to_host(coeffs);
    if (!pass(r1, static_cast<int>(n_), out)) throw Error(LIECL_B200_CAPACITY, "one projection exceeds 2^30 terms");
  }

  // beta_l = <V_l, h> for the loaded tuple (inner_product, R:src/operator.cpp:66-75)
  void overlaps_one(const int64_t nterms, const uint64_t* x, const uint64_t* z, const double* coef, double* beta) {
    Segs h, r1;
    const int64_t off[2] = {0, nterms};
    upload(off, x, z, coef, 1, h);
    std::fill(beta, beta + 2 * n_, 0.0);
    if (n_ == 0) return;
    if (!pass(h, static_cast<int>(n_), r1)) throw Error(LIECL_B200_CAPACITY, "one projection exceeds 2^30 terms");
    beta_to_host(beta);
  }

  // linear_combination (R:src/operator.cpp:164-181): from_terms(base_coeff * h
  // ++ coeffs[l] * V_l for l ascending); zero coefficients add only signed
  // zeros, which never change a slot that starts at +0, so they are skipped
  void combine_one(const int64_t nterms, const uint64_t* x, const uint64_t* z, const double* coef, double base_re,
                   double base_im, const double* coeffs, bool negate, Segs& out) {
    Segs h;
    const int64_t off[2] = {0, nterms};
    upload(off, x, z, coef, 1, h);
    std::vector<K> lk;
    std::vector<C2> lv;
    for (int64_t l = 0; l < n_; ++l)
      if (coeffs[2 * l] != 0.0 || coeffs[2 * l + 1] != 0.0) {
        lk.push_back(psum::kfrom_index<K>(l));
        lv.push_back({coeffs[2 * l], coeffs[2 * l + 1]});
      }
    beta_.shape(1, static_cast<int>(lk.size()));
    const int bo[2] = {0, static_cast<int>(lk.size())};
    CU(cudaMemcpyAsync(beta_.off.p, bo, sizeof bo, cudaMemcpyHostToDevice, ctx_->stream));
    if (!lk.empty()) {
      CU(cudaMemcpyAsync(beta_.key.p, lk.data(), lk.size() * sizeof(K), cudaMemcpyHostToDevice,
                         ctx_->stream));
      CU(cudaMemcpyAsync(beta_.val.p, lv.data(), lv.size() * sizeof(C2), cudaMemcpyHostToDevice, ctx_->stream));
    }
    need(run_seg_, std::max<size_t>(lk.size(), 1));
    CU(cudaMemsetAsync(run_seg_.p, 0, std::max<size_t>(lk.size(), 1) * sizeof(int), ctx_->stream));
    if (!combine(h, C2{base_re, base_im}, negate, out))
      throw Error(LIECL_B200_CAPACITY, "linear combination exceeds 2^30 terms");
    CU(cudaStreamSynchronize(ctx_->stream));  // host staging vectors above
  }

  // PauliSum::from_terms (R:src/pauli.cpp:78-115) of n raw terms (any order,
  // duplicates merged in input order from +0, drop rule, sorted by (z, x))
  void from_terms_one(int64_t n, const uint64_t* x, const uint64_t* z, const double* coef, Segs& out) {
    if (n > kMaxItems) throw Error(LIECL_B200_CAPACITY, "terms exceed 2^30");
    const uint64_t kmask = (q_ >= 64) ? ~0ull : ((1ull << q_) - 1);
    std::vector<K> hk(static_cast<size_t>(std::max<int64_t>(n, 1)));
    for (int64_t t = 0; t < n; ++t) {
      if ((x[t] & ~kmask) || (z[t] & ~kmask)) throw Error(LIECL_B200_INVALID_INPUT, "string mask exceeds qubits");
      hk[t] = psum::kpack<K>(x[t], z[t]);
      refuse_marker(hk[t]);
    }
    Segs raw;
    raw.shape(1, static_cast<int>(n));
    const int o[2] = {0, static_cast<int>(n)};
    CU(cudaMemcpyAsync(raw.off.p, o, sizeof o, cudaMemcpyHostToDevice, ctx_->stream));
    if (n > 0) {
      CU(cudaMemcpyAsync(raw.key.p, hk.data(), n * sizeof(K), cudaMemcpyHostToDevice, ctx_->stream));
      CU(cudaMemcpyAsync(raw.val.p, coef, n * sizeof(C2), cudaMemcpyHostToDevice, ctx_->stream));
    }
    merge(1, raw.off.p, raw.key.p, raw.val.p, static_cast<int>(n), true, out, static_cast<int>(q_),
          2 * static_cast<int>(q_));
    CU(cudaStreamSynchronize(ctx_->stream));  // host staging
  }

  bool is_gram() const { return gram_; }
  // result.gram of an Alg. 2 closure: A and A^{-1}, n x n column-major (host)
  void download_gram(double* a_out, double* ainv_out) {
    if (n_ == 0) return;
    const size_t pitch = static_cast<size_t>(gcap_) * sizeof(double2), w = static_cast<size_t>(n_) * sizeof(double2);
    if (a_out) CU(cudaMemcpy2DAsync(a_out, w, A_.p, pitch, w, n_, cudaMemcpyDeviceToHost, ctx_->stream));
    if (ainv_out) CU(cudaMemcpy2DAsync(ainv_out, w, Ainv_.p, pitch, w, n_, cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
  }

  // ||h|| of one host sum (norm, R:src/operator.cpp:77-82 -> sum_norm)
  double norm_one(const int64_t nterms, const uint64_t* x, const uint64_t* z, const double* coef) {
    Segs h;
    const int64_t off[2] = {0, nterms};
    upload(off, x, z, coef, 1, h);
    return norm_of(h);
  }

  // ||sum|| of segment 0 (sum_norm, R:src/pauli.cpp:202-228)
  double norm_of(const Segs& a) {
    need(rn_dev_, 1);
    psum::seg_norm_kernel<<<1, 1, 0, ctx_->stream>>>(a.off.p, 1, a.val.p, rn_dev_.p);
    launched(ctx_);
    double v = 0.0;
    CU(cudaMemcpyAsync(&v, rn_dev_.p, sizeof v, cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
    return v;
  }
  // segment 0 of `a` -> host (x, z, coef); returns the term count (writes
  // nothing when it exceeds cap)
  int64_t download_one(const Segs& a, uint64_t* x, uint64_t* z, double* coef, int64_t cap) {
    const int64_t nt = a.total;
    if (nt > cap || nt == 0) return nt;
    std::vector<K> k(static_cast<size_t>(nt));
    CU(cudaMemcpyAsync(k.data(), a.key.p, nt * sizeof(K), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaMemcpyAsync(coef, a.val.p, nt * sizeof(C2), cudaMemcpyDeviceToHost, ctx_->stream));
    CU(cudaStreamSynchronize(ctx_->stream));
    for (int64_t t = 0; t < nt; ++t) {
      x[t] = psum::kx(k[t]);
      z[t] = psum::kz(k[t]);
    }
    return nt;
  }

};

using SumEngine = SumEngineT<unsigned long long>;      // 1..31 qubits
using SumEngineWide = SumEngineT<psum::WKey>;          // 32..63 qubits
