// liecl drop-in: the closure translation unit of liecl, re-implemented on the
// B200 C-ABI (include/liecl_b200.h).
//
// A liecl consumer keeps the reference's headers (liecl/closure.hpp et al.)
// and its pauli / dense / operator / generators translation units, and links
// this file in place of R:src/closure.cpp. Every function declared by
// R:include/liecl/closure.hpp is defined here with the same signature:
//
//   run_closure                (R:include/liecl/closure.hpp:125-126) -> GPU for
//   close_orthonormalization   (:119-121)  orthonorm / orthonorm-dimonly
//   close_matrix_inversion     (:112-113)  matrix-inversion, with result.gram
//                                          (dense, Pauli strings, multi-term sums)
//   project_residual           (:139-140)  -> GPU (dense operators and Pauli sums)
//   check_matrix_inversion     (:132-134)  -> GPU (dense and Pauli)
//   GramState methods          (:28-55)    -> GPU (liecl_b200_gram_*)
//   to_string / method_from_string (:22-23), basis_listing (:143)
//   close_standard             (:108-109)  rank method (Alg. 1) -> GPU (dense)
// No closure arithmetic runs here: results are marshalled into the reference's
// types (PauliSum::from_terms / DenseOperator) and nothing else.
//
// Status codes of the C-ABI map back onto the reference's exception types
// (R:include/liecl/errors.hpp:10-61).
#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "liecl/closure.hpp"
#include "liecl/errors.hpp"
#include "liecl_b200.h"

namespace liecl {

namespace {

[[noreturn]] void raise(int status) {
  const std::string msg = liecl_b200_last_error();
  switch (status) {
  case LIECL_B200_INVALID_INPUT: throw InvalidInputError(msg);
  case LIECL_B200_CAPACITY: throw CapacityError(msg);
  case LIECL_B200_DEGENERACY: throw DegeneracyError(msg, 0);
  case LIECL_B200_TIMEOUT: throw TimeoutError(msg);
  case LIECL_B200_PARSE: throw ParseError(msg, 0, 0);
  default: throw Error("B200 backend: " + msg);
  }
}

void check(int status) {
  if (status != LIECL_B200_OK) raise(status);
}

// One device context per calling thread (stream + workspaces + cached
// engines), created on first use and released at thread exit: the reference's
// entry points are reentrant (R:include/liecl/closure.hpp:94-96), and a
// context serves one caller at a time (include/liecl_b200.h).
struct ThreadContext {
  liecl_b200_ctx* ctx = nullptr;
  int status = LIECL_B200_OK;
  ThreadContext() { status = liecl_b200_ctx_create(0, &ctx); }
  ~ThreadContext() {
    if (ctx) liecl_b200_ctx_destroy(ctx);
  }
};

liecl_b200_ctx* context() {
  thread_local ThreadContext t;
  if (t.status != LIECL_B200_OK) raise(t.status);
  return t.ctx;
}

liecl_b200_config to_native(const ClosureConfig& c) {
  liecl_b200_config n{};
  n.tolerance = c.tolerance;
  n.max_dim = c.max_dim;
  n.threads = c.threads;
  n.record_log = 0;
  n.batch_max = 0;
  n.conditioning_floor = c.conditioning_floor;
  n.gram_refresh_interval = c.gram_refresh_interval;
  n.rank_tolerance = c.rank_tolerance;
  if (c.deadline) {
    const double rel = std::chrono::duration<double>(*c.deadline - std::chrono::steady_clock::now()).count();
    n.deadline_seconds = rel > 0 ? rel : 1e-9;
  }
  return n;
}

// Shared backend of the tuple; nullopt when every generator is null
// (R:src/closure.cpp:476-496).
std::optional<Backend> validate(std::span<const Operator> generators) {
  if (generators.empty()) throw InvalidInputError("closure requires a non-empty generator tuple");
  std::optional<Backend> backend;
  Eigen::Index dim = 0;
  for (const Operator& g : generators) {
    if (g.is_null()) continue;
    if (!backend) {
      backend = g.backend();
      dim = g.dim();
    } else if (g.backend() != *backend || g.dim() != dim) {
      throw InvalidInputError("closure generators must share one backend and dimension");
    }
  }
  return backend;
}

std::vector<WarningRecord> parse_warnings(const std::vector<char>& buf) {
  std::vector<WarningRecord> out;
  const std::string s(buf.data());
  size_t pos = 0;
  while (pos < s.size()) {
    const size_t end = s.find('\n', pos);
    const std::string line = s.substr(pos, end == std::string::npos ? std::string::npos : end - pos);
    pos = end == std::string::npos ? s.size() : end + 1;
    const size_t t1 = line.find('\t'), t2 = line.find('\t', t1 + 1);
    if (t1 == std::string::npos || t2 == std::string::npos) continue;
    out.push_back({line.substr(0, t1), line.substr(t2 + 1), std::stod(line.substr(t1 + 1, t2 - t1 - 1))});
  }
  return out;
}

void fill_stats(ClosureResult& r, const liecl_b200_stats& st, const std::vector<char>& wbuf) {
  r.stats.commutators_evaluated = st.commutators_evaluated;
  r.stats.independence_checks = st.independence_checks;
  r.stats.accepted = st.accepted;
  r.stats.wall_seconds = st.wall_seconds;
  r.stats.warnings = parse_warnings(wbuf);
}

// n result vectors (what 0: result.basis, 1: result.orthonormal_basis) from
// the device-resident result straight into DenseOperators, through a bounded
// staging block: no host buffer is sized by the d^2 cap (R:src/closure.cpp:368-370
// uses d^2 only as a cap)
OperatorTuple fetch_dense(int32_t what, size_t n, Eigen::Index d) {
  OperatorTuple t;
  t.reserve(n);
  const size_t D = static_cast<size_t>(d) * static_cast<size_t>(d);
  const size_t block = std::max<size_t>(1, (size_t{32} << 20) / (16 * D));  // ~32 MB per copy
  std::vector<double> stage(2 * D * std::min(block, std::max<size_t>(n, 1)));
  for (size_t k0 = 0; k0 < n; k0 += block) {
    const size_t cnt = std::min(block, n - k0);
    check(liecl_b200_dense_fetch(context(), what, static_cast<int64_t>(k0), static_cast<int64_t>(cnt), stage.data()));
    for (size_t k = 0; k < cnt; ++k) {
      Eigen::MatrixXcd m(d, d);
      std::memcpy(static_cast<void*>(m.data()), stage.data() + 2 * D * k, sizeof(double) * 2 * D);
      t.emplace_back(DenseOperator(std::move(m)));
    }
  }
  return t;
}

std::vector<double> dense_generators(std::span<const Operator> generators, Eigen::Index d) {
  const size_t D = static_cast<size_t>(d) * static_cast<size_t>(d);
  std::vector<double> gens(2 * D * generators.size(), 0.0);
  for (size_t i = 0; i < generators.size(); ++i)
    if (!generators[i].is_null())
      std::memcpy(gens.data() + 2 * D * i, generators[i].dense().matrix().data(), sizeof(double) * 2 * D);
  return gens;
}

ClosureResult close_dense(std::span<const Operator> generators, const ClosureConfig& config, bool keep) {
  Eigen::Index d = 0;
  for (const Operator& g : generators)
    if (!g.is_null()) d = g.dim();
  const std::vector<double> gens = dense_generators(generators, d);
  liecl_b200_stats st{};
  std::vector<char> wbuf(1 << 20);
  const liecl_b200_config cfg = to_native(config);
  check(liecl_b200_closure_dense(context(), gens.data(), static_cast<int32_t>(generators.size()),
                                 static_cast<int32_t>(d), keep ? LIECL_B200_METHOD_ORTHONORM
                                                               : LIECL_B200_METHOD_ORTHONORM_DIMONLY,
                                 &cfg, nullptr, nullptr, 0, &st, wbuf.data(), static_cast<int64_t>(wbuf.size()),
                                 nullptr, 0, nullptr));
  ClosureResult r;
  r.basis = fetch_dense(0, st.dimension, d);
  r.orthonormal_basis = keep ? fetch_dense(1, st.dimension, d) : r.basis;
  r.dimension = st.dimension;
  r.method = keep ? Method::orthonorm : Method::orthonorm_dimonly;
  r.backend = Backend::dense;
  r.tolerance = config.tolerance;
  fill_stats(r, st, wbuf);
  return r;
}

// a device-built Gram state is installed through GramState::refresh() (a
// member, so it may set the private matrices) while it is staged here
thread_local const Eigen::MatrixXcd* g_pending_gram = nullptr;
thread_local const Eigen::MatrixXcd* g_pending_inverse = nullptr;
double* dp(Eigen::MatrixXcd& m) { return reinterpret_cast<double*>(m.data()); }
const double* dp(const Eigen::MatrixXcd& m) { return reinterpret_cast<const double*>(m.data()); }
const double* dp(const Eigen::VectorXcd& v) { return reinterpret_cast<const double*>(v.data()); }

// general (multi-term) sums: liecl_b200_closure_pauli_sums (orthonormal
// methods bit-exact; Alg. 2 with result.gram)
ClosureResult close_pauli_sums(std::span<const Operator> generators, const ClosureConfig& config, Method method) {
  const bool keep = method == Method::orthonorm;
  const bool gram = method == Method::matrix_inversion;
  std::uint32_t qubits = 0;
  std::vector<std::int64_t> off(1, 0);
  std::vector<std::uint64_t> x, z;
  std::vector<double> c;
  for (const Operator& g : generators) {
    if (!g.is_null()) {
      qubits = g.pauli().qubits();
      for (const auto& t : g.pauli().terms()) {
        x.push_back(t.string.x);
        z.push_back(t.string.z);
        c.push_back(t.coefficient.real());
        c.push_back(t.coefficient.imag());
      }
    }
    off.push_back(static_cast<std::int64_t>(x.size()));
  }
  const liecl_b200_config cfg = to_native(config);
  std::int64_t cap = config.max_dim ? static_cast<std::int64_t>(config.max_dim)
                                    : (qubits < 10 ? (std::int64_t{1} << (2 * qubits)) : (std::int64_t{1} << 20));
  std::int64_t tcap = std::max<std::int64_t>(std::int64_t{1} << 16, 8 * static_cast<std::int64_t>(x.size()));
  for (;;) {
    std::vector<std::int64_t> bo(cap + 1), oo(cap + 1), need(2);
    std::vector<std::uint64_t> bx(tcap), bz(tcap), ox(tcap), oz(tcap);
    std::vector<double> bc(2 * tcap), ocf(2 * tcap);
    liecl_b200_stats st{};
    std::vector<char> wbuf(1 << 20);
    const int32_t m = gram ? LIECL_B200_METHOD_MATRIX_INVERSION
                      : keep ? LIECL_B200_METHOD_ORTHONORM
                             : LIECL_B200_METHOD_ORTHONORM_DIMONLY;
    const int s = liecl_b200_closure_pauli_sums(
        context(), off.data(), x.data(), z.data(), c.data(), static_cast<int32_t>(generators.size()), qubits,
        m, &cfg, cap, bo.data(), bx.data(),
        bz.data(), bc.data(), tcap, oo.data(), ox.data(), oz.data(), ocf.data(), tcap, need.data(), &st, wbuf.data(),
        static_cast<std::int64_t>(wbuf.size()), nullptr, 0, nullptr);
    if (s == LIECL_B200_CAPACITY && std::string(liecl_b200_last_error()) == "output buffers too small") {
      // the result stays on the device: fetch it with exact sizes
      tcap = std::max(need[0], need[1]);
      cap = std::max<std::int64_t>(cap, static_cast<std::int64_t>(st.dimension));
      bo.assign(cap + 1, 0), oo.assign(cap + 1, 0);
      bx.assign(tcap, 0), bz.assign(tcap, 0), ox.assign(tcap, 0), oz.assign(tcap, 0);
      bc.assign(2 * tcap, 0.0), ocf.assign(2 * tcap, 0.0);
      check(liecl_b200_pauli_sums_fetch(context(), cap, bo.data(), bx.data(), bz.data(), bc.data(), tcap, oo.data(),
                                        ox.data(), oz.data(), ocf.data(), tcap));
    } else {
      check(s);
    }
    // unique sorted terms without -0 components: from_terms rebuilds the
    // engine's sums value for value
    auto unpack = [&](const std::vector<std::int64_t>& o, const std::vector<std::uint64_t>& xs,
                      const std::vector<std::uint64_t>& zs, const std::vector<double>& cs) {
      OperatorTuple t;
      t.reserve(st.dimension);
      std::vector<PauliSum::Term> terms;
      for (size_t k = 0; k < st.dimension; ++k) {
        terms.clear();
        for (std::int64_t i = o[k]; i < o[k + 1]; ++i)
          terms.push_back({PauliString{xs[i], zs[i], qubits}, Complex{cs[2 * i], cs[2 * i + 1]}});
        t.emplace_back(PauliSum::from_terms(qubits, terms));
      }
      return t;
    };
    ClosureResult r;
    r.basis = unpack(bo, bx, bz, bc);
    if (!gram) r.orthonormal_basis = unpack(oo, ox, oz, ocf);
    r.dimension = st.dimension;
    r.method = method;
    r.backend = Backend::pauli;
    if (gram) {  // the device Gram state (A, A^{-1}) as result.gram
      const Eigen::Index n = static_cast<Eigen::Index>(st.dimension);
      Eigen::MatrixXcd A(n, n), Ai(n, n);
      if (n > 0) check(liecl_b200_pauli_sums_fetch_gram(context(), dp(A), dp(Ai)));
      GramState state;
      g_pending_gram = &A;
      g_pending_inverse = &Ai;
      state.refresh();
      g_pending_gram = g_pending_inverse = nullptr;
      r.gram = std::move(state);
    }
    r.tolerance = config.tolerance;
    fill_stats(r, st, wbuf);
    return r;
  }
}

// single strings (every closure element stays one string); Alg. 2 here keeps
// an identity Gram state (see liecl_b200_closure_pauli)
ClosureResult close_pauli_single(std::span<const Operator> generators, const ClosureConfig& config, Method method) {
  const bool keep = method != Method::orthonorm_dimonly;
  std::uint32_t qubits = 0;
  std::vector<std::uint64_t> x, z;
  std::vector<double> c;
  for (const Operator& g : generators) {
    if (g.is_null() || g.pauli().empty()) {  // null / empty: zero coefficient, skipped as a null generator
      x.push_back(0);
      z.push_back(0);
      c.push_back(0.0);
      c.push_back(0.0);
      continue;
    }
    qubits = g.pauli().qubits();
    const auto& t = g.pauli().terms()[0];
    x.push_back(t.string.x);
    z.push_back(t.string.z);
    c.push_back(t.coefficient.real());
    c.push_back(t.coefficient.imag());
  }
  const size_t cap = config.max_dim ? config.max_dim : (qubits < 12 ? (size_t{1} << (2 * qubits)) : (size_t{1} << 24));
  std::vector<std::uint64_t> bx(cap), bz(cap);
  std::vector<double> bc(2 * cap), oc(2 * cap);
  liecl_b200_stats st{};
  std::vector<char> wbuf(1 << 20);
  const liecl_b200_config cfg = to_native(config);
  const int32_t m = method == Method::matrix_inversion ? LIECL_B200_METHOD_MATRIX_INVERSION
                    : keep                             ? LIECL_B200_METHOD_ORTHONORM
                                                       : LIECL_B200_METHOD_ORTHONORM_DIMONLY;
  check(liecl_b200_closure_pauli(context(), x.data(), z.data(), c.data(), static_cast<int32_t>(x.size()), qubits, m, &cfg,
                                 bx.data(), bz.data(), bc.data(), oc.data(), static_cast<int64_t>(cap), &st,
                                 wbuf.data(), static_cast<int64_t>(wbuf.size()), nullptr, 0, nullptr));
  // the engine hands back the exact coefficient bits of the reference's
  // one-term sums; rebuild the PauliSum values term for term
  auto unpack = [&](const std::vector<double>& coef) {
    OperatorTuple t;
    t.reserve(st.dimension);
    for (size_t k = 0; k < st.dimension; ++k) {
      const PauliSum::Term term{PauliString{bx[k], bz[k], qubits}, Complex{coef[2 * k], coef[2 * k + 1]}};
      t.emplace_back(PauliSum::single(term.string, Complex{1.0, 0.0}) * term.coefficient);
    }
    return t;
  };
  ClosureResult r;
  r.basis = unpack(bc);
  if (method != Method::matrix_inversion) r.orthonormal_basis = unpack(oc);
  r.dimension = st.dimension;
  r.method = method;
  r.backend = Backend::pauli;
  r.tolerance = config.tolerance;
  fill_stats(r, st, wbuf);
  return r;
}

ClosureResult close_pauli(std::span<const Operator> generators, const ClosureConfig& config, bool keep) {
  for (const Operator& g : generators)
    if (!g.is_null() && g.pauli().size() > 1)
      return close_pauli_sums(generators, config, keep ? Method::orthonorm : Method::orthonorm_dimonly);
  return close_pauli_single(generators, config, keep ? Method::orthonorm : Method::orthonorm_dimonly);
}

// the tuple of Pauli sums as (offsets, x, z, coef) arrays (null elements: no terms)
struct PauliTuple {
  std::uint32_t qubits = 0;
  std::vector<std::int64_t> off{0};
  std::vector<std::uint64_t> x, z;
  std::vector<double> c;
  void add(const Operator& op) {
    if (!op.is_null()) {
      qubits = op.pauli().qubits();
      for (const auto& t : op.pauli().terms()) {
        x.push_back(t.string.x);
        z.push_back(t.string.z);
        c.push_back(t.coefficient.real());
        c.push_back(t.coefficient.imag());
      }
    }
    off.push_back(static_cast<std::int64_t>(x.size()));
  }
};

// a device result sum back into a PauliSum (unique sorted terms, exact bits)
Operator pauli_result(std::uint32_t qubits, const std::vector<std::uint64_t>& x, const std::vector<std::uint64_t>& z,
                      const std::vector<double>& c, std::int64_t nt) {
  std::vector<PauliSum::Term> terms;
  terms.reserve(static_cast<size_t>(nt));
  for (std::int64_t t = 0; t < nt; ++t) terms.push_back({PauliString{x[t], z[t], qubits}, Complex{c[2 * t], c[2 * t + 1]}});
  return Operator(PauliSum::from_terms(qubits, terms));
}


} // namespace

std::string to_string(Method method) {
  switch (method) {
  case Method::standard_rank: return "standard-rank";
  case Method::matrix_inversion: return "matrix-inversion";
  case Method::orthonorm: return "orthonorm";
  case Method::orthonorm_dimonly: return "orthonorm-dimonly";
  }
  return "unknown";
}

Method method_from_string(const std::string& name) {
  if (name == "standard-rank") return Method::standard_rank;
  if (name == "matrix-inversion") return Method::matrix_inversion;
  if (name == "orthonorm") return Method::orthonorm;
  if (name == "orthonorm-dimonly") return Method::orthonorm_dimonly;
  throw InvalidInputError("unknown method '" + name +
                          "' (expected standard-rank, matrix-inversion, orthonorm or orthonorm-dimonly)");
}

// ---- GramState (R:include/liecl/closure.hpp:28-55; R:src/closure.cpp:44-105)
// on the device: the member functions ship the caller's n x n matrices to the
// C-ABI's Gram operations (liecl_b200_gram_*). A device-built state
// (close_matrix_inversion) is installed through refresh() (a member, so it may
// set the private matrices) while a pending state is staged.

double GramState::schur_complement(const Eigen::VectorXcd& beta) const {
  if (beta.size() != gram_.rows()) throw InvalidInputError("GramState: beta length does not match basis size");
  double s = 1.0;
  check(liecl_b200_gram_schur_complement(context(), dp(inverse_), beta.size(), dp(beta), &s));
  return s;
}

void GramState::expand(const Eigen::VectorXcd& beta, double conditioning_floor) {
  if (beta.size() != gram_.rows()) throw InvalidInputError("GramState: beta length does not match basis size");
  const Eigen::Index n = gram_.rows();
  Eigen::MatrixXcd a(n + 1, n + 1), ai(n + 1, n + 1);
  const int st = liecl_b200_gram_expand(context(), dp(gram_), dp(inverse_), n, dp(beta), conditioning_floor, dp(a),
                                        dp(ai));
  if (st == LIECL_B200_DEGENERACY)  // the reference's message and element index (R:src/closure.cpp:58-64)
    throw DegeneracyError(liecl_b200_last_error(), static_cast<std::size_t>(n));
  check(st);
  gram_ = std::move(a);
  inverse_ = std::move(ai);
}

void GramState::refresh() {
  if (g_pending_gram) {  // install a device-built state (close_matrix_inversion)
    gram_ = *g_pending_gram;
    inverse_ = *g_pending_inverse;
    return;
  }
  if (gram_.rows() == 0) return;
  Eigen::MatrixXcd ai(gram_.rows(), gram_.cols());
  check(liecl_b200_gram_refresh(context(), dp(gram_), gram_.rows(), dp(ai)));
  inverse_ = std::move(ai);
}

double GramState::inverse_error() const {
  double err = 0.0;
  check(liecl_b200_gram_inverse_error(context(), dp(gram_), dp(inverse_), gram_.rows(), &err));
  return err;
}

// Alg. 1, the rank method (R:src/closure.cpp:500-517) on the GPU: rank of
// [B | vec(h)] from the singular values of the small triangular factor
ClosureResult close_standard(std::span<const Operator> generators, const ClosureConfig& config) {
  const std::optional<Backend> backend = validate(generators);
  if (backend && *backend != Backend::dense)
    throw InvalidInputError("close_standard requires the dense backend; the rank check vectorizes operators");
  Eigen::Index d = 0;
  for (const Operator& g : generators)
    if (!g.is_null()) d = g.dim();
  ClosureResult r;
  r.method = Method::standard_rank;
  r.backend = Backend::dense;
  r.tolerance = config.tolerance;
  if (d == 0) {  // every generator null
    for (size_t i = 0; i < generators.size(); ++i)
      r.stats.warnings.push_back({"null_generator",
                                  "generator " + std::to_string(i) + " has norm " + std::to_string(0.0) +
                                      " and was skipped",
                                  0.0});
    return r;
  }
  const std::vector<double> gens = dense_generators(generators, d);
  liecl_b200_stats st{};
  std::vector<char> wbuf(1 << 20);
  const liecl_b200_config cfg = to_native(config);
  check(liecl_b200_closure_dense(context(), gens.data(), static_cast<int32_t>(generators.size()),
                                 static_cast<int32_t>(d), LIECL_B200_METHOD_STANDARD_RANK, &cfg, nullptr, nullptr, 0,
                                 &st, wbuf.data(), static_cast<int64_t>(wbuf.size()), nullptr, 0, nullptr));
  r.basis = fetch_dense(0, st.dimension, d);
  r.dimension = st.dimension;
  fill_stats(r, st, wbuf);
  return r;
}

// Alg. 2 (R:src/closure.cpp:519-527) on the GPU for dense generators
ClosureResult close_matrix_inversion(std::span<const Operator> generators, const ClosureConfig& config) {
  const std::optional<Backend> backend = validate(generators);
  if (backend && *backend != Backend::dense) {
    bool single = true;
    for (const Operator& g : generators) single = single && (g.is_null() || g.pauli().size() <= 1);
    if (!single) return close_pauli_sums(generators, config, Method::matrix_inversion);
    ClosureResult r = close_pauli_single(generators, config, Method::matrix_inversion);
    // distinct strings: A = I and A^{-1} = I exactly (GramState::expand with beta = 0, s = 1)
    const Eigen::Index n = static_cast<Eigen::Index>(r.dimension);
    const Eigen::MatrixXcd eye = Eigen::MatrixXcd::Identity(n, n);
    GramState state;
    g_pending_gram = &eye;
    g_pending_inverse = &eye;
    state.refresh();
    g_pending_gram = g_pending_inverse = nullptr;
    r.gram = std::move(state);
    return r;
  }
  Eigen::Index d = 0;
  for (const Operator& g : generators)
    if (!g.is_null()) d = g.dim();
  ClosureResult r;
  r.method = Method::matrix_inversion;
  r.backend = Backend::dense;
  r.tolerance = config.tolerance;
  if (d == 0) {
    r.gram = GramState{};
    return r;
  }
  const std::vector<double> gens = dense_generators(generators, d);
  liecl_b200_stats st{};
  std::vector<char> wbuf(1 << 20);
  liecl_b200_config cfg = to_native(config);
  cfg.conditioning_floor = config.conditioning_floor;
  cfg.gram_refresh_interval = config.gram_refresh_interval;
  check(liecl_b200_closure_dense_gram(context(), gens.data(), static_cast<int32_t>(generators.size()),
                                      static_cast<int32_t>(d), &cfg, nullptr, 0, nullptr, nullptr, &st, wbuf.data(),
                                      static_cast<int64_t>(wbuf.size()), nullptr, 0, nullptr));
  const Eigen::Index n = static_cast<Eigen::Index>(st.dimension);
  r.basis = fetch_dense(0, st.dimension, d);
  Eigen::MatrixXcd gram(n, n), inverse(n, n);
  if (n > 0) {
    check(liecl_b200_dense_fetch(context(), 2, 0, n, reinterpret_cast<double*>(gram.data())));
    check(liecl_b200_dense_fetch(context(), 3, 0, n, reinterpret_cast<double*>(inverse.data())));
  }
  GramState state;
  g_pending_gram = &gram;
  g_pending_inverse = &inverse;
  state.refresh();
  g_pending_gram = g_pending_inverse = nullptr;
  r.gram = std::move(state);
  r.dimension = st.dimension;
  fill_stats(r, st, wbuf);
  return r;
}

// the single Alg. 2 query (R:src/closure.cpp:107-140) on the caller's state:
// beta GEMM, x = A^{-1} beta, residual and norm on the device
std::pair<bool, CoefficientVector> check_matrix_inversion(const GramState& state, std::span<const Operator> basis,
                                                          const Operator& h, double tol) {
  if (static_cast<std::size_t>(state.size()) != basis.size())
    throw InvalidInputError("check_matrix_inversion: state size does not match basis size");
  for (const Operator& b : basis)
    if (!b.is_null() && !h.is_null() && (b.backend() != h.backend() || b.dim() != h.dim()))
      throw InvalidInputError("inner_product: operators have mismatched backends or dimensions");
  CoefficientVector beta(basis.size());
  std::int32_t ind = 0;
  const auto* inv = reinterpret_cast<const double*>(state.inverse().data());
  if (h.is_null()) {
    // beta = 0 and the residual is a zero operator (R:src/operator.cpp:66-70, 147-154)
    std::fill(beta.begin(), beta.end(), Complex{0.0, 0.0});
    return {0.0 > tol, std::move(beta)};
  }
  if (h.is_dense()) {
    const Eigen::Index d = h.dim();
    const size_t D = static_cast<size_t>(d) * static_cast<size_t>(d);
    std::vector<double> B(2 * D * basis.size(), 0.0);
    for (size_t l = 0; l < basis.size(); ++l)
      if (!basis[l].is_null()) std::memcpy(B.data() + 2 * D * l, basis[l].dense().matrix().data(), sizeof(double) * 2 * D);
    check(liecl_b200_check_matrix_inversion_dense(context(), B.data(), static_cast<int64_t>(basis.size()), inv,
                                                  reinterpret_cast<const double*>(h.dense().matrix().data()),
                                                  static_cast<int32_t>(d), tol, &ind,
                                                  reinterpret_cast<double*>(beta.data()), nullptr));
  } else {
    PauliTuple t;
    for (const Operator& b : basis) t.add(b);
    PauliTuple hh;
    hh.add(h);
    check(liecl_b200_check_matrix_inversion_pauli(context(), t.off.data(), t.x.data(), t.z.data(), t.c.data(),
                                                  static_cast<int64_t>(basis.size()), h.pauli().qubits(), inv,
                                                  hh.off[1], hh.x.data(), hh.z.data(), hh.c.data(), tol, &ind,
                                                  reinterpret_cast<double*>(beta.data()), nullptr));
  }
  return {ind != 0, std::move(beta)};
}

ClosureResult close_orthonormalization(std::span<const Operator> generators, const ClosureConfig& config,
                                       bool keep_original) {
  const Backend backend = validate(generators).value_or(Backend::pauli);
  bool any = false;
  for (const Operator& g : generators) any = any || !g.is_null();
  if (!any) {  // every generator null: empty closure, one warning each (R:src/closure.cpp:378-387)
    ClosureResult r;
    r.method = keep_original ? Method::orthonorm : Method::orthonorm_dimonly;
    r.backend = backend;
    r.tolerance = config.tolerance;
    r.orthonormal_basis = OperatorTuple{};
    for (size_t i = 0; i < generators.size(); ++i)
      r.stats.warnings.push_back({"null_generator",
                                  "generator " + std::to_string(i) + " has norm " + std::to_string(0.0) +
                                      " and was skipped",
                                  0.0});
    return r;
  }
  return backend == Backend::dense ? close_dense(generators, config, keep_original)
                                   : close_pauli(generators, config, keep_original);
}

ClosureResult run_closure(std::span<const Operator> generators, Method method, const ClosureConfig& config) {
  switch (method) {
  case Method::standard_rank: return close_standard(generators, config);
  case Method::matrix_inversion: return close_matrix_inversion(generators, config);
  case Method::orthonorm: return close_orthonormalization(generators, config, true);
  case Method::orthonorm_dimonly: return close_orthonormalization(generators, config, false);
  }
  throw InvalidInputError("run_closure: unknown method");
}

std::pair<Operator, CoefficientVector> project_residual(std::span<const Operator> orthonormal, const Operator& h) {
  if (orthonormal.empty()) return {h, {}};
  for (const Operator& v : orthonormal)
    if (!v.is_null() && !h.is_null() && (v.backend() != h.backend() || v.dim() != h.dim()))
      throw InvalidInputError("inner_product: operators have mismatched backends or dimensions");
  if (h.is_null()) {
    // every coefficient is <V_l, null> = 0 and the residual is the chained sum
    // null + 0 * V_0 + ... (R:src/operator.cpp:147-154): a zero operator of V's backend
    CoefficientVector zeros(orthonormal.size(), Complex{0.0, 0.0});
    for (const Operator& v : orthonormal)
      if (!v.is_null())
        return {v.is_dense() ? Operator(DenseOperator(Eigen::MatrixXcd::Zero(v.dim(), v.dim())))
                             : Operator(PauliSum::from_terms(v.pauli().qubits(), {})),
                std::move(zeros)};
    return {h, std::move(zeros)};
  }
  if (h.is_pauli()) {  // PauliSum backend on the device (SumEngine passes), bit-exact
    PauliTuple t;
    for (const Operator& v : orthonormal) t.add(v);
    PauliTuple hh;
    hh.add(h);
    const std::int64_t bound = hh.off[1] + t.off.back();  // no result has more terms
    std::vector<std::uint64_t> rx(static_cast<size_t>(std::max<std::int64_t>(bound, 1))),
        rz(static_cast<size_t>(std::max<std::int64_t>(bound, 1)));
    std::vector<double> rc(2 * static_cast<size_t>(std::max<std::int64_t>(bound, 1)));
    CoefficientVector coeffs(orthonormal.size());
    std::int64_t nt = 0;
    check(liecl_b200_project_residual_pauli(context(), t.off.data(), t.x.data(), t.z.data(), t.c.data(),
                                            static_cast<int64_t>(orthonormal.size()), h.pauli().qubits(), hh.off[1],
                                            hh.x.data(), hh.z.data(), hh.c.data(), rx.data(), rz.data(), rc.data(),
                                            bound, &nt, reinterpret_cast<double*>(coeffs.data())));
    return {pauli_result(h.pauli().qubits(), rx, rz, rc, nt), std::move(coeffs)};
  }
  const Eigen::Index d = h.dim();
  const size_t D = static_cast<size_t>(d) * d;
  std::vector<double> V(2 * D * orthonormal.size(), 0.0);
  for (size_t l = 0; l < orthonormal.size(); ++l) {
    if (orthonormal[l].is_null()) continue;
    if (!orthonormal[l].is_dense() || orthonormal[l].dim() != d)
      throw InvalidInputError("linear_combination: operators have mismatched backends or dimensions");
    std::memcpy(V.data() + 2 * D * l, orthonormal[l].dense().matrix().data(), sizeof(double) * 2 * D);
  }
  std::vector<double> r(2 * D), coeffs(2 * orthonormal.size());
  check(liecl_b200_project_residual_dense(context(), V.data(), static_cast<int64_t>(orthonormal.size()),
                                          reinterpret_cast<const double*>(h.dense().matrix().data()),
                                          static_cast<int32_t>(d), r.data(), coeffs.data()));
  Eigen::MatrixXcd m(d, d);
  std::memcpy(static_cast<void*>(m.data()), r.data(), sizeof(double) * 2 * D);
  CoefficientVector c(orthonormal.size());
  for (size_t l = 0; l < c.size(); ++l) c[l] = {coeffs[2 * l], coeffs[2 * l + 1]};
  return {Operator(DenseOperator(std::move(m))), std::move(c)};
}

std::string basis_listing(const ClosureResult& result) {
  std::string out;
  for (const Operator& op : result.basis) {
    out += format_operator(op);
    out += '\n';
  }
  return out;
}

} // namespace liecl
