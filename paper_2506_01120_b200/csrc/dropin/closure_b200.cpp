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
//   close_matrix_inversion     (:112-113)  matrix-inversion (dense), with result.gram
//   project_residual           (:139-140)  -> GPU (dense operators)
//   to_string / method_from_string (:22-23), basis_listing (:143)
//   GramState methods, check_matrix_inversion -- host utilities on the
//       caller's own state (the closure builds its state on the GPU)
//   close_standard             (:108-109)  rank method (Alg. 1) -> GPU (dense)
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

ClosureResult close_dense(std::span<const Operator> generators, const ClosureConfig& config, bool keep) {
  Eigen::Index d = 0;
  for (const Operator& g : generators)
    if (!g.is_null()) d = g.dim();
  const size_t D = static_cast<size_t>(d) * d;
  std::vector<double> gens(2 * D * generators.size(), 0.0);
  for (size_t i = 0; i < generators.size(); ++i)
    if (!generators[i].is_null())
      std::memcpy(gens.data() + 2 * D * i, generators[i].dense().matrix().data(), sizeof(double) * 2 * D);
  const size_t cap = config.max_dim ? config.max_dim : D;
  std::vector<double> basis(2 * D * cap), ortho(keep ? 2 * D * cap : 0);
  liecl_b200_stats st{};
  std::vector<char> wbuf(1 << 20);
  const liecl_b200_config cfg = to_native(config);
  check(liecl_b200_closure_dense(context(), gens.data(), static_cast<int32_t>(generators.size()),
                                 static_cast<int32_t>(d), keep ? LIECL_B200_METHOD_ORTHONORM
                                                               : LIECL_B200_METHOD_ORTHONORM_DIMONLY,
                                 &cfg, basis.data(), keep ? ortho.data() : nullptr, static_cast<int64_t>(cap), &st,
                                 wbuf.data(), static_cast<int64_t>(wbuf.size()), nullptr, 0, nullptr));
  auto unpack = [&](const std::vector<double>& src) {
    OperatorTuple t;
    t.reserve(st.dimension);
    for (size_t k = 0; k < st.dimension; ++k) {
      Eigen::MatrixXcd m(d, d);
      std::memcpy(static_cast<void*>(m.data()), src.data() + 2 * D * k, sizeof(double) * 2 * D);
      t.emplace_back(DenseOperator(std::move(m)));
    }
    return t;
  };
  ClosureResult r;
  r.basis = unpack(basis);
  r.orthonormal_basis = keep ? unpack(ortho) : r.basis;
  r.dimension = st.dimension;
  r.method = keep ? Method::orthonorm : Method::orthonorm_dimonly;
  r.backend = Backend::dense;
  r.tolerance = config.tolerance;
  fill_stats(r, st, wbuf);
  return r;
}

// general (multi-term) sums: liecl_b200_closure_pauli_sums, bit-exact
ClosureResult close_pauli_sums(std::span<const Operator> generators, const ClosureConfig& config, bool keep) {
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
    const int s = liecl_b200_closure_pauli_sums(
        context(), off.data(), x.data(), z.data(), c.data(), static_cast<int32_t>(generators.size()), qubits,
        keep ? LIECL_B200_METHOD_ORTHONORM : LIECL_B200_METHOD_ORTHONORM_DIMONLY, &cfg, cap, bo.data(), bx.data(),
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
    r.orthonormal_basis = unpack(oo, ox, oz, ocf);
    r.dimension = st.dimension;
    r.method = keep ? Method::orthonorm : Method::orthonorm_dimonly;
    r.backend = Backend::pauli;
    r.tolerance = config.tolerance;
    fill_stats(r, st, wbuf);
    return r;
  }
}

ClosureResult close_pauli(std::span<const Operator> generators, const ClosureConfig& config, bool keep) {
  for (const Operator& g : generators)
    if (!g.is_null() && g.pauli().size() > 1) return close_pauli_sums(generators, config, keep);
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
  check(liecl_b200_closure_pauli(context(), x.data(), z.data(), c.data(), static_cast<int32_t>(x.size()), qubits,
                                 keep ? LIECL_B200_METHOD_ORTHONORM : LIECL_B200_METHOD_ORTHONORM_DIMONLY, &cfg,
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
  r.orthonormal_basis = unpack(oc);
  r.dimension = st.dimension;
  r.method = keep ? Method::orthonorm : Method::orthonorm_dimonly;
  r.backend = Backend::pauli;
  r.tolerance = config.tolerance;
  fill_stats(r, st, wbuf);
  return r;
}

[[noreturn]] void off_path(const char* what) {
  throw InvalidInputError(std::string(what) +
                          ": not on the B200 hot path (the B200 build serves the orthonormalization methods)");
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

// ---- GramState (R:include/liecl/closure.hpp:28-55): the closure's own state
// is built on the GPU; these host methods serve callers that use GramState
// directly. The device result is installed through refresh() (a member, so it
// may set the private matrices) while a pending state is staged.
namespace {
thread_local const Eigen::MatrixXcd* g_pending_gram = nullptr;
thread_local const Eigen::MatrixXcd* g_pending_inverse = nullptr;
} // namespace

double GramState::schur_complement(const Eigen::VectorXcd& beta) const {
  if (beta.size() != gram_.rows()) throw InvalidInputError("GramState: beta length does not match basis size");
  if (beta.size() == 0) return 1.0;
  const Eigen::VectorXcd u = inverse_ * beta;
  return (Complex{1.0, 0.0} - beta.dot(u)).real();
}

void GramState::expand(const Eigen::VectorXcd& beta, double conditioning_floor) {
  const double s = schur_complement(beta);
  const Eigen::Index n = gram_.rows();
  if (s <= conditioning_floor)
    throw DegeneracyError("Gram expansion is numerically degenerate for element " + std::to_string(n) +
                              " (Schur complement " + std::to_string(s) +
                              "); the element should have been rejected as dependent",
                          static_cast<std::size_t>(n));
  Eigen::MatrixXcd a(n + 1, n + 1), ai(n + 1, n + 1);
  const Eigen::VectorXcd u = n > 0 ? Eigen::VectorXcd(inverse_ * beta) : Eigen::VectorXcd(0);
  for (Eigen::Index k = 0; k < n; ++k) {
    for (Eigen::Index i = 0; i < n; ++i) {
      a(i, k) = gram_(i, k);
      ai(i, k) = inverse_(i, k) + u(i) * std::conj(u(k)) / s;
    }
    a(k, n) = beta(k);
    a(n, k) = std::conj(beta(k));
    ai(k, n) = -u(k) / s;
    ai(n, k) = std::conj(ai(k, n));
  }
  a(n, n) = 1.0;
  ai(n, n) = n == 0 ? 1.0 : 1.0 / s;
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
  inverse_ = gram_.ldlt().solve(Eigen::MatrixXcd::Identity(gram_.rows(), gram_.cols()));
}

double GramState::inverse_error() const {
  if (gram_.rows() == 0) return 0.0;
  return ((gram_ * inverse_) - Eigen::MatrixXcd::Identity(gram_.rows(), gram_.cols())).cwiseAbs().maxCoeff();
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
  const size_t D = static_cast<size_t>(d) * d;
  std::vector<double> gens(2 * D * generators.size(), 0.0);
  for (size_t i = 0; i < generators.size(); ++i)
    if (!generators[i].is_null())
      std::memcpy(gens.data() + 2 * D * i, generators[i].dense().matrix().data(), sizeof(double) * 2 * D);
  const size_t cap = config.max_dim ? config.max_dim : D;
  std::vector<double> basis(2 * D * cap);
  liecl_b200_stats st{};
  std::vector<char> wbuf(1 << 20);
  const liecl_b200_config cfg = to_native(config);
  check(liecl_b200_closure_dense(context(), gens.data(), static_cast<int32_t>(generators.size()),
                                 static_cast<int32_t>(d), LIECL_B200_METHOD_STANDARD_RANK, &cfg, basis.data(), nullptr,
                                 static_cast<int64_t>(cap), &st, wbuf.data(), static_cast<int64_t>(wbuf.size()),
                                 nullptr, 0, nullptr));
  for (size_t k = 0; k < st.dimension; ++k) {
    Eigen::MatrixXcd m(d, d);
    std::memcpy(static_cast<void*>(m.data()), basis.data() + 2 * D * k, sizeof(double) * 2 * D);
    r.basis.emplace_back(DenseOperator(std::move(m)));
  }
  r.dimension = st.dimension;
  fill_stats(r, st, wbuf);
  return r;
}

// Alg. 2 (R:src/closure.cpp:519-527) on the GPU for dense generators
ClosureResult close_matrix_inversion(std::span<const Operator> generators, const ClosureConfig& config) {
  const std::optional<Backend> backend = validate(generators);
  if (backend && *backend != Backend::dense)
    off_path("close_matrix_inversion on Pauli generators");
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
  const size_t D = static_cast<size_t>(d) * d;
  std::vector<double> gens(2 * D * generators.size(), 0.0);
  for (size_t i = 0; i < generators.size(); ++i)
    if (!generators[i].is_null())
      std::memcpy(gens.data() + 2 * D * i, generators[i].dense().matrix().data(), sizeof(double) * 2 * D);
  const size_t cap = config.max_dim ? config.max_dim : D;
  std::vector<double> basis(2 * D * cap), A(2 * cap * cap), Ai(2 * cap * cap);
  liecl_b200_stats st{};
  std::vector<char> wbuf(1 << 20);
  liecl_b200_config cfg = to_native(config);
  cfg.conditioning_floor = config.conditioning_floor;
  cfg.gram_refresh_interval = config.gram_refresh_interval;
  check(liecl_b200_closure_dense_gram(context(), gens.data(), static_cast<int32_t>(generators.size()),
                                      static_cast<int32_t>(d), &cfg, basis.data(), static_cast<int64_t>(cap),
                                      A.data(), Ai.data(), &st, wbuf.data(), static_cast<int64_t>(wbuf.size()),
                                      nullptr, 0, nullptr));
  const Eigen::Index n = static_cast<Eigen::Index>(st.dimension);
  for (Eigen::Index k = 0; k < n; ++k) {
    Eigen::MatrixXcd m(d, d);
    std::memcpy(static_cast<void*>(m.data()), basis.data() + 2 * D * k, sizeof(double) * 2 * D);
    r.basis.emplace_back(DenseOperator(std::move(m)));
  }
  Eigen::MatrixXcd gram(n, n), inverse(n, n);
  std::memcpy(static_cast<void*>(gram.data()), A.data(), sizeof(double) * 2 * n * n);
  std::memcpy(static_cast<void*>(inverse.data()), Ai.data(), sizeof(double) * 2 * n * n);
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

// the single Alg. 2 query (R:src/closure.cpp:135-140): the reference's own
// operations on the caller's host-side state (no GPU batch to amortise)
std::pair<bool, CoefficientVector> check_matrix_inversion(const GramState& state, std::span<const Operator> basis,
                                                          const Operator& h, double tol) {
  if (static_cast<std::size_t>(state.size()) != basis.size())
    throw InvalidInputError("check_matrix_inversion: state size does not match basis size");
  CoefficientVector beta(basis.size());
  for (std::size_t l = 0; l < basis.size(); ++l) beta[l] = inner_product(basis[l], h);
  if (basis.empty()) return {norm(h) > tol, beta};
  const Eigen::VectorXcd x =
      state.inverse() * Eigen::VectorXcd(Eigen::Map<const Eigen::VectorXcd>(beta.data(), static_cast<Eigen::Index>(beta.size())));
  CoefficientVector neg(beta.size());
  for (std::size_t l = 0; l < neg.size(); ++l) neg[l] = -x(static_cast<Eigen::Index>(l));
  return {norm(linear_combination(h, Complex{1.0, 0.0}, basis, neg)) > tol, std::move(beta)};
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
  if (h.is_null() || !h.is_dense())
    off_path("project_residual on non-dense operators");
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
