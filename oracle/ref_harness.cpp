// oracle/_ref harness -- TEST INFRASTRUCTURE ONLY.
//
// Compiled together with the UNMODIFIED liecl reference sources
// (/root/reference/proj/core/src/*.cpp) against the Eigen-subset shim into
// oracle/_ref/libliecl_ref.so (recipe: oracle/Makefile). It exposes the
// reference's own public API through a flat extern "C" surface so the Python
// tests (and bench.py's cpu_baseline / --impl reference leg) can drive it with
// ctypes. Nothing here re-implements reference arithmetic: every number comes
// from liecl::run_closure / project_residual / commutator / norm /
// inner_product / from_pauli / string_product etc.
//
// The one piece of control flow written here is `liecl_ref_decision_log_*`,
// which replays run_engine's cursor loop (R:src/closure.cpp:356-473, incl. the
// speculative rule at :440) through the public operations so that the
// per-candidate verdict sequence -- which run_closure does not expose -- can be
// pinned. Tests assert it reproduces run_closure's basis bit-for-bit.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "liecl/closure.hpp"
#include "liecl/errors.hpp"
#include "liecl/generators.hpp"
#include "liecl/operator.hpp"
#include "liecl/pauli.hpp"
#include "parallel.hpp"

using liecl::Complex;
using liecl::DenseOperator;
using liecl::Operator;
using liecl::OperatorTuple;
using liecl::PauliString;
using liecl::PauliSum;

namespace {

enum Status : int {
  kOk = 0,
  kInvalidInput = 1,
  kCapacity = 2,
  kDegeneracy = 3,
  kTimeout = 4,
  kParse = 5,
  kOther = 9,
};

thread_local std::string g_last_error;

template <class F> int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const liecl::InvalidInputError& e) {
    g_last_error = e.what();
    return kInvalidInput;
  } catch (const liecl::CapacityError& e) {
    g_last_error = e.what();
    return kCapacity;
  } catch (const liecl::DegeneracyError& e) {
    g_last_error = e.what();
    return kDegeneracy;
  } catch (const liecl::TimeoutError& e) {
    g_last_error = e.what();
    return kTimeout;
  } catch (const liecl::ParseError& e) {
    g_last_error = e.what();
    return kParse;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return kOther;
  }
}

Operator dense_from(const double* p, int d) {
  Eigen::MatrixXcd m(d, d);
  std::memcpy(static_cast<void*>(m.data()), p, sizeof(double) * 2 * static_cast<std::size_t>(d) * d);
  return Operator(DenseOperator(std::move(m)));
}

void dense_to(const Operator& op, double* out, int d) {
  const std::size_t n = 2 * static_cast<std::size_t>(d) * d;
  if (op.is_null()) {
    std::memset(out, 0, sizeof(double) * n);
    return;
  }
  std::memcpy(out, op.dense().matrix().data(), sizeof(double) * n);
}

OperatorTuple dense_tuple(const double* p, std::int64_t count, int d) {
  OperatorTuple t;
  t.reserve(static_cast<std::size_t>(count));
  const std::size_t stride = 2 * static_cast<std::size_t>(d) * d;
  for (std::int64_t i = 0; i < count; ++i) t.push_back(dense_from(p + i * stride, d));
  return t;
}

// Pauli sums travel as (offsets[count+1], x[], z[], coef[2*terms]).
OperatorTuple pauli_tuple(const std::int64_t* offsets, const std::uint64_t* x,
                          const std::uint64_t* z, const double* coef, int count,
                          std::uint32_t qubits) {
  OperatorTuple t;
  for (int g = 0; g < count; ++g) {
    std::vector<PauliSum::Term> terms;
    for (std::int64_t k = offsets[g]; k < offsets[g + 1]; ++k)
      terms.push_back({PauliString{x[k], z[k], qubits}, Complex{coef[2 * k], coef[2 * k + 1]}});
    t.emplace_back(PauliSum::from_terms(qubits, terms));
  }
  return t;
}

// Writes a tuple of Pauli sums; returns total terms or -1 if over capacity.
std::int64_t pauli_out(const OperatorTuple& ops, std::int64_t* offsets, std::uint64_t* x,
                       std::uint64_t* z, double* coef, std::int64_t term_cap) {
  std::int64_t k = 0;
  offsets[0] = 0;
  for (std::size_t i = 0; i < ops.size(); ++i) {
    if (!ops[i].is_null()) {
      for (const auto& t : ops[i].pauli().terms()) {
        if (k >= term_cap) return -1;
        x[k] = t.string.x;
        z[k] = t.string.z;
        coef[2 * k] = t.coefficient.real();
        coef[2 * k + 1] = t.coefficient.imag();
        ++k;
      }
    }
    offsets[i + 1] = k;
  }
  return k;
}

double g_rank_tolerance = 0.0;  // ClosureConfig::rank_tolerance for the next calls (test knob)
thread_local std::optional<liecl::GramState> g_last_gram;  // result.gram of the last closure

liecl::ClosureConfig make_config(double tol, unsigned threads, std::uint64_t max_dim) {
  liecl::ClosureConfig cfg;
  cfg.tolerance = tol;
  cfg.rank_tolerance = g_rank_tolerance;
  cfg.threads = threads == 0 ? 1 : threads;
  cfg.max_dim = static_cast<std::size_t>(max_dim);
  return cfg;
}

void write_warnings(const liecl::ClosureStats& st, char* buf, std::int64_t len) {
  if (!buf || len <= 0) return;
  std::string s;
  for (const auto& w : st.warnings) {
    char v[64];
    std::snprintf(v, sizeof v, "%.17g", w.value);
    s += w.kind + "\t" + v + "\t" + w.detail + "\n";
  }
  const std::size_t n = std::min<std::size_t>(s.size(), static_cast<std::size_t>(len - 1));
  std::memcpy(buf, s.data(), n);
  buf[n] = '\0';
}

} // namespace

extern "C" {

void liecl_ref_set_rank_tolerance(double v) { g_rank_tolerance = v; }

struct RefStats {
  std::uint64_t commutators_evaluated;
  std::uint64_t independence_checks;
  std::uint64_t accepted;
  std::uint64_t dimension;
  std::uint64_t warnings;
  double wall_seconds;
};

/// One verdict of the cursor loop.
struct RefDecision {
  std::int64_t l, m;       // m = -1 for the generator loop (l = generator index)
  std::int32_t null_cand;  // commutator (or generator) fell at/below tol
  std::int32_t independent;
  std::int32_t rechecked;  // verdict recomputed against the current basis (:443)
  std::int32_t pad;
  double residual_norm;
};

const char* liecl_ref_last_error() { return g_last_error.c_str(); }
int liecl_ref_abi_version() { return 1; }

// ---- dense closure (R:include/liecl/closure.hpp:125 run_closure) -------------

int liecl_ref_closure_dense(const double* gens, int ngens, int d, int method, double tol,
                            unsigned threads, std::uint64_t max_dim, double* basis_out,
                            double* ortho_out, std::int64_t cap, RefStats* stats,
                            char* warn_buf, std::int64_t warn_len) {
  return guarded([&] {
    const OperatorTuple g = dense_tuple(gens, ngens, d);
    const auto res = liecl::run_closure(g, static_cast<liecl::Method>(method),
                                        make_config(tol, threads, max_dim));
    g_last_gram = res.gram;
    stats->commutators_evaluated = res.stats.commutators_evaluated;
    stats->independence_checks = res.stats.independence_checks;
    stats->accepted = res.stats.accepted;
    stats->dimension = res.dimension;
    stats->warnings = res.stats.warnings.size();
    stats->wall_seconds = res.stats.wall_seconds;
    write_warnings(res.stats, warn_buf, warn_len);
    if (static_cast<std::int64_t>(res.basis.size()) > cap)
      throw liecl::CapacityError("harness: basis output capacity too small");
    const std::size_t stride = 2 * static_cast<std::size_t>(d) * d;
    for (std::size_t i = 0; i < res.basis.size(); ++i) dense_to(res.basis[i], basis_out + i * stride, d);
    if (ortho_out && res.orthonormal_basis) {
      for (std::size_t i = 0; i < res.orthonormal_basis->size(); ++i)
        dense_to((*res.orthonormal_basis)[i], ortho_out + i * stride, d);
    }
  });
}

// ---- Pauli closure ----------------------------------------------------------

int liecl_ref_closure_pauli(const std::int64_t* offsets, const std::uint64_t* x,
                            const std::uint64_t* z, const double* coef, int ngens,
                            unsigned qubits, int method, double tol, unsigned threads,
                            std::uint64_t max_dim, std::int64_t* out_offsets,
                            std::uint64_t* out_x, std::uint64_t* out_z, double* out_coef,
                            std::int64_t term_cap, std::int64_t basis_cap, RefStats* stats,
                            char* warn_buf, std::int64_t warn_len) {
  return guarded([&] {
    const OperatorTuple g = pauli_tuple(offsets, x, z, coef, ngens, qubits);
    const auto res = liecl::run_closure(g, static_cast<liecl::Method>(method),
                                        make_config(tol, threads, max_dim));
    g_last_gram = res.gram;
    stats->commutators_evaluated = res.stats.commutators_evaluated;
    stats->independence_checks = res.stats.independence_checks;
    stats->accepted = res.stats.accepted;
    stats->dimension = res.dimension;
    stats->warnings = res.stats.warnings.size();
    stats->wall_seconds = res.stats.wall_seconds;
    write_warnings(res.stats, warn_buf, warn_len);
    if (static_cast<std::int64_t>(res.basis.size()) > basis_cap)
      throw liecl::CapacityError("harness: basis output capacity too small");
    if (pauli_out(res.basis, out_offsets, out_x, out_z, out_coef, term_cap) < 0)
      throw liecl::CapacityError("harness: term output capacity too small");
  });
}

// ---- cursor-loop replay with a verdict log ----------------------------------
// Follows run_engine (R:src/closure.cpp:356-473) for the orthonormal strategy
// (R:src/closure.cpp:267-310) using only the public operations.

namespace {

struct Outcome {
  bool independent = false;
  double residual_norm = 0.0;
  Operator residual_unit;
};

Outcome ortho_check(const OperatorTuple& v, const Operator& h, double tol) {
  auto [residual, coeffs] = liecl::project_residual(v, h);
  Outcome o;
  o.residual_norm = liecl::norm(residual);
  o.independent = o.residual_norm > tol;
  if (o.independent) o.residual_unit = Complex{1.0 / o.residual_norm, 0.0} * residual;
  return o;
}

struct Replay {
  OperatorTuple ortho, originals;
  std::vector<RefDecision> log;
};

void replay(const OperatorTuple& gens, double tol, bool keep_original, unsigned threads,
            std::uint64_t row_limit, Replay& st) {
  for (std::size_t i = 0; i < gens.size(); ++i) {
    const double gn = liecl::norm(gens[i]);
    RefDecision rec{static_cast<std::int64_t>(i), -1, 0, 0, 0, 0, gn};
    if (gn <= tol) {
      rec.null_cand = 1;
      st.log.push_back(rec);
      continue;
    }
    const Operator gu = Complex{1.0 / gn, 0.0} * gens[i];
    const Outcome o = ortho_check(st.ortho, gu, tol);
    rec.independent = o.independent;
    rec.residual_norm = o.residual_norm;
    st.log.push_back(rec);
    if (o.independent) {
      st.ortho.push_back(o.residual_unit);
      if (keep_original) st.originals.push_back(gu);
    }
  }
  for (std::size_t l = 1; l < (keep_original ? st.originals : st.ortho).size(); ++l) {
    if (row_limit && l >= row_limit) break;
    const OperatorTuple& basis = keep_original ? st.originals : st.ortho;
    std::vector<Operator> cand(l);
    std::vector<char> is_null(l, 1);
    liecl::detail::parallel_for(l, threads, [&](std::size_t m) {
      const Operator h = liecl::commutator(basis[l], basis[m]);
      const double hn = liecl::norm(h);
      if (hn > tol) {
        cand[m] = Complex{1.0 / hn, 0.0} * h;
        is_null[m] = 0;
      }
    });
    std::vector<Outcome> spec(l);
    const std::size_t version = st.ortho.size();
    liecl::detail::parallel_for(l, threads, [&](std::size_t m) {
      if (!is_null[m]) spec[m] = ortho_check(st.ortho, cand[m], tol);
    });
    for (std::size_t m = 0; m < l; ++m) {
      RefDecision rec{static_cast<std::int64_t>(l), static_cast<std::int64_t>(m), 1, 0, 0, 0, 0.0};
      if (is_null[m]) {
        st.log.push_back(rec);
        continue;
      }
      rec.null_cand = 0;
      Outcome o;
      if (st.ortho.size() == version || !spec[m].independent) {
        o = std::move(spec[m]);
      } else {
        o = ortho_check(st.ortho, cand[m], tol);
        rec.rechecked = 1;
      }
      rec.independent = o.independent;
      rec.residual_norm = o.residual_norm;
      st.log.push_back(rec);
      if (o.independent) {
        st.ortho.push_back(o.residual_unit);
        if (keep_original) st.originals.push_back(cand[m]);
      }
    }
  }
}

} // namespace

/// Dense replay. `log` holds up to log_cap records; *log_len receives the
/// total. Outputs the commutator basis (originals or orthonormal) like
/// run_closure's result.basis.
int liecl_ref_decision_log_dense(const double* gens, int ngens, int d, int keep_original,
                                 double tol, unsigned threads, std::uint64_t row_limit,
                                 RefDecision* log, std::int64_t log_cap, std::int64_t* log_len,
                                 double* basis_out, double* ortho_out, std::int64_t cap,
                                 std::int64_t* dim_out) {
  return guarded([&] {
    Replay st;
    replay(dense_tuple(gens, ngens, d), tol, keep_original != 0, threads ? threads : 1,
           row_limit, st);
    *log_len = static_cast<std::int64_t>(st.log.size());
    std::memcpy(log, st.log.data(),
                sizeof(RefDecision) * static_cast<std::size_t>(std::min<std::int64_t>(log_cap, *log_len)));
    const OperatorTuple& b = keep_original ? st.originals : st.ortho;
    *dim_out = static_cast<std::int64_t>(b.size());
    if (*dim_out > cap) throw liecl::CapacityError("harness: basis output capacity too small");
    const std::size_t stride = 2 * static_cast<std::size_t>(d) * d;
    for (std::size_t i = 0; i < b.size(); ++i) {
      if (basis_out) dense_to(b[i], basis_out + i * stride, d);
      if (ortho_out) dense_to(st.ortho[i], ortho_out + i * stride, d);
    }
  });
}

/// Pauli replay, same contract; basis written as term arrays.
int liecl_ref_decision_log_pauli(const std::int64_t* offsets, const std::uint64_t* x,
                                 const std::uint64_t* z, const double* coef, int ngens,
                                 unsigned qubits, int keep_original, double tol,
                                 unsigned threads, RefDecision* log, std::int64_t log_cap,
                                 std::int64_t* log_len, std::int64_t* out_offsets,
                                 std::uint64_t* out_x, std::uint64_t* out_z, double* out_coef,
                                 std::int64_t term_cap, std::int64_t basis_cap,
                                 std::int64_t* dim_out) {
  return guarded([&] {
    Replay st;
    replay(pauli_tuple(offsets, x, z, coef, ngens, qubits), tol, keep_original != 0,
           threads ? threads : 1, 0, st);
    *log_len = static_cast<std::int64_t>(st.log.size());
    std::memcpy(log, st.log.data(),
                sizeof(RefDecision) * static_cast<std::size_t>(std::min<std::int64_t>(log_cap, *log_len)));
    const OperatorTuple& b = keep_original ? st.originals : st.ortho;
    *dim_out = static_cast<std::int64_t>(b.size());
    if (*dim_out > basis_cap) throw liecl::CapacityError("harness: basis output capacity too small");
    if (pauli_out(b, out_offsets, out_x, out_z, out_coef, term_cap) < 0)
      throw liecl::CapacityError("harness: term output capacity too small");
  });
}

// ---- bracket window against a fixed basis (bench --impl reference) ---------
// The body of run_engine's row loop (R:src/closure.cpp:412-460) for rows
// [row_begin, row_end) of the dimension-only orthonormal closure with a
// saturated basis V (no acceptance can occur, so the speculative results are
// the verdicts). Candidates are evaluated with the reference's parallel_for
// over `threads` workers, exactly as run_engine does per row. If max_pairs > 0
// only the first max_pairs cursor pairs of the window are evaluated.

int liecl_ref_bracket_window_dense(const double* basis, std::int64_t n, int d, double tol,
                                   std::int64_t row_begin, std::int64_t row_end,
                                   std::int64_t max_pairs, unsigned threads,
                                   std::int64_t* pairs_done, std::int64_t* nulls,
                                   std::int64_t* independents, double* seconds) {
  return guarded([&] {
    const OperatorTuple v = dense_tuple(basis, n, d);
    const auto t0 = std::chrono::steady_clock::now();
    std::int64_t done = 0, nn = 0, ni = 0;
    for (std::int64_t l = row_begin; l < row_end && l < n; ++l) {
      std::int64_t cnt = l;
      if (max_pairs > 0) cnt = std::min<std::int64_t>(cnt, max_pairs - done);
      if (cnt <= 0) break;
      std::vector<char> is_null(static_cast<std::size_t>(cnt), 1), indep(static_cast<std::size_t>(cnt), 0);
      liecl::detail::parallel_for(static_cast<std::size_t>(cnt), threads ? threads : 1,
                                  [&](std::size_t m) {
        const Operator h = liecl::commutator(v[static_cast<std::size_t>(l)], v[m]);
        const double hn = liecl::norm(h);
        if (hn > tol) {
          is_null[m] = 0;
          indep[m] = ortho_check(v, Complex{1.0 / hn, 0.0} * h, tol).independent;
        }
      });
      for (std::int64_t m = 0; m < cnt; ++m) {
        nn += is_null[static_cast<std::size_t>(m)];
        ni += indep[static_cast<std::size_t>(m)];
      }
      done += cnt;
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *pairs_done = done;
    *nulls = nn;
    *independents = ni;
  });
}

/// Per-pair verdicts of a window of cursor rows against a fixed basis (the
/// saturated phase of run_engine, R:src/closure.cpp:412-460, where nothing is
/// accepted so every row's speculation is final): for each pair (l, m) in
/// order, null flag (||[B_l, B_m]|| <= tol, :419-420), verdict and CGS2
/// residual norm (OrthonormStrategy::check, :276-286). Arrays hold
/// min(max_pairs, window) entries.
int liecl_ref_bracket_window_log_dense(const double* basis, std::int64_t n, int d, double tol,
                                       std::int64_t row_begin, std::int64_t row_end, std::int64_t max_pairs,
                                       unsigned threads, std::int32_t* null_out, std::int32_t* indep_out,
                                       double* rn_out, std::int64_t* pairs_done) {
  return guarded([&] {
    const OperatorTuple v = dense_tuple(basis, n, d);
    std::int64_t done = 0;
    for (std::int64_t l = row_begin; l < row_end && l < n; ++l) {
      std::int64_t cnt = l;
      if (max_pairs > 0) cnt = std::min<std::int64_t>(cnt, max_pairs - done);
      if (cnt <= 0) break;
      const std::int64_t base = done;
      liecl::detail::parallel_for(static_cast<std::size_t>(cnt), threads ? threads : 1, [&](std::size_t m) {
        const Operator h = liecl::commutator(v[static_cast<std::size_t>(l)], v[m]);
        const double hn = liecl::norm(h);
        const std::int64_t k = base + static_cast<std::int64_t>(m);
        null_out[k] = hn > tol ? 0 : 1;
        indep_out[k] = 0;
        rn_out[k] = 0.0;
        if (hn > tol) {
          const Outcome o = ortho_check(v, Complex{1.0 / hn, 0.0} * h, tol);
          indep_out[k] = o.independent;
          rn_out[k] = o.residual_norm;
        }
      });
      done += cnt;
    }
    *pairs_done = done;
  });
}

/// Ordered independence check of unit-normalised candidates against an
/// orthonormal basis (config 3): each candidate is normalised as run_engine
/// does (R:src/closure.cpp:388), checked with project_residual
/// (R:src/closure.cpp:142-162, via the orthonormal strategy :276-286) and,
/// when independent, its residual unit is appended before the next candidate.
/// With `append` = 0 the basis stays fixed and candidates are checked in
/// parallel (threads workers) -- the CPU-baseline timing sample.
int liecl_ref_check_sequence_dense(const double* basis, std::int64_t n, const double* cands,
                                   std::int64_t ncand, int d, double tol, int append,
                                   unsigned threads, std::int32_t* independent,
                                   double* residual_norms, double* seconds) {
  return guarded([&] {
    OperatorTuple v = dense_tuple(basis, n, d);
    const OperatorTuple c = dense_tuple(cands, ncand, d);
    const auto t0 = std::chrono::steady_clock::now();
    if (append) {
      for (std::int64_t k = 0; k < ncand; ++k) {
        const Operator cu = Complex{1.0 / liecl::norm(c[static_cast<std::size_t>(k)]), 0.0} *
                            c[static_cast<std::size_t>(k)];
        const Outcome o = ortho_check(v, cu, tol);
        independent[k] = o.independent;
        residual_norms[k] = o.residual_norm;
        if (o.independent) v.push_back(o.residual_unit);
      }
    } else {
      liecl::detail::parallel_for(static_cast<std::size_t>(ncand), threads ? threads : 1,
                                  [&](std::size_t k) {
        const Operator cu = Complex{1.0 / liecl::norm(c[k]), 0.0} * c[k];
        const Outcome o = ortho_check(v, cu, tol);
        independent[k] = o.independent;
        residual_norms[k] = o.residual_norm;
      });
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

// ---- primitives ----------------------------------------------------------------

int liecl_ref_commutator_dense(const double* a, const double* b, int d, double* out) {
  return guarded([&] { dense_to(liecl::commutator(dense_from(a, d), dense_from(b, d)), out, d); });
}

int liecl_ref_inner_product_dense(const double* a, const double* b, int d, double* out2) {
  return guarded([&] {
    const Complex c = liecl::inner_product(dense_from(a, d), dense_from(b, d));
    out2[0] = c.real();
    out2[1] = c.imag();
  });
}

int liecl_ref_norm_dense(const double* a, int d, double* out) {
  return guarded([&] { *out = liecl::norm(dense_from(a, d)); });
}

int liecl_ref_project_residual_dense(const double* basis, std::int64_t n, const double* h, int d,
                                     double* residual_out, double* coeffs_out) {
  return guarded([&] {
    const OperatorTuple v = dense_tuple(basis, n, d);
    auto [r, coeffs] = liecl::project_residual(v, dense_from(h, d));
    dense_to(r, residual_out, d);
    for (std::size_t l = 0; l < coeffs.size(); ++l) {
      coeffs_out[2 * l] = coeffs[l].real();
      coeffs_out[2 * l + 1] = coeffs[l].imag();
    }
  });
}

int liecl_ref_linear_combination_dense(const double* base, double br, double bi,
                                       const double* tuple, const double* coeffs,
                                       std::int64_t n, int d, double* out) {
  return guarded([&] {
    const OperatorTuple t = dense_tuple(tuple, n, d);
    std::vector<Complex> c(static_cast<std::size_t>(n));
    for (std::int64_t l = 0; l < n; ++l) c[static_cast<std::size_t>(l)] = {coeffs[2 * l], coeffs[2 * l + 1]};
    dense_to(liecl::linear_combination(dense_from(base, d), Complex{br, bi}, t, c), out, d);
  });
}

/// from_pauli (R:src/dense.cpp:70-98) of one Pauli sum.
int liecl_ref_from_pauli(const std::uint64_t* x, const std::uint64_t* z, const double* coef,
                         std::int64_t nterms, unsigned qubits, double* out) {
  return guarded([&] {
    std::vector<PauliSum::Term> terms;
    for (std::int64_t k = 0; k < nterms; ++k)
      terms.push_back({PauliString{x[k], z[k], qubits}, Complex{coef[2 * k], coef[2 * k + 1]}});
    const auto m = liecl::from_pauli(PauliSum::from_terms(qubits, terms));
    dense_to(Operator(m), out, 1 << qubits);
  });
}

/// string_product (R:src/pauli.cpp:61-66) and strings_commute (:68-71).
int liecl_ref_string_product(std::uint64_t px, std::uint64_t pz, std::uint64_t qx,
                             std::uint64_t qz, unsigned qubits, std::uint64_t* rx,
                             std::uint64_t* rz, double* phase2, unsigned* exponent,
                             int* commute) {
  return guarded([&] {
    const PauliString p{px, pz, qubits}, q{qx, qz, qubits};
    const auto [r, ph] = liecl::string_product(p, q);
    *rx = r.x;
    *rz = r.z;
    phase2[0] = ph.real();
    phase2[1] = ph.imag();
    *exponent = liecl::product_phase_exponent(p, q);
    *commute = liecl::strings_commute(p, q) ? 1 : 0;
  });
}

/// sum_commutator (R:src/pauli.cpp:179-200) of two Pauli sums.
int liecl_ref_sum_commutator(const std::int64_t* offsets, const std::uint64_t* x,
                             const std::uint64_t* z, const double* coef, unsigned qubits,
                             std::int64_t* out_offsets, std::uint64_t* out_x,
                             std::uint64_t* out_z, double* out_coef, std::int64_t term_cap) {
  return guarded([&] {
    const OperatorTuple ab = pauli_tuple(offsets, x, z, coef, 2, qubits);
    const OperatorTuple r{liecl::commutator(ab[0], ab[1])};
    if (pauli_out(r, out_offsets, out_x, out_z, out_coef, term_cap) < 0)
      throw liecl::CapacityError("harness: term output capacity too small");
  });
}

/// linear_combination (R:src/operator.cpp:137-182) over Pauli sums: operator 0
/// is the base, 1..n the tuple; is_null[0..n] marks null operators (an empty
/// but non-null sum is a PauliSum with no terms).
int liecl_ref_linear_combination_pauli(const std::int64_t* offsets, const std::uint64_t* x,
                                       const std::uint64_t* z, const double* coef, std::int64_t n,
                                       unsigned qubits, const int* is_null, double br, double bi,
                                       const double* coeffs, std::int64_t* out_offsets, std::uint64_t* out_x,
                                       std::uint64_t* out_z, double* out_coef, std::int64_t term_cap,
                                       int* out_null) {
  return guarded([&] {
    OperatorTuple all = pauli_tuple(offsets, x, z, coef, static_cast<int>(n + 1), qubits);
    for (std::int64_t k = 0; k <= n; ++k)
      if (is_null[k]) all[static_cast<std::size_t>(k)] = Operator{};
    std::vector<Complex> c(static_cast<std::size_t>(n));
    for (std::int64_t l = 0; l < n; ++l) c[static_cast<std::size_t>(l)] = {coeffs[2 * l], coeffs[2 * l + 1]};
    const Operator r = liecl::linear_combination(all[0], Complex{br, bi},
                                                 std::span<const Operator>(all).subspan(1), c);
    *out_null = r.is_null() ? 1 : 0;
    if (pauli_out(OperatorTuple{r}, out_offsets, out_x, out_z, out_coef, term_cap) < 0)
      throw liecl::CapacityError("harness: term output capacity too small");
  });
}

// ---- Alg. 2 pieces: GramState, check_matrix_inversion (R:src/closure.cpp:44-140)

namespace {
// a GramState built like close_matrix_inversion builds it: element k expands
// with beta_l = <B_l, B_k> (l < k)
liecl::GramState gram_of(const OperatorTuple& b, double floor) {
  liecl::GramState st;
  for (std::size_t k = 0; k < b.size(); ++k) {
    Eigen::VectorXcd beta(static_cast<Eigen::Index>(k));
    for (std::size_t l = 0; l < k; ++l) beta(static_cast<Eigen::Index>(l)) = liecl::inner_product(b[l], b[k]);
    st.expand(beta, floor);
  }
  return st;
}
void mat_out(const Eigen::MatrixXcd& m, double* out) {
  std::memcpy(out, m.data(), sizeof(double) * 2 * static_cast<std::size_t>(m.size()));
}
} // namespace

/// GramState through its public API: built from the dense tuple B (n
/// operators) by successive expand calls (schur_complement recorded before
/// each), then A, A^{-1}, refresh()'s inverse and inverse_error().
int liecl_ref_gram_state_dense(const double* basis, std::int64_t n, int d, double floor, double* schur_out,
                               double* gram_out, double* inverse_out, double* refreshed_out, double* err_out) {
  return guarded([&] {
    const OperatorTuple b = dense_tuple(basis, n, d);
    liecl::GramState st;
    for (std::int64_t k = 0; k < n; ++k) {
      Eigen::VectorXcd beta(static_cast<Eigen::Index>(k));
      for (std::int64_t l = 0; l < k; ++l)
        beta(static_cast<Eigen::Index>(l)) =
            liecl::inner_product(b[static_cast<std::size_t>(l)], b[static_cast<std::size_t>(k)]);
      schur_out[k] = st.schur_complement(beta);
      st.expand(beta, floor);
    }
    mat_out(st.gram(), gram_out);
    mat_out(st.inverse(), inverse_out);
    *err_out = st.inverse_error();
    st.refresh();
    mat_out(st.inverse(), refreshed_out);
  });
}

/// check_matrix_inversion(state built from B, B, h, tol), dense or Pauli tuple
int liecl_ref_check_matrix_inversion_dense(const double* basis, std::int64_t n, int d, const double* h, double tol,
                                           double floor, int* independent, double* beta_out) {
  return guarded([&] {
    const OperatorTuple b = dense_tuple(basis, n, d);
    const liecl::GramState st = gram_of(b, floor);
    auto [ind, beta] = liecl::check_matrix_inversion(st, b, dense_from(h, d), tol);
    *independent = ind ? 1 : 0;
    std::memcpy(beta_out, beta.data(), sizeof(double) * 2 * beta.size());
  });
}

int liecl_ref_check_matrix_inversion_pauli(const std::int64_t* offsets, const std::uint64_t* x,
                                           const std::uint64_t* z, const double* coef, std::int64_t n,
                                           unsigned qubits, double tol, double floor, double* gram_out,
                                           double* inverse_out, int* independent, double* beta_out) {
  return guarded([&] {
    const OperatorTuple all = pauli_tuple(offsets, x, z, coef, static_cast<int>(n + 1), qubits);  // B..., h
    const OperatorTuple b(all.begin(), all.begin() + n);
    const liecl::GramState st = gram_of(b, floor);
    mat_out(st.gram(), gram_out);
    mat_out(st.inverse(), inverse_out);
    auto [ind, beta] = liecl::check_matrix_inversion(st, b, all[static_cast<std::size_t>(n)], tol);
    *independent = ind ? 1 : 0;
    std::memcpy(beta_out, beta.data(), sizeof(double) * 2 * beta.size());
  });
}

/// project_residual over Pauli sums: tuple = sums 0..n-1, h = sum n
int liecl_ref_project_residual_pauli(const std::int64_t* offsets, const std::uint64_t* x, const std::uint64_t* z,
                                     const double* coef, std::int64_t n, unsigned qubits, std::int64_t* out_offsets,
                                     std::uint64_t* out_x, std::uint64_t* out_z, double* out_coef,
                                     std::int64_t term_cap, double* coeffs_out) {
  return guarded([&] {
    const OperatorTuple all = pauli_tuple(offsets, x, z, coef, static_cast<int>(n + 1), qubits);
    const OperatorTuple v(all.begin(), all.begin() + n);
    auto [r, coeffs] = liecl::project_residual(v, all[static_cast<std::size_t>(n)]);
    for (std::size_t l = 0; l < coeffs.size(); ++l) {
      coeffs_out[2 * l] = coeffs[l].real();
      coeffs_out[2 * l + 1] = coeffs[l].imag();
    }
    if (pauli_out(OperatorTuple{r}, out_offsets, out_x, out_z, out_coef, term_cap) < 0)
      throw liecl::CapacityError("harness: term output capacity too small");
  });
}

/// result.gram of the last closure run through liecl_ref_closure_* on this thread
int liecl_ref_last_gram(std::int64_t n, double* gram_out, double* inverse_out) {
  return guarded([&] {
    if (!g_last_gram || g_last_gram->size() != n) throw liecl::InvalidInputError("harness: no Gram state of that size");
    mat_out(g_last_gram->gram(), gram_out);
    mat_out(g_last_gram->inverse(), inverse_out);
  });
}

/// parse_pauli_sum (R:src/pauli.cpp:230-395): terms, or the ParseError's
/// message / line / column (status 5)
int liecl_ref_parse_pauli_sum(const char* text, std::int64_t len, unsigned qubits, std::uint64_t* x, std::uint64_t* z,
                              double* coef, std::int64_t cap, std::int64_t* nterms, std::int64_t* line,
                              std::int64_t* col) {
  try {
    const PauliSum s = liecl::parse_pauli_sum(std::string_view(text, static_cast<std::size_t>(len)), qubits);
    std::int64_t offs[2];
    *nterms = pauli_out(OperatorTuple{Operator(s)}, offs, x, z, coef, cap);
    if (*nterms < 0) throw liecl::CapacityError("harness: term output capacity too small");
    return 0;
  } catch (const liecl::ParseError& e) {
    *line = static_cast<std::int64_t>(e.line());
    *col = static_cast<std::int64_t>(e.column());
    g_last_error = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 1;
  }
}

/// Generator catalog (R:src/generators.cpp:132-148) as Pauli term arrays.
int liecl_ref_build_generators(int family, unsigned qubits, std::uint64_t seed, double delta,
                               std::int64_t* out_offsets, std::uint64_t* out_x,
                               std::uint64_t* out_z, double* out_coef, std::int64_t term_cap,
                               std::int64_t* count) {
  return guarded([&] {
    liecl::AnsatzSpec spec;
    spec.family = static_cast<liecl::AnsatzFamily>(family);
    spec.qubits = qubits;
    spec.seed = seed;
    spec.delta = delta;
    OperatorTuple ops;
    for (auto& s : liecl::build_generators(spec)) ops.emplace_back(std::move(s));
    *count = static_cast<std::int64_t>(ops.size());
    if (pauli_out(ops, out_offsets, out_x, out_z, out_coef, term_cap) < 0)
      throw liecl::CapacityError("harness: term output capacity too small");
  });
}

/// realize_generators on the dense backend (R:src/generators.cpp:171-194),
/// with or without the zero-magnetization restriction
int liecl_ref_realize_generators_dense(int family, unsigned qubits, std::uint64_t seed, double delta, int restrict_zm,
                                       double* out, std::int64_t cap, std::int64_t* count, std::int64_t* dim) {
  return guarded([&] {
    liecl::AnsatzSpec spec;
    spec.family = static_cast<liecl::AnsatzFamily>(family);
    spec.qubits = qubits;
    spec.seed = seed;
    spec.delta = delta;
    spec.restrict_zero_magnetization = restrict_zm != 0;
    const OperatorTuple ops = liecl::realize_generators(spec, liecl::Backend::dense);
    *count = static_cast<std::int64_t>(ops.size());
    const int d = static_cast<int>(ops[0].dim());
    *dim = d;
    if (static_cast<std::int64_t>(ops.size()) * 2 * d * d > cap)
      throw liecl::CapacityError("harness: output capacity too small");
    for (std::size_t i = 0; i < ops.size(); ++i) dense_to(ops[i], out + i * 2 * static_cast<std::size_t>(d) * d, d);
  });
}

/// format_pauli_sum / parse round trip helper (R:src/pauli.cpp:390-422).
int liecl_ref_format_pauli(const std::uint64_t* x, const std::uint64_t* z, const double* coef,
                           std::int64_t nterms, unsigned qubits, char* buf, std::int64_t len) {
  return guarded([&] {
    std::vector<PauliSum::Term> terms;
    for (std::int64_t k = 0; k < nterms; ++k)
      terms.push_back({PauliString{x[k], z[k], qubits}, Complex{coef[2 * k], coef[2 * k + 1]}});
    const std::string s = liecl::format_pauli_sum(PauliSum::from_terms(qubits, terms));
    const std::size_t n = std::min<std::size_t>(s.size(), static_cast<std::size_t>(len - 1));
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  });
}

/// format_operator of a dense operator (R:src/operator.cpp:206-226).
int liecl_ref_format_dense(const double* a, int d, char* buf, std::int64_t len) {
  return guarded([&] {
    const std::string s = liecl::format_operator(dense_from(a, d));
    const std::size_t n = std::min<std::size_t>(s.size(), static_cast<std::size_t>(len - 1));
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  });
}

} // extern "C"
