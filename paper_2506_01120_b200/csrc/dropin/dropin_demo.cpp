// A liecl consumer linked against the B200 drop-in (closure_b200.cpp in place
// of R:src/closure.cpp): builds configs 0 and 4 with the reference's own
// Pauli/dense API and runs liecl::run_closure. Prints one JSON object; the GPU
// test (tests/test_gpu_dropin.py) compares it with the golden fixtures.
#include <bit>
#include <complex>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "liecl/closure.hpp"
#include "liecl/dense.hpp"
#include "liecl/errors.hpp"
#include "liecl/generators.hpp"
#include "liecl/pauli.hpp"

#ifndef LIECL_DROPIN_SRC_SHA
#define LIECL_DROPIN_SRC_SHA "unknown"
#endif

using namespace liecl;

static void print_stats(const ClosureResult& r) {
  std::printf("{\"dimension\": %zu, \"commutators_evaluated\": %llu, \"independence_checks\": %llu, "
              "\"accepted\": %llu, \"warnings\": %zu",
              r.dimension, static_cast<unsigned long long>(r.stats.commutators_evaluated),
              static_cast<unsigned long long>(r.stats.independence_checks),
              static_cast<unsigned long long>(r.stats.accepted), r.stats.warnings.size());
}

int main() {
  const Complex I{0.0, 1.0};
  ClosureConfig cfg;
  cfg.tolerance = 1e-10;
  std::printf("{");
  // config 0 (dense): i*(X0+X1+X2), i*(Z0Z1+Z1Z2)
  {
    const std::uint32_t n = 3;
    std::vector<PauliSum::Term> t0, t1;
    for (std::uint32_t j = 0; j < n; ++j) t0.push_back({PauliString{1ull << j, 0, n}, I});
    for (std::uint32_t j = 0; j + 1 < n; ++j) t1.push_back({PauliString{0, (1ull << j) | (1ull << (j + 1)), n}, I});
    const std::vector<Operator> gens{Operator(from_pauli(PauliSum::from_terms(n, t0))),
                                     Operator(from_pauli(PauliSum::from_terms(n, t1)))};
    for (const Method m : {Method::orthonorm_dimonly, Method::orthonorm, Method::standard_rank}) {
      const ClosureResult r = run_closure(gens, m, cfg);
      std::printf("\"c0_%s\": ", to_string(m).c_str());
      print_stats(r);
      std::printf(", \"basis\": [");
      for (size_t k = 0; k < r.basis.size(); ++k) {
        const auto& mat = r.basis[k].dense().matrix();
        std::printf("%s[", k ? "," : "");
        for (Eigen::Index e = 0; e < mat.size(); ++e)
          std::printf("%s%.17g,%.17g", e ? "," : "", mat(e).real(), mat(e).imag());
        std::printf("]");
      }
      std::printf("]}, ");
    }
    // Alg. 2 through the same entry point, with the Gram state
    const ClosureResult r = run_closure(gens, Method::matrix_inversion, cfg);
    std::printf("\"c0_matrix-inversion\": ");
    print_stats(r);
    std::printf(", \"gram_size\": %td, \"inverse_error\": %.3g}, ", static_cast<std::ptrdiff_t>(r.gram->size()),
                r.gram->inverse_error());
  }
  // config 4 (Pauli): n=10 ring, i*XX, i*YY, i*Z single strings
  {
    const std::uint32_t n = 10;
    std::vector<Operator> gens;
    for (std::uint32_t j = 0; j < n; ++j) {
      const std::uint64_t b = (1ull << j) | (1ull << ((j + 1) % n));
      gens.emplace_back(PauliSum::single(PauliString{b, 0, n}, I));
    }
    for (std::uint32_t j = 0; j < n; ++j) {
      const std::uint64_t b = (1ull << j) | (1ull << ((j + 1) % n));
      gens.emplace_back(PauliSum::single(PauliString{b, b, n}, I));
    }
    for (std::uint32_t j = 0; j < n; ++j) gens.emplace_back(PauliSum::single(PauliString{0, 1ull << j, n}, I));
    const ClosureResult r = run_closure(gens, Method::orthonorm_dimonly, cfg);
    std::printf("\"c4\": ");
    print_stats(r);
    std::printf(", \"strings\": [");
    for (size_t k = 0; k < r.basis.size(); ++k) {
      const auto& t = r.basis[k].pauli().terms()[0];
      std::printf("%s[%llu,%llu,%.17g,%.17g]", k ? "," : "", static_cast<unsigned long long>(t.string.x),
                  static_cast<unsigned long long>(t.string.z), t.coefficient.real(), t.coefficient.imag());
    }
    std::printf("]}, ");
  }
  // past 32 qubits (128-bit string keys): config 4's ring and the reference's
  // TFIM-open n = 4 generators relabelled onto 48 qubits (the reference's
  // default cap d^2 overflows there, so max_dim is explicit, as a caller must)
  {
    const std::uint32_t q = 48;
    const std::uint32_t ring[10] = {0, 5, 11, 17, 23, 29, 35, 41, 44, 47};
    auto relabel = [](std::uint64_t m, const std::uint32_t* pos, int n) {
      std::uint64_t out = 0;
      for (int j = 0; j < n; ++j)
        if ((m >> j) & 1u) out |= 1ull << pos[j];
      return out;
    };
    ClosureConfig wide = cfg;
    wide.max_dim = 4096;
    std::vector<Operator> gens;
    for (std::uint32_t j = 0; j < 10; ++j) {
      const std::uint64_t b = relabel((1ull << j) | (1ull << ((j + 1) % 10)), ring, 10);
      gens.emplace_back(PauliSum::single(PauliString{b, 0, q}, I));
    }
    for (std::uint32_t j = 0; j < 10; ++j) {
      const std::uint64_t b = relabel((1ull << j) | (1ull << ((j + 1) % 10)), ring, 10);
      gens.emplace_back(PauliSum::single(PauliString{b, b, q}, I));
    }
    for (std::uint32_t j = 0; j < 10; ++j) gens.emplace_back(PauliSum::single(PauliString{0, 1ull << ring[j], q}, I));
    const ClosureResult r = run_closure(gens, Method::orthonorm_dimonly, wide);
    std::printf("\"c4_q48\": ");
    print_stats(r);
    std::printf(", \"strings\": [");
    for (size_t k = 0; k < r.basis.size(); ++k) {
      const auto& t = r.basis[k].pauli().terms()[0];
      std::printf("%s[\"%llu\",\"%llu\",%.17g,%.17g]", k ? "," : "", static_cast<unsigned long long>(t.string.x),
                  static_cast<unsigned long long>(t.string.z), t.coefficient.real(), t.coefficient.imag());
    }
    std::printf("]}, ");
    AnsatzSpec spec;
    spec.family = AnsatzFamily::tfim_hva_open;
    spec.qubits = 4;
    const std::uint32_t tf[4] = {3, 31, 40, 47};
    std::vector<Operator> sums;
    for (auto& s : build_generators(spec)) {
      std::vector<PauliSum::Term> terms;
      for (const auto& t : s.terms())
        terms.push_back({PauliString{relabel(t.string.x, tf, 4), relabel(t.string.z, tf, 4), q}, t.coefficient});
      sums.emplace_back(PauliSum::from_terms(q, terms));
    }
    const ClosureResult rs = run_closure(sums, Method::orthonorm_dimonly, wide);
    std::printf("\"tfim4_q48\": ");
    print_stats(rs);
    std::printf(", \"sums\": [");
    for (size_t k = 0; k < rs.basis.size(); ++k) {
      std::printf("%s[", k ? "," : "");
      const auto terms = rs.basis[k].pauli().terms();
      for (size_t i = 0; i < terms.size(); ++i)
        std::printf("%s[\"%llu\",\"%llu\",%.17g,%.17g]", i ? "," : "",
                    static_cast<unsigned long long>(terms[i].string.x), static_cast<unsigned long long>(terms[i].string.z),
                    terms[i].coefficient.real(), terms[i].coefficient.imag());
      std::printf("]");
    }
    std::printf("]}, ");
  }
  // multi-term Pauli sums: the reference's TFIM-open HVA generators, n = 6
  for (const Method m : {Method::orthonorm_dimonly, Method::orthonorm}) {
    AnsatzSpec spec;
    spec.family = AnsatzFamily::tfim_hva_open;
    spec.qubits = 6;
    std::vector<Operator> gens;
    for (auto& s : build_generators(spec)) gens.emplace_back(std::move(s));
    const ClosureResult r = run_closure(gens, m, cfg);
    std::printf("\"tfim6_%s\": ", to_string(m).c_str());
    print_stats(r);
    std::printf(", \"sums\": [");
    for (size_t k = 0; k < r.basis.size(); ++k) {
      std::printf("%s[", k ? "," : "");
      const auto terms = r.basis[k].pauli().terms();
      for (size_t i = 0; i < terms.size(); ++i)
        std::printf("%s[%llu,%llu,%.17g,%.17g]", i ? "," : "", static_cast<unsigned long long>(terms[i].string.x),
                    static_cast<unsigned long long>(terms[i].string.z), terms[i].coefficient.real(),
                    terms[i].coefficient.imag());
      std::printf("]");
    }
    std::printf("]}, ");
  }
  // project_residual and the error mapping
  {
    std::vector<PauliSum::Term> xs{{PauliString{1, 0, 1}, Complex{1.0, 0.0}}};
    std::vector<PauliSum::Term> zs{{PauliString{0, 1, 1}, Complex{1.0, 0.0}}};
    std::vector<PauliSum::Term> mix{{PauliString{1, 0, 1}, Complex{1.0, 0.0}}, {PauliString{0, 1, 1}, Complex{2.0, 0.0}}};
    const std::vector<Operator> V{Operator(from_pauli(PauliSum::from_terms(1, xs)))};
    const auto [r, c] = project_residual(V, Operator(from_pauli(PauliSum::from_terms(1, mix))));
    const Operator zexp(from_pauli(PauliSum::from_terms(1, zs)));
    const auto diff = r.dense().matrix() - Complex{2.0, 0.0} * zexp.dense().matrix();
    std::printf("\"project_residual\": {\"coeff\": [%.17g, %.17g], \"residual_err\": %.3g}, ", c[0].real(), c[0].imag(),
                diff.norm());
    bool threw = false;
    try {
      ClosureConfig tiny = cfg;
      tiny.max_dim = 2;  // {X, Z} closes to su(2): the third accept must raise
      run_closure(std::vector<Operator>{V[0], zexp}, Method::orthonorm_dimonly, tiny);
    } catch (const CapacityError&) {
      threw = true;
    }
    std::printf("\"capacity_error\": %s, ", threw ? "true" : "false");
  }
  // round 2: what the drop-in used to refuse -- Alg. 2 on Pauli generators
  // (single strings and multi-term sums), project_residual and
  // check_matrix_inversion on Pauli sums, GramState on the caller's state,
  // and a d = 128 dense closure sized from the result (not the d^2 cap)
  {
    AnsatzSpec hea;
    hea.family = AnsatzFamily::hea;
    hea.qubits = 3;
    std::vector<Operator> gens;
    for (auto& g : build_generators(hea)) gens.emplace_back(std::move(g));
    const ClosureResult r = close_matrix_inversion(gens, cfg);
    std::printf("\"hea3_matrix-inversion\": ");
    print_stats(r);
    std::printf(", \"gram_size\": %td, \"inverse_error\": %.3g}, ", static_cast<std::ptrdiff_t>(r.gram->size()),
                r.gram->inverse_error());
    AnsatzSpec tf;
    tf.family = AnsatzFamily::tfim_hva_open;
    tf.qubits = 4;
    std::vector<Operator> sums;
    for (auto& g : build_generators(tf)) sums.emplace_back(std::move(g));
    const ClosureResult rs = close_matrix_inversion(sums, cfg);
    std::printf("\"tfim4_matrix-inversion\": ");
    print_stats(rs);
    std::printf(", \"gram_size\": %td, \"inverse_error\": %.3g, \"sums\": [",
                static_cast<std::ptrdiff_t>(rs.gram->size()), rs.gram->inverse_error());
    for (size_t k = 0; k < rs.basis.size(); ++k) {
      std::printf("%s[", k ? "," : "");
      const auto terms = rs.basis[k].pauli().terms();
      for (size_t i = 0; i < terms.size(); ++i)
        std::printf("%s[%llu,%llu,%.17g,%.17g]", i ? "," : "", static_cast<unsigned long long>(terms[i].string.x),
                    static_cast<unsigned long long>(terms[i].string.z), terms[i].coefficient.real(),
                    terms[i].coefficient.imag());
      std::printf("]");
    }
    std::printf("]}, ");
    // project_residual of a bracket against the first orthonormal elements of the TFIM closure
    const ClosureResult o = close_orthonormalization(sums, cfg, false);
    const std::vector<Operator> V(o.basis.begin(), o.basis.begin() + 6);
    const Operator h = commutator(sums[0], o.basis[7]);
    const auto [res, coeffs] = project_residual(V, h);
    std::printf("\"pauli_project_residual\": {\"terms\": %zu, \"norm_bits\": \"%016llx\", \"coeff0\": [%.17g, %.17g]}, ",
                res.pauli().size(), static_cast<unsigned long long>(std::bit_cast<std::uint64_t>(norm(res))),
                coeffs[0].real(), coeffs[0].imag());
    // check_matrix_inversion with the Alg. 2 state: an accepted element is dependent, a new bracket is not
    const OperatorTuple& B = rs.basis;
    const auto [dep, b1] = check_matrix_inversion(*rs.gram, B, B[2], 1e-10);
    std::printf("\"pauli_check_matrix_inversion\": {\"member_independent\": %s, \"beta2\": [%.17g, %.17g]}, ",
                dep ? "true" : "false", b1[2].real(), b1[2].imag());
    // GramState driven by hand: expand twice, refresh
    GramState gs;
    gs.expand(Eigen::VectorXcd(0), 1e-12);
    Eigen::VectorXcd beta(1);
    beta(0) = Complex{0.5, 0.0};
    const double s = gs.schur_complement(beta);
    gs.expand(beta, 1e-12);
    gs.refresh();
    std::printf("\"gram_state\": {\"schur\": %.17g, \"inv01\": %.17g, \"err\": %.3g}, ", s,
                gs.inverse()(0, 1).real(), gs.inverse_error());
  }
  {
    // d = 128 (7 qubits): X0 and Z0 close to su(2) (dimension 3); the drop-in
    // sizes its output from the result, not from the 16384-element cap
    const std::uint32_t n = 7;
    std::vector<PauliSum::Term> xs{{PauliString{1, 0, n}, I}}, zs{{PauliString{0, 1, n}, I}};
    const std::vector<Operator> gens{Operator(from_pauli(PauliSum::from_terms(n, xs))),
                                     Operator(from_pauli(PauliSum::from_terms(n, zs)))};
    const ClosureResult r = run_closure(gens, Method::orthonorm, cfg);
    std::printf("\"d128\": ");
    print_stats(r);
    std::printf("}, ");
  }
  // concurrent callers (the reference's entry points are reentrant): four
  // threads, each closing config 0 densely and a 6-qubit HEA as Pauli strings;
  // every result must equal the serial one bit for bit
  {
    const std::uint32_t n = 3;
    std::vector<PauliSum::Term> t0, t1;
    for (std::uint32_t j = 0; j < n; ++j) t0.push_back({PauliString{1ull << j, 0, n}, I});
    for (std::uint32_t j = 0; j + 1 < n; ++j) t1.push_back({PauliString{0, (1ull << j) | (1ull << (j + 1)), n}, I});
    const std::vector<Operator> dense{Operator(from_pauli(PauliSum::from_terms(n, t0))),
                                      Operator(from_pauli(PauliSum::from_terms(n, t1)))};
    std::vector<Operator> strings;
    for (std::uint32_t j = 0; j < 6; ++j) {
      const std::vector<PauliSum::Term> x{{PauliString{1ull << j, 0, 6}, Complex{1.0, 0.0}}};
      const std::vector<PauliSum::Term> z{{PauliString{0, 1ull << j, 6}, Complex{1.0, 0.0}}};
      strings.emplace_back(PauliSum::from_terms(6, x));
      strings.emplace_back(PauliSum::from_terms(6, z));
    }
    auto fingerprint = [](const ClosureResult& r) {
      std::vector<double> f{static_cast<double>(r.dimension), static_cast<double>(r.stats.commutators_evaluated)};
      for (const Operator& b : r.basis) {
        if (b.backend() == Backend::dense) {
          const auto& m = b.dense().matrix();
          for (Eigen::Index e = 0; e < m.size(); ++e) f.push_back(m(e).real()), f.push_back(m(e).imag());
        } else {
          for (const auto& t : b.pauli().terms())
            f.push_back(static_cast<double>(t.string.x)), f.push_back(static_cast<double>(t.string.z)),
                f.push_back(t.coefficient.real()), f.push_back(t.coefficient.imag());
        }
      }
      return f;
    };
    const auto want_d = fingerprint(run_closure(dense, Method::orthonorm_dimonly, cfg));
    const auto want_p = fingerprint(run_closure(strings, Method::orthonorm_dimonly, cfg));
    std::vector<int> ok(4, 0);
    std::vector<std::thread> pool;
    for (int t = 0; t < 4; ++t)
      pool.emplace_back([&, t] {
        try {
          bool good = true;
          for (int rep = 0; rep < 3; ++rep) {
            const auto d = fingerprint(run_closure(dense, Method::orthonorm_dimonly, cfg));
            const auto p = fingerprint(run_closure(strings, Method::orthonorm_dimonly, cfg));
            good = good && d.size() == want_d.size() && p.size() == want_p.size() &&
                   std::memcmp(d.data(), want_d.data(), d.size() * sizeof(double)) == 0 &&
                   std::memcmp(p.data(), want_p.data(), p.size() * sizeof(double)) == 0;
          }
          ok[t] = good ? 1 : 0;
        } catch (...) {
          ok[t] = 0;
        }
      });
    for (auto& th : pool) th.join();
    std::printf("\"concurrent_identical\": %s, ", (ok[0] && ok[1] && ok[2] && ok[3]) ? "true" : "false");
  }
  // the sources this binary was built from (tests refuse a stale binary)
  std::printf("\"src_sha\": \"%s\"}\n", LIECL_DROPIN_SRC_SHA);
  return 0;
}
