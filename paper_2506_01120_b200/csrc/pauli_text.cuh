// Pauli-sum text input (R:src/pauli.cpp:230-395, the grammar of
// parse_pauli_sum): host-side tokenizer for the C-ABI. Included by engine.cu
// inside its anonymous namespace (Error). The terms it yields are merged by
// PauliSum::from_terms on the device (SumEngine::from_terms_one).
//
//   sum    := term ( ws* ('+' | '-') ws* term )*        (leading ws allowed)
//   term   := coeff ws+ word
//   coeff  := real | '(' ws* real ws* ',' ws* real ws* ')'
//   real   := [+-]? [0-9.]* ([eE] [+-]? [0-9]*)?  (one std::from_chars double)
//   word   := exactly `qubits` letters of I X Y Z, letter j on qubit j
//
// A malformed text is a ParseError at 1-based (line, column) of the offending
// character; the messages are the reference's.

struct PauliTextError {
  std::string msg;
  int64_t line, col;
};

struct PauliTerm {
  uint64_t x, z;
  double re, im;
};

class PauliTextReader {
public:
  PauliTextReader(const char* text, size_t len, uint32_t qubits) : s_(text), n_(len), q_(qubits) {}

  std::vector<PauliTerm> terms() {
    std::vector<PauliTerm> out;
    blanks();
    if (done()) fail("empty operator expression");
    out.push_back(term(1.0));
    for (blanks(); !done(); blanks()) {
      const char c = cur();
      if (c != '+' && c != '-') fail("expected '+' or '-' between terms");
      step();
      blanks();
      out.push_back(term(c == '-' ? -1.0 : 1.0));
    }
    return out;
  }

private:
  static bool blank(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n'; }
  bool done() const { return i_ >= n_; }
  char cur() const { return s_[i_]; }
  void step() {
    if (s_[i_] == '\n') {
      ++line_;
      col_ = 1;
    } else {
      ++col_;
    }
    ++i_;
  }
  void blanks() {
    while (!done() && blank(cur())) step();
  }
  [[noreturn]] void fail(const std::string& m) const { throw PauliTextError{m, line_, col_}; }
  void want(char c) {
    if (done() || cur() != c) fail(std::string("expected '") + c + "'");
    step();
  }

  PauliTerm term(double sign) {
    double re, im = 0.0;
    if (!done() && cur() == '(') {
      step();
      blanks();
      re = number();
      blanks();
      want(',');
      blanks();
      im = number();
      blanks();
      want(')');
    } else {
      re = number();
    }
    if (!done() && !blank(cur())) fail("expected whitespace between coefficient and Pauli word");
    blanks();
    PauliTerm t = word();
    t.re = sign * re;  // double * Complex: each component scaled
    t.im = sign * im;
    return t;
  }

  double number() {
    const size_t a = i_;
    auto digits = [&] {
      while (!done() && (std::isdigit(static_cast<unsigned char>(cur())) || cur() == '.')) step();
    };
    if (!done() && (cur() == '+' || cur() == '-')) step();
    digits();
    if (!done() && (cur() == 'e' || cur() == 'E')) {
      step();
      if (!done() && (cur() == '+' || cur() == '-')) step();
      while (!done() && std::isdigit(static_cast<unsigned char>(cur()))) step();
    }
    double v = 0.0;
    const auto r = std::from_chars(s_ + a, s_ + i_, v);
    // reported where scanning stopped (the reference rewinds its cursor but not its line / column)
    if (i_ == a || r.ec != std::errc{} || r.ptr != s_ + i_) fail("malformed real number");
    return v;
  }

  PauliTerm word() {
    if (done()) fail("expected Pauli word");
    PauliTerm t{0, 0, 0.0, 0.0};
    uint32_t j = 0;
    for (; !done() && !blank(cur()) && cur() != '+' && cur() != '-'; step(), ++j) {
      if (j >= q_) fail("Pauli word longer than " + std::to_string(q_) + " qubits");
      const uint64_t bit = uint64_t(1) << j;
      switch (cur()) {
      case 'I': break;
      case 'X': t.x |= bit; break;
      case 'Z': t.z |= bit; break;
      case 'Y': t.x |= bit, t.z |= bit; break;
      default: fail(std::string("invalid Pauli letter '") + cur() + "'");
      }
    }
    if (j != q_) fail("Pauli word has " + std::to_string(j) + " letters, expected " + std::to_string(q_));
    return t;
  }

  const char* s_;
  size_t n_;
  uint32_t q_;
  size_t i_ = 0;
  int64_t line_ = 1, col_ = 1;
};

// ---- the generator catalog (R:src/generators.cpp:9-110, 132-148) -----------
// Term lists only (strings and real coefficients, in the reference's order);
// the sums are merged by from_terms and expanded by from_pauli on the device.
// SplitMix64 and uniform_symmetric as R:include/liecl/rng.hpp:20-39.
struct CatalogRng {
  uint64_t state;
  uint64_t next() {
    uint64_t z = (state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double symmetric() { return 2.0 * (static_cast<double>(next() >> 11) * 0x1.0p-53) - 1.0; }
};

// family: 0 hea, 1 spin_glass_hva, 2 xxz_hva, 3 tfim_hva_open (liecl::AnsatzFamily)
inline std::vector<std::vector<PauliTerm>> catalog_terms(int family, uint32_t n, uint64_t seed, double delta) {
  static const char* names[] = {"hea", "spin_glass_hva", "xxz_hva", "tfim_hva_open"};
  if (family < 0 || family > 3) throw Error(LIECL_B200_INVALID_INPUT, "build_generators: unknown family");
  if (n < 2) throw Error(LIECL_B200_INVALID_INPUT, std::string(names[family]) + " requires at least 2 qubits");
  if (family == 2 && n % 2 != 0)
    throw Error(LIECL_B200_INVALID_INPUT, std::string(names[family]) + " requires an even qubit count");
  if (n > 64) throw Error(LIECL_B200_INVALID_INPUT, "qubit count above the 64-qubit mask width");
  auto bit = [](uint32_t q) { return uint64_t(1) << q; };
  std::vector<std::vector<PauliTerm>> g;
  if (family == 0) {  // X_i, Z_i, Z_i Z_{i+1}: one term per generator
    for (uint32_t i = 0; i < n; ++i) g.push_back({{bit(i), 0, 1.0, 0.0}});
    for (uint32_t i = 0; i < n; ++i) g.push_back({{0, bit(i), 1.0, 0.0}});
    for (uint32_t i = 0; i + 1 < n; ++i) g.push_back({{0, bit(i) | bit(i + 1), 1.0, 0.0}});
  } else if (family == 1) {  // a_i Z_i, then J_ij Z_i Z_j (i < j); sum_i X_i
    CatalogRng rng{seed};
    std::vector<PauliTerm> h1, h2;
    for (uint32_t i = 0; i < n; ++i) h1.push_back({0, bit(i), rng.symmetric(), 0.0});
    for (uint32_t i = 0; i < n; ++i)
      for (uint32_t j = i + 1; j < n; ++j) h1.push_back({0, bit(i) | bit(j), rng.symmetric(), 0.0});
    for (uint32_t i = 0; i < n; ++i) h2.push_back({bit(i), 0, 1.0, 0.0});
    g = {h1, h2};
  } else if (family == 2) {  // even / odd bonds of XX + YY + delta ZZ, periodic
    for (uint32_t parity = 0; parity < 2; ++parity) {
      std::vector<PauliTerm> h;
      for (uint32_t i = parity; i < n; i += 2) {
        const uint64_t b = bit(i) | bit((i + 1) % n);
        h.push_back({b, 0, 1.0, 0.0});
        h.push_back({b, b, 1.0, 0.0});
        h.push_back({0, b, delta, 0.0});
      }
      g.push_back(h);
    }
  } else {  // open ZZ chain; sum_i X_i
    std::vector<PauliTerm> h1, h2;
    for (uint32_t i = 0; i + 1 < n; ++i) h1.push_back({0, bit(i) | bit(i + 1), 1.0, 0.0});
    for (uint32_t i = 0; i < n; ++i) h2.push_back({bit(i), 0, 1.0, 0.0});
    g = {h1, h2};
  }
  return g;
}
