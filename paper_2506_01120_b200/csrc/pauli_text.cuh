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
