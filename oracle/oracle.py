"""ctypes bindings for the two CPU checkers -- TEST INFRASTRUCTURE ONLY.

* `Ref`    : oracle/_ref/libliecl_ref.so -- the unmodified liecl reference
             sources compiled against the Eigen-subset shim (oracle/Makefile).
* `Port`   : oracle/_build/liecl_oracle.so -- the plain-C restatement
             (oracle/liecl_oracle.c), pinned against `Ref` by
             tests/test_oracle_pin.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this module, and only as the checker or the
timed CPU baseline; the CUDA product path never calls it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libliecl_ref.so")
# the reference's default-ISA rounding (no FMA contraction in any file), see Makefile
REF_EXACT_SO = os.path.join(HERE, "_ref", "libliecl_ref_exact.so")
PORT_SO = os.path.join(HERE, "_build", "liecl_oracle.so")
REF_SOURCES = "/root/reference/proj/core"

METHODS = {"standard-rank": 0, "matrix-inversion": 1, "orthonorm": 2, "orthonorm-dimonly": 3}
FAMILIES = {"hea": 0, "spin_glass_hva": 1, "xxz_hva": 2, "tfim_hva_open": 3}

DP = C.POINTER(C.c_double)
I64P = C.POINTER(C.c_int64)
U64P = C.POINTER(C.c_uint64)
I32P = C.POINTER(C.c_int32)


def build(ref: bool = True) -> None:
    """Compile the restatement (always) and the reference (when its sources exist)."""
    targets = ["port"] + (["ref"] if ref and os.path.isdir(REF_SOURCES) else [])
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


class Stats(C.Structure):
    _fields_ = [("commutators_evaluated", C.c_uint64), ("independence_checks", C.c_uint64),
                ("accepted", C.c_uint64), ("dimension", C.c_uint64), ("extra", C.c_uint64),
                ("wall_seconds", C.c_double)]


class Decision(C.Structure):
    _fields_ = [("l", C.c_int64), ("m", C.c_int64), ("null_cand", C.c_int32),
                ("independent", C.c_int32), ("rechecked", C.c_int32), ("pad", C.c_int32),
                ("residual_norm", C.c_double)]


DECISION_DTYPE = np.dtype([("l", np.int64), ("m", np.int64), ("null_cand", np.int32),
                           ("independent", np.int32), ("rechecked", np.int32), ("pad", np.int32),
                           ("residual_norm", np.float64)])


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"status {status}: {msg}")
        self.status = status


def _p(a, t=DP):
    return a.ctypes.data_as(t) if a is not None else None


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


@dataclass
class ClosureOut:
    dimension: int
    basis: np.ndarray | None
    ortho: np.ndarray | None
    stats: dict
    log: np.ndarray | None = None
    warnings: str = ""


def _stats(s: Stats) -> dict:
    return {"commutators_evaluated": s.commutators_evaluated, "independence_checks": s.independence_checks,
            "accepted": s.accepted, "dimension": s.dimension, "extra": s.extra,
            "wall_seconds": s.wall_seconds}


class Ref:
    """The reference library (real liecl control flow, shim arithmetic)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing; run `make -C oracle ref` where /root/reference exists")
        self.lib = L = C.CDLL(path)
        L.liecl_ref_last_error.restype = C.c_char_p

    def _check(self, status):
        if status != 0:
            raise OracleError(status, self.lib.liecl_ref_last_error().decode())

    # -- closures ------------------------------------------------------------
    def closure_dense(self, gens, d, method="orthonorm-dimonly", tol=1e-10, threads=1, max_dim=0, rank_tol=0.0):
        self.lib.liecl_ref_set_rank_tolerance(C.c_double(rank_tol))
        gens = _c128(gens)
        cap = max_dim or d * d
        basis = np.zeros((cap, d * d), np.complex128)
        ortho = np.zeros((cap, d * d), np.complex128)
        st = Stats()
        wbuf = C.create_string_buffer(1 << 20)
        self._check(self.lib.liecl_ref_closure_dense(
            _p(gens.view(np.float64)), C.c_int(len(gens)), C.c_int(d), C.c_int(METHODS[method]),
            C.c_double(tol), C.c_uint(threads), C.c_uint64(max_dim), _p(basis.view(np.float64)),
            _p(ortho.view(np.float64)), C.c_int64(cap), C.byref(st), wbuf, C.c_int64(len(wbuf))))
        n = st.dimension
        has_ortho = method.startswith("orthonorm")
        return ClosureOut(n, basis[:n].copy(), ortho[:n].copy() if has_ortho else None, _stats(st),
                          warnings=wbuf.value.decode())

    def closure_pauli(self, offsets, x, z, coef, qubits, method="orthonorm-dimonly", tol=1e-10,
                      threads=1, max_dim=0, basis_cap=None, term_cap=None):
        offsets = np.ascontiguousarray(offsets, np.int64)
        x = np.ascontiguousarray(x, np.uint64)
        z = np.ascontiguousarray(z, np.uint64)
        coef = np.ascontiguousarray(coef, np.float64)
        basis_cap = basis_cap or (max_dim or 4 ** qubits)
        term_cap = term_cap or max(basis_cap * 4, 1 << 20)
        oo = np.zeros(basis_cap + 1, np.int64)
        ox = np.zeros(term_cap, np.uint64)
        oz = np.zeros(term_cap, np.uint64)
        oc = np.zeros((term_cap, 2), np.float64)
        st = Stats()
        wbuf = C.create_string_buffer(1 << 20)
        self._check(self.lib.liecl_ref_closure_pauli(
            _p(offsets, I64P), _p(x, U64P), _p(z, U64P), _p(coef), C.c_int(len(offsets) - 1),
            C.c_uint(qubits), C.c_int(METHODS[method]), C.c_double(tol), C.c_uint(threads),
            C.c_uint64(max_dim), _p(oo, I64P), _p(ox, U64P), _p(oz, U64P), _p(oc),
            C.c_int64(term_cap), C.c_int64(basis_cap), C.byref(st), wbuf, C.c_int64(len(wbuf))))
        n = st.dimension
        t = oo[n]
        return ClosureOut(n, (oo[: n + 1].copy(), ox[:t].copy(), oz[:t].copy(), oc[:t].copy()), None,
                          _stats(st), warnings=wbuf.value.decode())

    def decision_log_dense(self, gens, d, keep_original=False, tol=1e-10, threads=1, row_limit=0,
                           log_cap=None):
        gens = _c128(gens)
        cap = d * d
        log_cap = log_cap or (cap * cap // 2 + 64 if row_limit == 0 else row_limit * row_limit + 64)
        log = np.zeros(log_cap, DECISION_DTYPE)
        basis = np.zeros((cap, d * d), np.complex128)
        ortho = np.zeros((cap, d * d), np.complex128)
        nlog = C.c_int64()
        dim = C.c_int64()
        self._check(self.lib.liecl_ref_decision_log_dense(
            _p(gens.view(np.float64)), C.c_int(len(gens)), C.c_int(d), C.c_int(int(keep_original)),
            C.c_double(tol), C.c_uint(threads), C.c_uint64(row_limit), log.ctypes.data_as(C.c_void_p),
            C.c_int64(log_cap), C.byref(nlog), _p(basis.view(np.float64)), _p(ortho.view(np.float64)),
            C.c_int64(cap), C.byref(dim)))
        n = dim.value
        return ClosureOut(n, basis[:n].copy(), ortho[:n].copy(), {}, log[: min(nlog.value, log_cap)].copy())

    def decision_log_pauli(self, offsets, x, z, coef, qubits, keep_original=False, tol=1e-10, threads=1,
                           term_cap=None, basis_cap=None):
        offsets = np.ascontiguousarray(offsets, np.int64)
        x = np.ascontiguousarray(x, np.uint64)
        z = np.ascontiguousarray(z, np.uint64)
        coef = np.ascontiguousarray(coef, np.float64)
        basis_cap = basis_cap or 4 ** qubits
        term_cap = term_cap or max(basis_cap * 4, 1 << 20)
        log_cap = 1 << 22
        log = np.zeros(log_cap, DECISION_DTYPE)
        oo = np.zeros(basis_cap + 1, np.int64)
        ox = np.zeros(term_cap, np.uint64)
        oz = np.zeros(term_cap, np.uint64)
        oc = np.zeros((term_cap, 2), np.float64)
        nlog = C.c_int64()
        dim = C.c_int64()
        self._check(self.lib.liecl_ref_decision_log_pauli(
            _p(offsets, I64P), _p(x, U64P), _p(z, U64P), _p(coef), C.c_int(len(offsets) - 1),
            C.c_uint(qubits), C.c_int(int(keep_original)), C.c_double(tol), C.c_uint(threads),
            log.ctypes.data_as(C.c_void_p), C.c_int64(log_cap), C.byref(nlog), _p(oo, I64P),
            _p(ox, U64P), _p(oz, U64P), _p(oc), C.c_int64(term_cap), C.c_int64(basis_cap),
            C.byref(dim)))
        n = dim.value
        t = oo[n]
        return ClosureOut(n, (oo[: n + 1].copy(), ox[:t].copy(), oz[:t].copy(), oc[:t].copy()), None, {},
                          log[: min(nlog.value, log_cap)].copy())

    def bracket_window_dense(self, basis, d, row_begin, row_end, tol=1e-10, max_pairs=0, threads=1):
        basis = _c128(basis)
        done, nulls, ind = C.c_int64(), C.c_int64(), C.c_int64()
        secs = C.c_double()
        self._check(self.lib.liecl_ref_bracket_window_dense(
            _p(basis.view(np.float64)), C.c_int64(len(basis)), C.c_int(d), C.c_double(tol),
            C.c_int64(row_begin), C.c_int64(row_end), C.c_int64(max_pairs), C.c_uint(threads),
            C.byref(done), C.byref(nulls), C.byref(ind), C.byref(secs)))
        return {"pairs": done.value, "nulls": nulls.value, "independent": ind.value, "seconds": secs.value}

    def realize_generators_dense(self, family, qubits, seed=0, delta=1.5, restrict=False):
        cap = 1 << 26
        out = np.zeros(cap // 2, np.complex128)
        cnt, dim = C.c_int64(), C.c_int64()
        self._check(self.lib.liecl_ref_realize_generators_dense(
            C.c_int(FAMILIES[family]), C.c_uint(qubits), C.c_uint64(seed), C.c_double(delta), C.c_int(int(restrict)),
            _p(out.view(np.float64)), C.c_int64(cap), C.byref(cnt), C.byref(dim)))
        k, m = cnt.value, dim.value
        return out[: k * m * m].reshape(k, m * m).copy(), m

    def parse_pauli_sum(self, text, qubits, cap=4096):
        """(x, z, coef) of parse_pauli_sum, or ("error", message, line, column)."""
        b = text.encode()
        x, z, c = np.zeros(cap, np.uint64), np.zeros(cap, np.uint64), np.zeros((cap, 2))
        n, line, col = C.c_int64(), C.c_int64(), C.c_int64()
        st = self.lib.liecl_ref_parse_pauli_sum(b, C.c_int64(len(b)), C.c_uint(qubits), _p(x, U64P), _p(z, U64P),
                                                _p(c), C.c_int64(cap), C.byref(n), C.byref(line), C.byref(col))
        if st == 5:
            return ("error", self.lib.liecl_ref_last_error().decode(), line.value, col.value)
        self._check(st)
        k = n.value
        return x[:k].copy(), z[:k].copy(), c[:k].copy()

    # -- Alg. 2 pieces (ref_harness.cpp) ---------------------------------------
    def last_gram(self, n):
        """result.gram (A, A^-1) of the last closure_* call (matrix inversion)."""
        A = np.zeros(max(n * n, 1), np.complex128)
        Ai = np.zeros(max(n * n, 1), np.complex128)
        self._check(self.lib.liecl_ref_last_gram(C.c_int64(n), _p(A.view(np.float64)), _p(Ai.view(np.float64))))
        return A[: n * n].reshape(n, n, order="F"), Ai[: n * n].reshape(n, n, order="F")

    def gram_state_dense(self, basis, d, floor=1e-12):
        """GramState built by expand over the dense tuple: (schur before each
        expand, A, A^-1, refreshed A^-1, inverse_error before the refresh)."""
        basis = _c128(basis)
        n = len(basis)
        schur = np.zeros(max(n, 1))
        A = np.zeros(max(n * n, 1), np.complex128)
        Ai = np.zeros(max(n * n, 1), np.complex128)
        Ar = np.zeros(max(n * n, 1), np.complex128)
        err = C.c_double()
        self._check(self.lib.liecl_ref_gram_state_dense(
            _p(basis.view(np.float64)), C.c_int64(n), C.c_int(d), C.c_double(floor), _p(schur),
            _p(A.view(np.float64)), _p(Ai.view(np.float64)), _p(Ar.view(np.float64)), C.byref(err)))
        f = lambda m: m[: n * n].reshape(n, n, order="F")
        return schur[:n], f(A), f(Ai), f(Ar), err.value

    def check_matrix_inversion_dense(self, basis, d, h, tol=1e-10, floor=1e-12):
        basis = _c128(basis)
        n = len(basis)
        ind = C.c_int()
        beta = np.zeros(max(n, 1), np.complex128)
        self._check(self.lib.liecl_ref_check_matrix_inversion_dense(
            _p(basis.view(np.float64)), C.c_int64(n), C.c_int(d), _p(_c128(h).view(np.float64)), C.c_double(tol),
            C.c_double(floor), C.byref(ind), _p(beta.view(np.float64))))
        return bool(ind.value), beta[:n]

    def check_matrix_inversion_pauli(self, offsets, x, z, coef, n, qubits, tol=1e-10, floor=1e-12):
        """Tuple = sums 0..n-1, h = sum n: (independent, beta, A, A^-1)."""
        ind = C.c_int()
        beta = np.zeros(max(n, 1), np.complex128)
        A = np.zeros(max(n * n, 1), np.complex128)
        Ai = np.zeros(max(n * n, 1), np.complex128)
        self._check(self.lib.liecl_ref_check_matrix_inversion_pauli(
            _p(np.ascontiguousarray(offsets, np.int64), I64P), _p(np.ascontiguousarray(x, np.uint64), U64P),
            _p(np.ascontiguousarray(z, np.uint64), U64P), _p(np.ascontiguousarray(coef, np.float64)), C.c_int64(n),
            C.c_uint(qubits), C.c_double(tol), C.c_double(floor), _p(A.view(np.float64)), _p(Ai.view(np.float64)),
            C.byref(ind), _p(beta.view(np.float64))))
        f = lambda m: m[: n * n].reshape(n, n, order="F")
        return bool(ind.value), beta[:n], f(A), f(Ai)

    def project_residual_pauli(self, offsets, x, z, coef, n, qubits, term_cap=1 << 16):
        """Tuple = sums 0..n-1, h = sum n: ((x, z, coef) of the residual, coeffs)."""
        oo = np.zeros(2, np.int64)
        ox = np.zeros(term_cap, np.uint64)
        oz = np.zeros(term_cap, np.uint64)
        oc = np.zeros((term_cap, 2))
        coeffs = np.zeros(max(n, 1), np.complex128)
        self._check(self.lib.liecl_ref_project_residual_pauli(
            _p(np.ascontiguousarray(offsets, np.int64), I64P), _p(np.ascontiguousarray(x, np.uint64), U64P),
            _p(np.ascontiguousarray(z, np.uint64), U64P), _p(np.ascontiguousarray(coef, np.float64)), C.c_int64(n),
            C.c_uint(qubits), _p(oo, I64P), _p(ox, U64P), _p(oz, U64P), _p(oc), C.c_int64(term_cap),
            _p(coeffs.view(np.float64))))
        t = int(oo[1])
        return (ox[:t].copy(), oz[:t].copy(), oc[:t].copy()), coeffs[:n]

    def bracket_window_log_dense(self, basis, d, row_begin, row_end, tol=1e-10, max_pairs=0, threads=1):
        """Per-pair (null, independent, residual_norm) of a window of rows
        against the fixed basis (the saturated phase; ref_harness.cpp)."""
        basis = _c128(basis)
        total = sum(min(l, len(basis)) for l in range(row_begin, min(row_end, len(basis))))
        if max_pairs > 0:
            total = min(total, max_pairs)
        nul = np.zeros(max(total, 1), np.int32)
        ind = np.zeros(max(total, 1), np.int32)
        rn = np.zeros(max(total, 1))
        done = C.c_int64()
        self._check(self.lib.liecl_ref_bracket_window_log_dense(
            _p(basis.view(np.float64)), C.c_int64(len(basis)), C.c_int(d), C.c_double(tol),
            C.c_int64(row_begin), C.c_int64(row_end), C.c_int64(max_pairs), C.c_uint(threads),
            _p(nul, I32P), _p(ind, I32P), _p(rn), C.byref(done)))
        k = done.value
        return nul[:k], ind[:k], rn[:k]

    def check_sequence_dense(self, basis, cands, d, tol=1e-10, append=True, threads=1):
        basis = _c128(basis)
        cands = _c128(cands)
        ind = np.zeros(len(cands), np.int32)
        rn = np.zeros(len(cands), np.float64)
        secs = C.c_double()
        self._check(self.lib.liecl_ref_check_sequence_dense(
            _p(basis.view(np.float64)), C.c_int64(len(basis)), _p(cands.view(np.float64)),
            C.c_int64(len(cands)), C.c_int(d), C.c_double(tol), C.c_int(int(append)), C.c_uint(threads),
            _p(ind, I32P), _p(rn), C.byref(secs)))
        return ind, rn, secs.value

    # -- primitives ----------------------------------------------------------
    def commutator_dense(self, a, b, d):
        out = np.zeros(d * d, np.complex128)
        self._check(self.lib.liecl_ref_commutator_dense(_p(_c128(a).view(np.float64)),
                                                        _p(_c128(b).view(np.float64)), C.c_int(d),
                                                        _p(out.view(np.float64))))
        return out

    def inner_product_dense(self, a, b, d):
        out = np.zeros(2)
        self._check(self.lib.liecl_ref_inner_product_dense(_p(_c128(a).view(np.float64)),
                                                           _p(_c128(b).view(np.float64)), C.c_int(d), _p(out)))
        return complex(out[0], out[1])

    def norm_dense(self, a, d):
        out = C.c_double()
        self._check(self.lib.liecl_ref_norm_dense(_p(_c128(a).view(np.float64)), C.c_int(d), C.byref(out)))
        return out.value

    def project_residual_dense(self, basis, h, d):
        basis = _c128(basis)
        r = np.zeros(d * d, np.complex128)
        coeffs = np.zeros(max(len(basis), 1), np.complex128)
        self._check(self.lib.liecl_ref_project_residual_dense(
            _p(basis.view(np.float64)), C.c_int64(len(basis)), _p(_c128(h).view(np.float64)), C.c_int(d),
            _p(r.view(np.float64)), _p(coeffs.view(np.float64))))
        return r, coeffs[: len(basis)]

    def from_pauli(self, x, z, coef, qubits):
        x = np.ascontiguousarray(x, np.uint64)
        z = np.ascontiguousarray(z, np.uint64)
        coef = np.ascontiguousarray(coef, np.float64).reshape(-1, 2)
        d = 1 << qubits
        out = np.zeros(d * d, np.complex128)
        self._check(self.lib.liecl_ref_from_pauli(_p(x, U64P), _p(z, U64P), _p(coef), C.c_int64(len(x)),
                                                  C.c_uint(qubits), _p(out.view(np.float64))))
        return out

    def string_product(self, p, q, qubits):
        rx, rz = C.c_uint64(), C.c_uint64()
        ph = np.zeros(2)
        e = C.c_uint()
        com = C.c_int()
        self._check(self.lib.liecl_ref_string_product(C.c_uint64(p[0]), C.c_uint64(p[1]), C.c_uint64(q[0]),
                                                      C.c_uint64(q[1]), C.c_uint(qubits), C.byref(rx),
                                                      C.byref(rz), _p(ph), C.byref(e), C.byref(com)))
        return (rx.value, rz.value), complex(ph[0], ph[1]), e.value, bool(com.value)

    def format_pauli(self, x, z, coef, qubits):
        x = np.ascontiguousarray(x, np.uint64)
        z = np.ascontiguousarray(z, np.uint64)
        coef = np.ascontiguousarray(coef, np.float64).reshape(-1, 2)
        buf = C.create_string_buffer(1 << 20)
        self._check(self.lib.liecl_ref_format_pauli(_p(x, U64P), _p(z, U64P), _p(coef), C.c_int64(len(x)),
                                                    C.c_uint(qubits), buf, C.c_int64(len(buf))))
        return buf.value.decode()

    def format_dense(self, a, d):
        buf = C.create_string_buffer(1 << 22)
        self._check(self.lib.liecl_ref_format_dense(_p(_c128(a).view(np.float64)), C.c_int(d), buf,
                                                    C.c_int64(len(buf))))
        return buf.value.decode()

    def build_generators(self, family, qubits, seed=0, delta=1.5):
        cap = 4096
        oo = np.zeros(64, np.int64)
        ox = np.zeros(cap, np.uint64)
        oz = np.zeros(cap, np.uint64)
        oc = np.zeros((cap, 2))
        cnt = C.c_int64()
        self._check(self.lib.liecl_ref_build_generators(
            C.c_int(FAMILIES[family]), C.c_uint(qubits), C.c_uint64(seed), C.c_double(delta), _p(oo, I64P),
            _p(ox, U64P), _p(oz, U64P), _p(oc), C.c_int64(cap), C.byref(cnt)))
        n = cnt.value
        t = oo[n]
        return oo[: n + 1].copy(), ox[:t].copy(), oz[:t].copy(), oc[:t].copy()


class Port:
    """The plain-C restatement (oracle/liecl_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing; run `make -C oracle port`")
        self.lib = C.CDLL(path)
        self.lib.oracle_dense_norm.restype = C.c_double

    @staticmethod
    def _check(status):
        if status != 0:
            raise OracleError(status, "oracle restatement error")

    def closure_dense(self, gens, d, keep_original=False, tol=1e-10, threads=1, max_dim=0, row_limit=0,
                      log_cap=None):
        gens = _c128(gens)
        cap = max_dim or d * d
        basis = np.zeros((cap, d * d), np.complex128)
        ortho = np.zeros((cap, d * d), np.complex128)
        log_cap = log_cap if log_cap is not None else (1 << 16)
        log = np.zeros(max(log_cap, 1), DECISION_DTYPE)
        nlog = C.c_int64()
        st = Stats()
        self._check(self.lib.oracle_closure_dense(
            _p(gens.view(np.float64)), C.c_int(len(gens)), C.c_int(d), C.c_int(int(keep_original)),
            C.c_double(tol), C.c_int(threads), C.c_uint64(max_dim), C.c_int64(row_limit),
            _p(basis.view(np.float64)), _p(ortho.view(np.float64)), C.c_int64(cap), C.byref(st),
            log.ctypes.data_as(C.c_void_p), C.c_int64(log_cap), C.byref(nlog)))
        n = st.dimension
        stats = _stats(st)
        stats["borderline"] = stats.pop("extra")
        return ClosureOut(n, basis[:n].copy(), ortho[:n].copy(), stats, log[: min(nlog.value, log_cap)].copy())

    def closure_pauli_single(self, x, z, coef, qubits, keep_original=False, tol=1e-10, max_dim=0,
                             log_cap=1 << 22):
        x = np.ascontiguousarray(x, np.uint64)
        z = np.ascontiguousarray(z, np.uint64)
        coef = np.ascontiguousarray(coef, np.float64).reshape(-1, 2)
        cap = max_dim or 4 ** qubits
        bx = np.zeros(cap, np.uint64)
        bz = np.zeros(cap, np.uint64)
        bc = np.zeros((cap, 2))
        oc = np.zeros((cap, 2))
        log = np.zeros(log_cap, DECISION_DTYPE)
        nlog = C.c_int64()
        st = Stats()
        self._check(self.lib.oracle_closure_pauli_single(
            _p(x, U64P), _p(z, U64P), _p(coef), C.c_int(len(x)), C.c_uint(qubits), C.c_int(int(keep_original)),
            C.c_double(tol), C.c_uint64(max_dim), _p(bx, U64P), _p(bz, U64P), _p(bc), _p(oc), C.c_int64(cap),
            C.byref(st), log.ctypes.data_as(C.c_void_p), C.c_int64(log_cap), C.byref(nlog)))
        n = st.dimension
        stats = _stats(st)
        stats["borderline"] = stats.pop("extra")
        return ClosureOut(n, (bx[:n].copy(), bz[:n].copy(), bc[:n].copy()), oc[:n].copy(), stats,
                          log[: min(nlog.value, log_cap)].copy())

    def bracket_window_dense(self, basis, d, row_begin, row_end, tol=1e-10, max_pairs=0, threads=1):
        basis = _c128(basis)
        total = sum(min(l, len(basis)) for l in range(row_begin, min(row_end, len(basis))))
        total = min(total, max_pairs) if max_pairs > 0 else total
        nul = np.zeros(max(total, 1), np.int32)
        ind = np.zeros(max(total, 1), np.int32)
        rn = np.zeros(max(total, 1))
        done = C.c_int64()
        self._check(self.lib.oracle_bracket_window_dense(
            _p(basis.view(np.float64)), C.c_int64(len(basis)), C.c_int(d), C.c_double(tol), C.c_int64(row_begin),
            C.c_int64(row_end), C.c_int64(max_pairs), C.c_int(threads), _p(nul, I32P), _p(ind, I32P), _p(rn),
            C.byref(done)))
        k = done.value
        return nul[:k], ind[:k], rn[:k]

    def check_sequence_dense(self, basis, cands, d, tol=1e-10, append=True, threads=1):
        basis = _c128(basis)
        cands = _c128(cands)
        n = len(basis)
        room = np.zeros((n + (len(cands) if append else 0), d * d), np.complex128)
        room[:n] = basis
        ind = np.zeros(len(cands), np.int32)
        rn = np.zeros(len(cands))
        self._check(self.lib.oracle_check_sequence_dense(
            _p(room.view(np.float64)), C.c_int64(n), _p(cands.view(np.float64)), C.c_int64(len(cands)),
            C.c_int(d), C.c_double(tol), C.c_int(int(append)), C.c_int(threads), _p(ind, I32P), _p(rn)))
        return ind, rn, room[: n + int(ind.sum())] if append else None

    def commutator_dense(self, a, b, d):
        out = np.zeros(d * d, np.complex128)
        self._check(self.lib.oracle_dense_commutator(_p(_c128(a).view(np.float64)), _p(_c128(b).view(np.float64)),
                                                     C.c_int(d), _p(out.view(np.float64))))
        return out

    def inner_product_dense(self, a, b, d):
        out = np.zeros(2)
        self._check(self.lib.oracle_dense_inner_product(_p(_c128(a).view(np.float64)),
                                                        _p(_c128(b).view(np.float64)), C.c_int(d), _p(out)))
        return complex(out[0], out[1])

    def norm_dense(self, a, d):
        return self.lib.oracle_dense_norm(_p(_c128(a).view(np.float64)), C.c_int(d))

    def project_residual_dense(self, basis, h, d):
        basis = _c128(basis)
        r = np.zeros(d * d, np.complex128)
        coeffs = np.zeros(max(len(basis), 1), np.complex128)
        self._check(self.lib.oracle_dense_project_residual(
            _p(basis.view(np.float64)), C.c_int64(len(basis)), _p(_c128(h).view(np.float64)), C.c_int(d),
            _p(r.view(np.float64)), _p(coeffs.view(np.float64))))
        return r, coeffs[: len(basis)]

    def from_pauli(self, x, z, coef, qubits):
        x = np.ascontiguousarray(x, np.uint64)
        z = np.ascontiguousarray(z, np.uint64)
        coef = np.ascontiguousarray(coef, np.float64).reshape(-1, 2)
        d = 1 << qubits
        out = np.zeros(d * d, np.complex128)
        self._check(self.lib.oracle_from_pauli(_p(x, U64P), _p(z, U64P), _p(coef), C.c_int64(len(x)),
                                               C.c_uint(qubits), _p(out.view(np.float64))))
        return out


def pauli_single_arrays(x, z, coef):
    """(offsets, x, z, coef) for a tuple of one-term sums."""
    n = len(x)
    return (np.arange(n + 1, dtype=np.int64), np.asarray(x, np.uint64), np.asarray(z, np.uint64),
            np.asarray(coef, np.float64).reshape(-1, 2))
