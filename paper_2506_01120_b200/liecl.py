"""Python mirror of the liecl closure interface over the B200 C-ABI.

Same names, argument meaning and error behaviour as the reference's C++ API
(R: = /root/reference/proj/core/):

  run_closure(generators, method, config)          R:include/liecl/closure.hpp:125-126
  close_orthonormalization(generators, config, keep_original=True)   :119-121
  project_residual(orthonormal, h)                 R:include/liecl/closure.hpp:139-140
  commutator / inner_product / norm                R:include/liecl/operator.hpp:54-60
  Method, ClosureConfig, ClosureStats, ClosureResult, WarningRecord
                                                   R:include/liecl/closure.hpp:15-103
  Error, InvalidInputError, CapacityError, DegeneracyError, ParseError,
  TimeoutError                                     R:include/liecl/errors.hpp:10-61

Operators are `DenseOperator` (a d x d complex128 matrix) or `PauliSum`
(terms over a fixed qubit count; the B200 Pauli path takes single-string
generators). Every computation runs through libliecl_b200.so on a B200; there
is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from collections.abc import Sequence
import enum
import time
from dataclasses import dataclass, field

import numpy as np

from . import native

# ------------------------------------------------------------------ errors --


class Error(RuntimeError):
    """liecl::Error."""


class InvalidInputError(Error):
    pass


class CapacityError(Error):
    pass


class DegeneracyError(Error):
    def __init__(self, what: str, element_index: int = -1):
        super().__init__(what)
        self.element_index = element_index


class ParseError(Error):
    pass


class TimeoutError(Error):  # noqa: A001 - mirrors liecl::TimeoutError
    pass


class DeviceError(Error):
    """CUDA / driver failure (no reference counterpart)."""


_STATUS = {native.INVALID_INPUT: InvalidInputError, native.CAPACITY: CapacityError,
           native.DEGENERACY: DegeneracyError, native.TIMEOUT: TimeoutError, native.PARSE: ParseError,
           native.CUDA: DeviceError, native.NOMEM: DeviceError, native.INTERNAL: Error}


def _check(status: int) -> None:
    if status != native.OK:
        raise _STATUS.get(status, Error)(native.last_error())


# --------------------------------------------------------------- types ------


class Method(enum.Enum):
    standard_rank = native.METHOD_STANDARD_RANK
    matrix_inversion = native.METHOD_MATRIX_INVERSION
    orthonorm = native.METHOD_ORTHONORM
    orthonorm_dimonly = native.METHOD_ORTHONORM_DIMONLY


_METHOD_NAMES = {Method.standard_rank: "standard-rank", Method.matrix_inversion: "matrix-inversion",
                 Method.orthonorm: "orthonorm", Method.orthonorm_dimonly: "orthonorm-dimonly"}


def to_string(method: Method) -> str:
    return _METHOD_NAMES[method]


def method_from_string(name: str) -> Method:
    """R:src/closure.cpp:34-42."""
    for m, s in _METHOD_NAMES.items():
        if s == name:
            return m
    raise InvalidInputError(f"unknown method '{name}' (expected standard-rank, matrix-inversion, "
                            "orthonorm or orthonorm-dimonly)")


class Backend(enum.Enum):
    pauli = 0
    dense = 1


@dataclass
class DenseOperator:
    """Square complex matrix operator (R:include/liecl/dense.hpp:12-33)."""
    matrix: np.ndarray

    def __post_init__(self):
        m = np.asarray(self.matrix, dtype=np.complex128)
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise InvalidInputError("DenseOperator: matrix must be square")
        self.matrix = m

    @property
    def dim(self) -> int:
        return self.matrix.shape[0]

    def vec(self) -> np.ndarray:
        return np.asfortranarray(self.matrix).ravel(order="F")

    @staticmethod
    def from_vec(v: np.ndarray, d: int, copy: bool = True) -> "DenseOperator":
        m = np.asarray(v).reshape(d, d, order="F")  # a view of a contiguous vec
        return DenseOperator(m.copy() if copy else m)


class DenseOperatorList(Sequence):
    """result.basis / orthonormal_basis of a dense closure without copying:
    element k is a DenseOperator viewing row k of the (n, d*d) result array
    (column-major d x d), built on access."""

    def __init__(self, arr: np.ndarray, d: int):
        self.arr, self.d = arr, d

    def __len__(self) -> int:
        return len(self.arr)

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[i] for i in range(*k.indices(len(self)))]
        return DenseOperator.from_vec(self.arr[k], self.d, copy=False)

    def __eq__(self, other):
        if not isinstance(other, (list, tuple, DenseOperatorList)) or len(other) != len(self):
            return NotImplemented if not isinstance(other, (list, tuple, DenseOperatorList)) else False
        return all(np.array_equal(a.matrix, b.matrix) for a, b in zip(self, other))


@dataclass(frozen=True)
class PauliString:
    """R:include/liecl/pauli.hpp:24-38."""
    x: int
    z: int
    qubits: int

    def str(self) -> str:
        letters = "IXZY"
        return "".join(letters[((self.x >> j) & 1) | (((self.z >> j) & 1) << 1)] for j in range(self.qubits))


@dataclass
class PauliSum:
    """Sorted unique terms over `qubits` (R:include/liecl/pauli.hpp:65-109)."""
    qubits: int
    terms: list = field(default_factory=list)  # [(PauliString, complex)]

    @staticmethod
    def single(string: PauliString, coefficient: complex) -> "PauliSum":
        return PauliSum(string.qubits, [(string, complex(coefficient))])

    @property
    def dim(self) -> int:
        return 1 << self.qubits


class PauliSingleList(Sequence):
    """result.basis / orthonormal_basis of a single-string Pauli closure
    without building n PauliSum objects up front: element k is the one-term
    sum (x[k], z[k], coef[k]), built on access."""

    def __init__(self, x: np.ndarray, z: np.ndarray, coef: np.ndarray, qubits: int):
        self.x, self.z, self.coef, self.qubits = x, z, coef, qubits

    def __len__(self) -> int:
        return len(self.x)

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[i] for i in range(*k.indices(len(self)))]
        if k < 0:
            k += len(self)
        if not 0 <= k < len(self):
            raise IndexError(k)
        return PauliSum.single(PauliString(int(self.x[k]), int(self.z[k]), self.qubits),
                               complex(self.coef[k, 0], self.coef[k, 1]))

    def __eq__(self, other):
        if not isinstance(other, (list, tuple, PauliSingleList)):
            return NotImplemented
        return len(other) == len(self) and all(a == b for a, b in zip(self, other))


class PauliSumList(Sequence):
    """result.basis / orthonormal_basis of a multi-term Pauli closure: element
    k is the sum of terms [off[k], off[k+1]) of the (x, z, coef) arrays,
    built on access (a closure can hold 10^5 terms)."""

    def __init__(self, off: np.ndarray, x: np.ndarray, z: np.ndarray, coef: np.ndarray, qubits: int):
        self.off, self.x, self.z, self.coef, self.qubits = off, x, z, coef, qubits

    def __len__(self) -> int:
        return len(self.off) - 1

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[i] for i in range(*k.indices(len(self)))]
        if k < 0:
            k += len(self)
        if not 0 <= k < len(self):
            raise IndexError(k)
        return _sum_from_arrays(self.qubits, self.x[self.off[k]:], self.z[self.off[k]:], self.coef[self.off[k]:],
                                int(self.off[k + 1] - self.off[k]))

    def __eq__(self, other):
        if not isinstance(other, (list, tuple, PauliSumList)):
            return NotImplemented
        return len(other) == len(self) and all(a == b for a, b in zip(self, other))


@dataclass
class WarningRecord:
    kind: str
    detail: str
    value: float = 0.0


@dataclass
class ClosureStats:
    commutators_evaluated: int = 0
    independence_checks: int = 0
    accepted: int = 0
    wall_seconds: float = 0.0
    warnings: list = field(default_factory=list)
    engine: dict = field(default_factory=dict)  # batches / survivors / rechecks / kernels


@dataclass
class ClosureConfig:
    """R:include/liecl/closure.hpp:85-103 (+ engine knobs)."""
    tolerance: float = 1e-8
    rank_tolerance: float = 0.0
    max_dim: int = 0
    threads: int = 1
    gram_refresh_interval: int = 256
    conditioning_floor: float = 1e-12
    deadline: float | None = None  # absolute time.monotonic() value
    record_log: bool = False
    batch_max: int = 0
    # "auto": exactly anti-Hermitian operators (i*H, every dense BASELINE
    # config) take the packed-real path; "complex": always the general path
    field: str = "auto"
    # extension (not in the reference): stop the dense orthonormal closure once
    # the basis provably spans every bracket; the basis is unchanged, the
    # pair counts cover only the pairs visited
    stop_when_complete: bool = False

    def native(self) -> native.Config:
        rel = 0.0
        if self.deadline is not None:
            rel = self.deadline - time.monotonic()
            if rel <= 0:
                rel = 1e-9
        if self.field not in ("auto", "complex"):
            raise InvalidInputError(f"unknown field '{self.field}' (expected auto or complex)")
        return native.Config(float(self.tolerance), int(self.max_dim), int(self.threads), int(self.record_log),
                             rel, int(self.batch_max), 1 if self.field == "complex" else 0,
                             int(bool(self.stop_when_complete)),
                             float(self.conditioning_floor), int(self.gram_refresh_interval),
                             float(self.rank_tolerance))


@dataclass
class ClosureResult:
    basis: list
    orthonormal_basis: list | None
    dimension: int
    method: Method
    backend: Backend
    tolerance: float
    stats: ClosureStats
    decision_log: np.ndarray | None = None
    basis_array: np.ndarray | None = None  # dense: (n, d*d) vec layout; pauli: (x, z, coef)
    ortho_array: np.ndarray | None = None
    gram: tuple | None = None  # (A, A^{-1}) for matrix inversion (R:include/liecl/closure.hpp:81-82)


DECISION_DTYPE = np.dtype([("l", np.int64), ("m", np.int64), ("null_cand", np.int32),
                           ("independent", np.int32), ("rechecked", np.int32), ("pad", np.int32),
                           ("residual_norm", np.float64)])


def _parse_warnings(buf: bytes) -> list:
    out = []
    for line in buf.decode(errors="replace").splitlines():
        if not line:
            continue
        kind, value, detail = line.split("\t", 2)
        out.append(WarningRecord(kind, detail, float(value)))
    return out


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


# -------------------------------------------------------------- closures ----


def _validate(generators) -> tuple:
    """validate_generators (R:src/closure.cpp:476-496)."""
    if len(generators) == 0:
        raise InvalidInputError("closure requires a non-empty generator tuple")
    backend, dim = None, None
    for g in generators:
        if g is None:
            continue
        b = Backend.dense if isinstance(g, DenseOperator) else Backend.pauli
        if backend is None:
            backend, dim = b, g.dim
        elif b != backend or g.dim != dim:
            raise InvalidInputError("closure generators must share one backend and dimension")
    return backend or Backend.pauli, dim


def closure_dense_arrays(gens: np.ndarray, d: int, method: Method = Method.orthonorm_dimonly,
                         config: ClosureConfig | None = None, device: int = 0) -> ClosureResult:
    """Array-level entry: gens is (ngens, d*d) complex128 in vec layout."""
    config = config or ClosureConfig()
    gens = np.ascontiguousarray(gens, dtype=np.complex128)
    lib = native.load()
    cap = int(config.max_dim or d * d)
    if method == Method.matrix_inversion:
        return _closure_dense_gram(gens, d, config, device, cap)
    keep = method == Method.orthonorm
    st = native.Stats()
    wbuf = C.create_string_buffer(1 << 20)
    log_cap = (cap * cap // 2 + 64 + len(gens)) if config.record_log else 0
    log = np.zeros(max(log_cap, 1), DECISION_DTYPE)
    log_len = C.c_int64()
    cfg = config.native()
    _check(lib.liecl_b200_closure_dense(
        native.context(device), _dp(gens.view(np.float64)), C.c_int32(len(gens)), C.c_int32(d),
        C.c_int32(method.value), C.byref(cfg), None, None, C.c_int64(0), C.byref(st), wbuf,
        C.c_int64(len(wbuf)), log.ctypes.data_as(C.c_void_p) if config.record_log else None, C.c_int64(log_cap),
        C.byref(log_len)))
    n = int(st.dimension)
    # the result stays on the device: fetch exactly n elements (not the d^2 cap)
    basis = _dense_fetch(device, 0, n, d)
    ortho = _dense_fetch(device, 1, n, d) if keep else None
    warnings = _parse_warnings(wbuf.value)
    stats = ClosureStats(st.commutators_evaluated, st.independence_checks, st.accepted, st.wall_seconds, warnings,
                         {k: v for k, v in st.as_dict().items() if k in ("batches", "survivors", "rechecks", "kernels")})
    b = basis[:n]
    o = ortho[:n] if ortho is not None else (b[:0] if method == Method.standard_rank else b)
    return ClosureResult(DenseOperatorList(b, d), DenseOperatorList(o, d), n,
                         method, Backend.dense, config.tolerance, stats,
                         log[: log_len.value].copy() if config.record_log else None, b, o)


def _dense_fetch(device: int, what: int, n: int, d: int) -> np.ndarray:
    """liecl_b200_dense_fetch: the last dense closure's vectors (what 0 / 1, n x d*d)
    or Gram matrices (what 2 / 3, n x n column-major)."""
    lib = native.load()
    if what >= 2:
        out = np.zeros(n * n, np.complex128)
        if n:
            _check(lib.liecl_b200_dense_fetch(native.context(device), C.c_int32(what), C.c_int64(0), C.c_int64(n),
                                              _dp(out.view(np.float64))))
        return out.reshape(n, n, order="F")
    out = np.zeros((n, d * d), np.complex128)
    if n:
        _check(lib.liecl_b200_dense_fetch(native.context(device), C.c_int32(what), C.c_int64(0), C.c_int64(n),
                                          _dp(out.view(np.float64))))
    return out


def _closure_dense_gram(gens, d, config, device, cap) -> ClosureResult:
    """close_matrix_inversion (Alg. 2): basis = accepted unit candidates, gram = (A, A^{-1})."""
    lib = native.load()
    st = native.Stats()
    wbuf = C.create_string_buffer(1 << 20)
    log_cap = (cap * cap // 2 + 64 + len(gens)) if config.record_log else 0
    log = np.zeros(max(log_cap, 1), DECISION_DTYPE)
    log_len = C.c_int64()
    cfg = config.native()
    _check(lib.liecl_b200_closure_dense_gram(
        native.context(device), _dp(gens.view(np.float64)), C.c_int32(len(gens)), C.c_int32(d), C.byref(cfg),
        None, C.c_int64(0), None, None,
        C.byref(st), wbuf, C.c_int64(len(wbuf)), log.ctypes.data_as(C.c_void_p) if config.record_log else None,
        C.c_int64(log_cap), C.byref(log_len)))
    n = int(st.dimension)
    basis = _dense_fetch(device, 0, n, d)
    stats = ClosureStats(st.commutators_evaluated, st.independence_checks, st.accepted, st.wall_seconds,
                         _parse_warnings(wbuf.value),
                         {k: v for k, v in st.as_dict().items() if k in ("batches", "survivors", "rechecks", "kernels")})
    b = basis[:n]
    A = _dense_fetch(device, 2, n, d)
    Ai = _dense_fetch(device, 3, n, d)
    res = ClosureResult(DenseOperatorList(b, d), None, n, Method.matrix_inversion, Backend.dense,
                        config.tolerance, stats, log[: log_len.value].copy() if config.record_log else None, b, None)
    res.gram = (A, Ai)
    return res


def closure_pauli_arrays(x, z, coef, qubits: int, method: Method = Method.orthonorm_dimonly,
                         config: ClosureConfig | None = None, device: int = 0) -> ClosureResult:
    """Array-level entry for single-string generators: x, z uint64 masks, coef (n, 2) re/im."""
    config = config or ClosureConfig()
    x = np.ascontiguousarray(x, np.uint64)
    z = np.ascontiguousarray(z, np.uint64)
    coef = np.ascontiguousarray(coef, np.float64).reshape(-1, 2)
    lib = native.load()
    cap = int(config.max_dim or min(4 ** qubits, 1 << 24))
    bx = np.zeros(cap, np.uint64)
    bz = np.zeros(cap, np.uint64)
    bc = np.zeros((cap, 2))
    oc = np.zeros((cap, 2))
    st = native.Stats()
    wbuf = C.create_string_buffer(1 << 20)
    log_cap = (1 << 24) if config.record_log else 0
    log = np.zeros(max(log_cap, 1), DECISION_DTYPE)
    log_len = C.c_int64()
    cfg = config.native()
    u64 = C.POINTER(C.c_uint64)
    _check(lib.liecl_b200_closure_pauli(
        native.context(device), x.ctypes.data_as(u64), z.ctypes.data_as(u64), _dp(coef), C.c_int32(len(x)),
        C.c_uint32(qubits), C.c_int32(method.value), C.byref(cfg), bx.ctypes.data_as(u64), bz.ctypes.data_as(u64),
        _dp(bc), _dp(oc), C.c_int64(cap), C.byref(st), wbuf, C.c_int64(len(wbuf)),
        log.ctypes.data_as(C.c_void_p) if config.record_log else None, C.c_int64(log_cap), C.byref(log_len)))
    n = int(st.dimension)
    warnings = _parse_warnings(wbuf.value)
    stats = ClosureStats(st.commutators_evaluated, st.independence_checks, st.accepted, st.wall_seconds, warnings,
                         {k: v for k, v in st.as_dict().items() if k in ("batches", "survivors", "rechecks", "kernels")})

    gram = method == Method.matrix_inversion
    bx, bz, bc, oc = bx[:n].copy(), bz[:n].copy(), bc[:n].copy(), oc[:n].copy()
    res = ClosureResult(PauliSingleList(bx, bz, bc, qubits), None if gram else PauliSingleList(bx, bz, oc, qubits),
                        n, method, Backend.pauli, config.tolerance, stats,
                        log[: log_len.value].copy() if config.record_log else None,
                        (bx, bz, bc), None if gram else oc)
    if gram:  # distinct strings: A = A^{-1} = I exactly (see liecl_b200_closure_pauli)
        res.gram = (np.eye(n, dtype=np.complex128), np.eye(n, dtype=np.complex128))
    return res


def closure_pauli_sums_arrays(offsets, x, z, coef, qubits: int, method: Method = Method.orthonorm_dimonly,
                              config: ClosureConfig | None = None, device: int = 0,
                              term_cap: int | None = None) -> ClosureResult:
    """Array-level entry for general (multi-term) Pauli generators: generator i
    = terms [offsets[i], offsets[i+1]) of x, z (uint64 masks) and coef (t, 2),
    in PauliSum form. Result sums are returned as PauliSum lists and as arrays
    (`basis_array` = (offsets, x, z, coef))."""
    config = config or ClosureConfig()
    offsets = np.ascontiguousarray(offsets, np.int64)
    x = np.ascontiguousarray(x, np.uint64)
    z = np.ascontiguousarray(z, np.uint64)
    coef = np.ascontiguousarray(coef, np.float64).reshape(-1, 2)
    lib = native.load()
    u64, i64 = C.POINTER(C.c_uint64), C.POINTER(C.c_int64)
    cap = int(config.max_dim or min(4 ** qubits, 1 << 20))
    tcap = term_cap or max(1 << 16, 8 * len(x))  # first guess; a larger result is fetched, not recomputed
    while True:
        bo, oo = np.zeros(cap + 1, np.int64), np.zeros(cap + 1, np.int64)
        bx, bz, bc = np.zeros(tcap, np.uint64), np.zeros(tcap, np.uint64), np.zeros((tcap, 2))
        ox, oz, ocf = np.zeros(tcap, np.uint64), np.zeros(tcap, np.uint64), np.zeros((tcap, 2))
        need = np.zeros(2, np.int64)
        st = native.Stats()
        wbuf = C.create_string_buffer(1 << 20)
        log_cap = (1 << 24) if config.record_log else 0
        log = np.zeros(max(log_cap, 1), DECISION_DTYPE)
        log_len = C.c_int64()
        cfg = config.native()
        status = lib.liecl_b200_closure_pauli_sums(
            native.context(device), offsets.ctypes.data_as(i64), x.ctypes.data_as(u64), z.ctypes.data_as(u64),
            _dp(coef), C.c_int32(len(offsets) - 1), C.c_uint32(qubits), C.c_int32(method.value), C.byref(cfg),
            C.c_int64(cap), bo.ctypes.data_as(i64), bx.ctypes.data_as(u64), bz.ctypes.data_as(u64), _dp(bc),
            C.c_int64(tcap), oo.ctypes.data_as(i64), ox.ctypes.data_as(u64), oz.ctypes.data_as(u64), _dp(ocf),
            C.c_int64(tcap), need.ctypes.data_as(i64), C.byref(st), wbuf, C.c_int64(len(wbuf)),
            log.ctypes.data_as(C.c_void_p) if config.record_log else None, C.c_int64(log_cap), C.byref(log_len))
        if status == native.CAPACITY and native.last_error() == "output buffers too small" \
                and (need.max() > tcap or int(st.dimension) > cap):
            # the result stays on the device: fetch it with exact sizes
            tcap = int(need.max())
            cap = max(cap, int(st.dimension))
            bo, oo = np.zeros(cap + 1, np.int64), np.zeros(cap + 1, np.int64)
            bx, bz, bc = np.zeros(tcap, np.uint64), np.zeros(tcap, np.uint64), np.zeros((tcap, 2))
            ox, oz, ocf = np.zeros(tcap, np.uint64), np.zeros(tcap, np.uint64), np.zeros((tcap, 2))
            status = lib.liecl_b200_pauli_sums_fetch(
                native.context(device), C.c_int64(cap), bo.ctypes.data_as(i64), bx.ctypes.data_as(u64),
                bz.ctypes.data_as(u64), _dp(bc), C.c_int64(tcap), oo.ctypes.data_as(i64), ox.ctypes.data_as(u64),
                oz.ctypes.data_as(u64), _dp(ocf), C.c_int64(tcap))
        _check(status)
        break
    n = int(st.dimension)
    warnings = _parse_warnings(wbuf.value)
    stats = ClosureStats(st.commutators_evaluated, st.independence_checks, st.accepted, st.wall_seconds, warnings,
                         {k: v for k, v in st.as_dict().items() if k in ("batches", "survivors", "rechecks", "kernels")})

    def arrays(off, xs, zs, cs):
        t = int(off[n])
        return off[: n + 1].copy(), xs[:t].copy(), zs[:t].copy(), cs[:t].copy()
    gram = method == Method.matrix_inversion
    ba = arrays(bo, bx, bz, bc)
    oa = None if gram else arrays(oo, ox, oz, ocf)
    res = ClosureResult(PauliSumList(*ba, qubits), None if gram else PauliSumList(*oa, qubits), n, method,
                        Backend.pauli, config.tolerance, stats,
                        log[: log_len.value].copy() if config.record_log else None, ba, oa)
    if gram:  # result.gram from the device (liecl_b200_pauli_sums_fetch_gram)
        A = np.zeros(n * n, np.complex128)
        Ai = np.zeros(n * n, np.complex128)
        if n:
            _check(lib.liecl_b200_pauli_sums_fetch_gram(native.context(device), _dp(A.view(np.float64)),
                                                        _dp(Ai.view(np.float64))))
        res.gram = (A.reshape(n, n, order="F"), Ai.reshape(n, n, order="F"))
    return res


def run_closure(generators, method: Method, config: ClosureConfig | None = None, device: int = 0) -> ClosureResult:
    """R:src/closure.cpp:541-564: every method on dense generators; orthonormal
    methods and matrix inversion on single-string and multi-term Pauli
    generators (the rank method expands Pauli generators to dense, as the
    reference does, R:src/closure.cpp:545-553)."""
    backend, dim = _validate(generators)
    if method == Method.standard_rank and backend != Backend.dense:
        dense = [None if g is None else from_pauli([g], device)[0] for g in generators]
        return run_closure(dense, method, config, device)
    if backend == Backend.dense:
        gens = np.stack([g.vec() if g is not None else np.zeros(dim * dim, np.complex128) for g in generators])
        return closure_dense_arrays(gens, dim, method, config, device)
    qubits = next(g.qubits for g in generators if g is not None)
    if any(g is not None and len(g.terms) > 1 for g in generators):
        # general sums: the multi-term engine
        offs, xs, zs, cs = [0], [], [], []
        for g in generators:
            for s_, c in (g.terms if g is not None else []):
                xs.append(s_.x); zs.append(s_.z); cs.append((complex(c).real, complex(c).imag))
            offs.append(len(xs))
        return closure_pauli_sums_arrays(np.array(offs, np.int64), np.array(xs, np.uint64), np.array(zs, np.uint64),
                                         np.array(cs, np.float64).reshape(-1, 2), qubits, method, config, device)
    xs, zs, cs = [], [], []
    for g in generators:
        if g is None or len(g.terms) == 0:
            xs.append(0); zs.append(0); cs.append((0.0, 0.0))
            continue
        s, c = g.terms[0]
        xs.append(s.x); zs.append(s.z); cs.append((complex(c).real, complex(c).imag))
    return closure_pauli_arrays(np.array(xs, np.uint64), np.array(zs, np.uint64), np.array(cs), qubits, method,
                                config, device)


def close_orthonormalization(generators, config: ClosureConfig | None = None, keep_original: bool = True,
                             device: int = 0) -> ClosureResult:
    """R:include/liecl/closure.hpp:119-121 (Alg. 3 / dimension only)."""
    return run_closure(generators, Method.orthonorm if keep_original else Method.orthonorm_dimonly, config, device)


def close_matrix_inversion(generators, config: ClosureConfig | None = None, device: int = 0) -> ClosureResult:
    """R:include/liecl/closure.hpp:112-113 (Alg. 2); result.gram = (A, A^-1)."""
    return run_closure(generators, Method.matrix_inversion, config, device)


def close_standard(generators, config: ClosureConfig | None = None, device: int = 0) -> ClosureResult:
    """R:include/liecl/closure.hpp:107-108 (Alg. 1, the rank method; dense
    generators -- run_closure expands Pauli generators first, close_standard
    refuses them, R:src/closure.cpp:500-506)."""
    backend, _ = _validate(generators)
    if backend != Backend.dense and any(g is not None for g in generators):
        raise InvalidInputError("close_standard requires the dense backend; the rank check vectorizes operators")
    return run_closure(generators, Method.standard_rank, config, device)


# ------------------------------------------------- I/O plumbing (§8 f3) ----


def pauli_sum_from_terms(qubits: int, terms) -> PauliSum:
    """PauliSum::from_terms (R:src/pauli.cpp:78-115) on the device: merge
    duplicate strings in input order, drop |c| <= 1e-14 * max|c|, sort by (z, x)."""
    terms = list(terms)
    for s, _ in terms:
        if s.qubits != qubits:
            raise InvalidInputError("PauliSum::from_terms: term qubit count mismatch")
    n = len(terms)
    x = np.array([s.x for s, _ in terms], np.uint64)
    z = np.array([s.z for s, _ in terms], np.uint64)
    cf = np.array([(complex(c).real, complex(c).imag) for _, c in terms], np.float64).reshape(-1, 2)
    m = max(n, 1)
    rx, rz, rc = np.zeros(m, np.uint64), np.zeros(m, np.uint64), np.zeros((m, 2))
    nt = C.c_int64()
    u64 = C.POINTER(C.c_uint64)
    _check(native.load().liecl_b200_pauli_from_terms(
        native.context(0), C.c_int64(n), x.ctypes.data_as(u64), z.ctypes.data_as(u64), _dp(cf), C.c_uint32(qubits),
        rx.ctypes.data_as(u64), rz.ctypes.data_as(u64), _dp(rc), C.c_int64(m), C.byref(nt)))
    return _sum_from_arrays(qubits, rx, rz, rc, nt.value)


FAMILIES = {"hea": 0, "spin_glass_hva": 1, "xxz_hva": 2, "tfim_hva_open": 3}


def realize_generators(family: str, qubits: int, backend: Backend = Backend.pauli, seed: int = 0,
                       delta: float = 1.5, restrict_zero_magnetization: bool = False, device: int = 0) -> list:
    """realize_generators (R:src/generators.cpp:171-194) through the C-ABI: the
    catalog family as PauliSums, or dense operators (from_pauli on the device;
    the zero-magnetization restriction implies dense)."""
    if family not in FAMILIES:
        raise InvalidInputError(f"unknown ansatz family '{family}'")
    lib = native.load()
    count = C.c_int32()
    dense = backend == Backend.dense or restrict_zero_magnetization
    u64, i64 = C.POINTER(C.c_uint64), C.POINTER(C.c_int64)
    if not dense:
        cap = 4 * qubits * qubits + 64
        off = np.zeros(3 * qubits + 1, np.int64)
        x, z, c = np.zeros(cap, np.uint64), np.zeros(cap, np.uint64), np.zeros((cap, 2))
        _check(lib.liecl_b200_realize_generators(
            native.context(device), C.c_int32(FAMILIES[family]), C.c_uint32(qubits), C.c_uint64(seed),
            C.c_double(delta), C.c_int32(0), C.c_int32(0), C.byref(count), off.ctypes.data_as(i64),
            x.ctypes.data_as(u64), z.ctypes.data_as(u64), _dp(c), C.c_int64(cap), None, None, C.c_int64(0)))
        return [_sum_from_arrays(qubits, x[off[i]:], z[off[i]:], c[off[i]:], int(off[i + 1] - off[i]))
                for i in range(count.value)]
    d = 1 << qubits
    out = np.zeros(max(3 * qubits - 1, 2) * d * d, np.complex128)
    dim = C.c_int32()
    _check(lib.liecl_b200_realize_generators(
        native.context(device), C.c_int32(FAMILIES[family]), C.c_uint32(qubits), C.c_uint64(seed), C.c_double(delta),
        C.c_int32(int(restrict_zero_magnetization)), C.c_int32(1), C.byref(count), None, None, None, None,
        C.c_int64(0), C.byref(dim), _dp(out.view(np.float64)), C.c_int64(2 * len(out))))
    m = dim.value
    return [DenseOperator.from_vec(out[i * m * m:(i + 1) * m * m], m) for i in range(count.value)]


def parse_pauli_sum(text: str, qubits: int, device: int = 0) -> PauliSum:
    """parse_pauli_sum (R:src/pauli.cpp:230-395): the reference's grammar, e.g.
    "1.5 XIZ - (0,2) YYI"; letter j acts on qubit j. Malformed text raises
    ParseError with the reference's message and .line / .column."""
    b = text.encode()
    cap = max(1, b.count(b"X") + b.count(b"Y") + b.count(b"Z") + b.count(b"I"))
    x, z, c = np.zeros(cap, np.uint64), np.zeros(cap, np.uint64), np.zeros((cap, 2))
    n, line, col = C.c_int64(), C.c_int64(), C.c_int64()
    u64 = C.POINTER(C.c_uint64)
    st = native.load().liecl_b200_parse_pauli_sum(native.context(device), b, C.c_int64(len(b)), C.c_uint32(qubits),
                                                  x.ctypes.data_as(u64), z.ctypes.data_as(u64), _dp(c),
                                                  C.c_int64(cap), C.byref(n), C.byref(line), C.byref(col))
    if st == native.PARSE:
        e = ParseError(f"{native.last_error()} (line {line.value}, column {col.value})")
        e.line, e.column = line.value, col.value
        raise e
    _check(st)
    return _sum_from_arrays(qubits, x, z, c, n.value)


def from_pauli(sums, device: int = 0):
    """Dense expansion on the GPU, bit-exact with R:src/dense.cpp:70-98. Takes
    one PauliSum or a list (terms in PauliSum order); returns DenseOperator(s)."""
    single = isinstance(sums, PauliSum)
    sums = [sums] if single else list(sums)
    if not sums:
        return []
    n = sums[0].qubits
    offsets = np.zeros(len(sums) + 1, np.int64)
    xs, zs, cs = [], [], []
    for i, s in enumerate(sums):
        if s.qubits != n:
            raise InvalidInputError("from_pauli: mixed qubit counts")
        for st, c in s.terms:
            xs.append(st.x); zs.append(st.z); cs.append((complex(c).real, complex(c).imag))
        offsets[i + 1] = len(xs)
    x = np.array(xs or [0], np.uint64)
    z = np.array(zs or [0], np.uint64)
    c = np.array(cs or [(0.0, 0.0)], np.float64)
    d = 1 << n
    out = np.zeros((len(sums), d * d), np.complex128)
    u64 = C.POINTER(C.c_uint64)
    _check(native.load().liecl_b200_from_pauli(
        native.context(device), offsets.ctypes.data_as(C.POINTER(C.c_int64)), x.ctypes.data_as(u64),
        z.ctypes.data_as(u64), _dp(c), C.c_int32(len(sums)), C.c_uint32(n), _dp(out.view(np.float64)), C.c_int32(0)))
    ops = [DenseOperator.from_vec(v, d) for v in out]
    return ops[0] if single else ops


def _fmt_real(v: float) -> str:
    return "%.17g" % v


def format_pauli_sum(s: PauliSum) -> str:
    """R:src/pauli.cpp:397-422."""
    if not s.terms:
        return "0 " + "I" * s.qubits
    out = []
    for k, (st, c) in enumerate(s.terms):
        c = complex(c)
        if c.imag == 0.0:
            re = c.real
            if k:
                out.append(" - " if re < 0.0 else " + ")
                re = abs(re)
            out.append(_fmt_real(re))
        else:
            if k:
                out.append(" + ")
            out.append("(" + _fmt_real(c.real) + "," + _fmt_real(c.imag) + ")")
        out.append(" " + st.str())
    return "".join(out)


def format_operator(op) -> str:
    """R:src/operator.cpp:206-226: Pauli text, or full-precision row-major dense entries."""
    if op is None:
        return "null"
    if isinstance(op, PauliSum):
        return format_pauli_sum(op)
    m = op.matrix
    rows = []
    for r in range(m.shape[0]):
        rows.append(" ".join("(%.17g,%.17g)" % (m[r, c].real, m[r, c].imag) for c in range(m.shape[1])) + "\n")
    return "".join(rows)


def basis_listing(result: ClosureResult) -> str:
    """R:src/closure.cpp:566-573."""
    return "".join(format_operator(op) + "\n" for op in result.basis)


# ------------------------------------------------------------ primitives ----


def _sums_arrays(sums):
    """A tuple of PauliSums (None = null: no terms) -> (offsets, x, z, coef (t, 2))."""
    offs, xs, zs, cs = [0], [], [], []
    for g in sums:
        for s_, c in (g.terms if g is not None else []):
            c = complex(c)
            xs.append(s_.x); zs.append(s_.z); cs.append((c.real, c.imag))
        offs.append(len(xs))
    return (np.array(offs, np.int64), np.array(xs, np.uint64), np.array(zs, np.uint64),
            np.array(cs, np.float64).reshape(-1, 2))


def _sum_args(sums, h, qubits):
    o, x, z, c = _sums_arrays(sums)
    ho, hx, hz, hc = _sums_arrays([h])
    u64, i64 = C.POINTER(C.c_uint64), C.POINTER(C.c_int64)
    keep = (o, x, z, c, hx, hz, hc)
    args = [o.ctypes.data_as(i64), x.ctypes.data_as(u64), z.ctypes.data_as(u64), _dp(c), C.c_int64(len(sums)),
            C.c_uint32(qubits), C.c_int64(len(hx)), hx.ctypes.data_as(u64), hz.ctypes.data_as(u64), _dp(hc)]
    return args, keep, int(ho[-1] + o[-1])


def _sum_from_arrays(qubits, x, z, c, nt) -> PauliSum:
    return PauliSum(qubits, [(PauliString(int(x[t]), int(z[t]), qubits), complex(c[t, 0], c[t, 1]))
                             for t in range(nt)])


def _pauli_project_residual(orthonormal, h: PauliSum, device: int):
    """project_residual over Pauli sums on the device (SumEngine passes), bit-exact."""
    args, keep, bound = _sum_args(orthonormal, h, h.qubits)
    bound = max(bound, 1)
    rx, rz, rc = np.zeros(bound, np.uint64), np.zeros(bound, np.uint64), np.zeros((bound, 2))
    nt = C.c_int64()
    coeffs = np.zeros(max(len(orthonormal), 1), np.complex128)
    u64 = C.POINTER(C.c_uint64)
    _check(native.load().liecl_b200_project_residual_pauli(
        native.context(device), *args, rx.ctypes.data_as(u64), rz.ctypes.data_as(u64), _dp(rc), C.c_int64(bound),
        C.byref(nt), _dp(coeffs.view(np.float64))))
    return _sum_from_arrays(h.qubits, rx, rz, rc, nt.value), list(coeffs[: len(orthonormal)])


def _pauli_linear_combination(base: PauliSum, base_coeff: complex, tuple_, coeffs, device: int) -> PauliSum:
    """from_terms(base_coeff * base ++ coeffs[l] * tuple_[l]) on the device."""
    args, keep, bound = _sum_args(tuple_, base, base.qubits)
    bound = max(bound, 1)
    cf = np.array([[complex(c).real, complex(c).imag] for c in coeffs] or [[0.0, 0.0]], np.float64)
    rx, rz, rc = np.zeros(bound, np.uint64), np.zeros(bound, np.uint64), np.zeros((bound, 2))
    nt = C.c_int64()
    u64 = C.POINTER(C.c_uint64)
    _check(native.load().liecl_b200_linear_combination_pauli(
        native.context(device), *args, C.c_double(complex(base_coeff).real), C.c_double(complex(base_coeff).imag),
        _dp(cf), rx.ctypes.data_as(u64), rz.ctypes.data_as(u64), _dp(rc), C.c_int64(bound), C.byref(nt)))
    return _sum_from_arrays(base.qubits, rx, rz, rc, nt.value)


def check_matrix_inversion(gram: tuple, basis, h, tol: float, device: int = 0):
    """check_matrix_inversion (R:src/closure.cpp:107-140) on the device:
    (independent, beta). gram = (A, A^{-1}) n x n; basis = n operators."""
    A, Ai = gram
    n = len(basis)
    if Ai.shape != (n, n):
        raise InvalidInputError("check_matrix_inversion: state size does not match basis size")
    if h is None:
        return 0.0 > tol, [0j] * n
    ind = C.c_int32()
    beta = np.zeros(max(n, 1), np.complex128)
    inv = np.asfortranarray(Ai, np.complex128).ravel(order="F")
    if isinstance(h, PauliSum):
        args, keep, _ = _sum_args(basis, h, h.qubits)
        ao = args[:6]
        _check(native.load().liecl_b200_check_matrix_inversion_pauli(
            native.context(device), *ao, _dp(inv.view(np.float64)), *args[6:], C.c_double(tol), C.byref(ind),
            _dp(beta.view(np.float64)), None))
    else:
        d = h.dim
        B = np.ascontiguousarray(np.stack([b.vec() if b is not None else np.zeros(d * d, np.complex128)
                                           for b in basis]) if n else np.zeros((1, d * d), np.complex128))
        hv = np.ascontiguousarray(h.vec())
        _check(native.load().liecl_b200_check_matrix_inversion_dense(
            native.context(device), _dp(B.view(np.float64)), C.c_int64(n), _dp(inv.view(np.float64)),
            _dp(hv.view(np.float64)), C.c_int32(d), C.c_double(tol), C.byref(ind), _dp(beta.view(np.float64)), None))
    return bool(ind.value), list(beta[:n])


class GramState:
    """GramState (R:include/liecl/closure.hpp:28-55; R:src/closure.cpp:44-105)
    with its operations on the device (liecl_b200_gram_*)."""

    def __init__(self, gram=None, inverse=None, device: int = 0):
        self.gram = np.zeros((0, 0), np.complex128) if gram is None else np.asarray(gram, np.complex128)
        self.inverse = np.zeros((0, 0), np.complex128) if inverse is None else np.asarray(inverse, np.complex128)
        self.device = device

    def size(self) -> int:
        return self.gram.shape[0]

    @staticmethod
    def _f(m):
        return np.ascontiguousarray(np.asarray(m, np.complex128).ravel(order="F"))

    def schur_complement(self, beta) -> float:
        beta = np.ascontiguousarray(beta, np.complex128)
        if len(beta) != self.size():
            raise InvalidInputError("GramState: beta length does not match basis size")
        s = C.c_double()
        inv = self._f(self.inverse)
        _check(native.load().liecl_b200_gram_schur_complement(native.context(self.device), _dp(inv.view(np.float64)),
                                                              C.c_int64(len(beta)), _dp(beta.view(np.float64)),
                                                              C.byref(s)))
        return s.value

    def expand(self, beta, conditioning_floor: float) -> None:
        beta = np.ascontiguousarray(beta, np.complex128)
        n = self.size()
        if len(beta) != n:
            raise InvalidInputError("GramState: beta length does not match basis size")
        a = np.zeros((n + 1) ** 2, np.complex128)
        ai = np.zeros((n + 1) ** 2, np.complex128)
        g, inv = self._f(self.gram), self._f(self.inverse)
        st = native.load().liecl_b200_gram_expand(
            native.context(self.device), _dp(g.view(np.float64)), _dp(inv.view(np.float64)), C.c_int64(n),
            _dp(beta.view(np.float64)), C.c_double(conditioning_floor), _dp(a.view(np.float64)),
            _dp(ai.view(np.float64)))
        if st == native.DEGENERACY:
            raise DegeneracyError(native.last_error(), n)
        _check(st)
        self.gram = a.reshape(n + 1, n + 1, order="F")
        self.inverse = ai.reshape(n + 1, n + 1, order="F")

    def refresh(self) -> None:
        n = self.size()
        if n == 0:
            return
        ai = np.zeros(n * n, np.complex128)
        g = self._f(self.gram)
        _check(native.load().liecl_b200_gram_refresh(native.context(self.device), _dp(g.view(np.float64)),
                                                     C.c_int64(n), _dp(ai.view(np.float64))))
        self.inverse = ai.reshape(n, n, order="F")

    def inverse_error(self) -> float:
        e = C.c_double()
        g, inv = self._f(self.gram), self._f(self.inverse)
        _check(native.load().liecl_b200_gram_inverse_error(native.context(self.device), _dp(g.view(np.float64)),
                                                           _dp(inv.view(np.float64)), C.c_int64(self.size()),
                                                           C.byref(e)))
        return e.value


def project_residual(orthonormal, h, device: int = 0):
    """(residual, first-pass coefficients), R:src/closure.cpp:142-162; dense
    operators or Pauli sums, on the device."""
    orthonormal = list(orthonormal)
    if not orthonormal:
        return h, []
    if isinstance(h, PauliSum):
        if any(not isinstance(v, PauliSum) or v.qubits != h.qubits for v in orthonormal if v is not None):
            raise InvalidInputError("inner_product: operators have mismatched backends or dimensions")
        return _pauli_project_residual(orthonormal, h, device)
    d = h.dim
    V = np.ascontiguousarray(np.stack([v.vec() for v in orthonormal]) if len(orthonormal) else
                             np.zeros((0, d * d), np.complex128))
    r = np.zeros(d * d, np.complex128)
    coeffs = np.zeros(max(len(orthonormal), 1), np.complex128)
    hv = np.ascontiguousarray(h.vec())
    _check(native.load().liecl_b200_project_residual_dense(
        native.context(device), _dp(V.view(np.float64)) if len(V) else None, C.c_int64(len(V)),
        _dp(hv.view(np.float64)), C.c_int32(d), _dp(r.view(np.float64)), _dp(coeffs.view(np.float64))))
    return DenseOperator.from_vec(r, d), list(coeffs[: len(orthonormal)])


def commutator(a: DenseOperator, b: DenseOperator, device: int = 0) -> DenseOperator:
    if a.dim != b.dim:
        raise InvalidInputError("commutator: operators have mismatched backends or dimensions")
    out = np.zeros(a.dim * a.dim, np.complex128)
    av, bv = np.ascontiguousarray(a.vec()), np.ascontiguousarray(b.vec())
    _check(native.load().liecl_b200_commutator_dense(native.context(device), _dp(av.view(np.float64)),
                                                     _dp(bv.view(np.float64)), C.c_int32(a.dim),
                                                     _dp(out.view(np.float64))))
    return DenseOperator.from_vec(out, a.dim)


def inner_product(a, b, device: int = 0) -> complex:
    """(1/d) tr(a^dagger b) (R:src/operator.cpp:66-75): null -> 0; Pauli sums by
    the sorted merge of sum_inner_product (R:src/pauli.cpp:202-220); dense on
    the GPU."""
    if a is None or b is None:
        return complex(0.0, 0.0)
    if isinstance(a, PauliSum) or isinstance(b, PauliSum):
        if not (isinstance(a, PauliSum) and isinstance(b, PauliSum)) or a.qubits != b.qubits:
            raise InvalidInputError("inner_product: operators have mismatched backends or dimensions")
        args, keep, _ = _sum_args([a], b, a.qubits)
        out = np.zeros(1, np.complex128)
        _check(native.load().liecl_b200_overlaps_pauli(native.context(device), *args, _dp(out.view(np.float64))))
        return complex(out[0])
    if a.dim != b.dim:
        raise InvalidInputError("inner_product: operators have mismatched backends or dimensions")
    out = np.zeros(2)
    av, bv = np.ascontiguousarray(a.vec()), np.ascontiguousarray(b.vec())
    _check(native.load().liecl_b200_inner_product_dense(native.context(device), _dp(av.view(np.float64)),
                                                        _dp(bv.view(np.float64)), C.c_int32(a.dim), _dp(out)))
    return complex(out[0], out[1])


def norm(a, device: int = 0) -> float:
    """sqrt(inner_product(a, a)) (R:src/operator.cpp:77-82): null -> 0; Pauli
    sums sqrt(sum |c|^2) in term order (R:src/pauli.cpp:222-228); dense on the
    GPU."""
    if a is None:
        return 0.0
    if isinstance(a, PauliSum):
        _, hx, hz, hc = _sums_arrays([a])
        out = C.c_double()
        u64 = C.POINTER(C.c_uint64)
        _check(native.load().liecl_b200_norm_pauli(native.context(device), C.c_int64(len(hx)),
                                                   hx.ctypes.data_as(u64), hz.ctypes.data_as(u64), _dp(hc),
                                                   C.c_uint32(a.qubits), C.byref(out)))
        return out.value
    out = C.c_double()
    av = np.ascontiguousarray(a.vec())
    _check(native.load().liecl_b200_norm_dense(native.context(device), _dp(av.view(np.float64)), C.c_int32(a.dim),
                                               C.byref(out)))
    return out.value


def axpy_dot(tuple_, coeffs, device: int = 0):
    """sum_l coeffs[l] * tuple_[l]; the empty combination is null
    (R:src/operator.cpp:123-135)."""
    tuple_, coeffs = list(tuple_), list(coeffs)
    if len(tuple_) != len(coeffs):
        raise InvalidInputError(f"axpy_dot: tuple and coefficient lengths differ ({len(tuple_)} vs {len(coeffs)})")
    if not tuple_:
        return None
    return linear_combination(tuple_[0], coeffs[0], tuple_[1:], coeffs[1:], device)


def is_zero(a, tol: float, device: int = 0) -> bool:
    """norm(a) <= tol (R:src/operator.cpp:183-188)."""
    if tol < 0.0:
        raise InvalidInputError("is_zero: tolerance must be non-negative")
    return norm(a, device) <= tol


def normalized(a, device: int = 0):
    """Complex{1/norm(a), 0} * a (R:src/operator.cpp:190-196)."""
    n = norm(a, device)
    if n == 0.0:
        raise InvalidInputError("normalized: null operator")
    s = complex(1.0 / n, 0.0)
    if isinstance(a, PauliSum):
        return _pauli_scale(a, s, device)
    return _linear_combination_dense(a, s, [], [], device)


def _pauli_add(a: PauliSum, b: PauliSum, device: int = 0) -> PauliSum:
    """PauliSum::operator+ (R:src/pauli.cpp:128-159) on the device: the sorted
    merge a + b with the drop rule is from_terms(1 * a ++ 1 * b) (slots start at
    +0, so the sums are the same)."""
    if a.qubits != b.qubits:
        raise InvalidInputError("PauliSum::operator+: qubit counts differ")
    return _pauli_linear_combination(a, 1.0, [b], [1.0], device)


def _pauli_scale(a: PauliSum, c: complex, device: int = 0) -> PauliSum:
    """PauliSum::operator*(Complex) (R:src/pauli.cpp:166-177): every term times
    c, no merge or drop (a sum's strings are already unique)."""
    c = complex(c)
    if c == 0:
        return PauliSum(a.qubits, [])
    _, x, z, cf = _sums_arrays([a])
    out = np.zeros((max(len(x), 1), 2))
    _check(native.load().liecl_b200_scale_terms(native.context(device), C.c_int64(len(x)), _dp(cf),
                                                C.c_double(c.real), C.c_double(c.imag), _dp(out)))
    return PauliSum(a.qubits, [(s, complex(out[t, 0], out[t, 1])) for t, (s, _) in enumerate(a.terms)])


def linear_combination(base, base_coeff: complex, tuple_, coeffs, device: int = 0):
    """linear_combination (R:src/operator.cpp:137-182): base_coeff * base +
    sum_l coeffs[l] * tuple_[l] in index order. Operators are DenseOperator,
    PauliSum or None (null). Dense: on the GPU, products and sums rounded one
    by one as the reference does. Pauli: one from_terms over the scaled terms
    (the reference's construction). A null or empty-Pauli base falls back to
    the chained addition of the reference (:147-154)."""
    tuple_ = list(tuple_)
    coeffs = [complex(c) for c in coeffs]
    if len(tuple_) != len(coeffs):
        raise InvalidInputError("linear_combination: tuple and coefficient lengths differ")
    ops = [o for o in [base] + tuple_ if o is not None]
    if ops:
        kind, dim = type(ops[0]), ops[0].dim
        if any(type(o) is not kind or o.dim != dim for o in ops):
            raise InvalidInputError("linear_combination: operators have mismatched backends or dimensions")
    if base is None or (isinstance(base, PauliSum) and not base.terms):
        if ops and isinstance(ops[0], DenseOperator):
            return _linear_combination_dense(None, 0j, tuple_, coeffs, device)
        acc = base
        for op, c in zip(tuple_, coeffs):
            if op is None:
                continue
            term = _pauli_scale(op, c, device)
            acc = term if acc is None else _pauli_add(acc, term, device)
        return acc
    if isinstance(base, DenseOperator):
        return _linear_combination_dense(base, complex(base_coeff), tuple_, coeffs, device)
    # the PauliSum branch (R:src/operator.cpp:164-181) on the device
    keep = [(op, c) for op, c in zip(tuple_, coeffs) if op is not None]
    return _pauli_linear_combination(base, base_coeff, [o for o, _ in keep], [c for _, c in keep], device)


def _linear_combination_dense(base, base_coeff, tuple_, coeffs, device):
    ref = base if base is not None else next(o for o in tuple_ if o is not None)
    d = ref.dim
    n = len(tuple_)
    T = np.zeros((max(n, 1), d * d), np.complex128)
    nul = np.zeros(max(n, 1), np.int32)
    for l, op in enumerate(tuple_):
        if op is None:
            nul[l] = 1
        else:
            T[l] = op.vec()
    cf = np.array([[c.real, c.imag] for c in coeffs] or [[0.0, 0.0]], np.float64)
    out = np.zeros(d * d, np.complex128)
    out_null = C.c_int32()
    bv = np.ascontiguousarray(base.vec()) if base is not None else None
    _check(native.load().liecl_b200_linear_combination_dense(
        native.context(device), _dp(bv.view(np.float64)) if bv is not None else None, C.c_double(base_coeff.real),
        C.c_double(base_coeff.imag), _dp(T.view(np.float64)), _dp(cf), nul.ctypes.data_as(C.POINTER(C.c_int32)),
        C.c_int64(n), C.c_int32(d), _dp(out.view(np.float64)), C.byref(out_null)))
    return None if out_null.value else DenseOperator.from_vec(out, d)


# --------------------------------------------------------------- sessions ---


def shard_range(d: int, nranks: int, rank: int) -> tuple[int, int]:
    """Elements [lo, hi) of a d*d operator held by D-shard `rank` of `nranks`."""
    lo, hi = C.c_int64(), C.c_int64()
    _check(native.load().liecl_b200_shard_range(C.c_int32(d), C.c_int32(nranks), C.c_int32(rank), C.byref(lo),
                                                 C.byref(hi)))
    return lo.value, hi.value


def loop_shard_range(d: int, nranks: int, rank: int) -> tuple[int, int]:
    """Elements [lo, hi) whose projections rank `rank` of a D-sharded closure
    loop computes (even bounds, on the GEMMs' 128-row tiles when the slices are wide
    enough; liecl_b200_loop_shard_range)."""
    lo, hi = C.c_int64(), C.c_int64()
    _check(native.load().liecl_b200_loop_shard_range(C.c_int32(d), C.c_int32(nranks), C.c_int32(rank), C.byref(lo),
                                                     C.byref(hi)))
    return lo.value, hi.value


def _resident_nccl() -> None:
    """Make torch's NCCL the process's libnccl.so.2 before the engine dlopens
    one: a later `import torch` would otherwise bind libtorch_cuda to whichever
    libnccl.so.2 is already loaded (an older system copy lacks its symbols)."""
    try:
        import torch  # noqa: F401  (loads libtorch_cuda and its bundled libnccl)
    except ImportError:
        pass


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes) for ClosureSession.set_shards."""
    _resident_nccl()
    buf = (C.c_uint8 * 128)()
    _check(native.load().liecl_b200_nccl_unique_id(buf))
    return bytes(buf)


class ClosureSession:
    """Device-resident basis + cursor loop (include/liecl_b200.h sessions)."""

    def __init__(self, d: int, keep_original: bool = False, config: ClosureConfig | None = None, device: int = 0,
                 ctx=None):
        self.d = d
        self.width = d * d  # elements of each operator this session holds (a slice once D-sharded)
        self.device = device
        self.lib = native.load()
        cfg = (config or ClosureConfig()).native()
        self.ptr = C.c_void_p()
        self._reduce = None
        # the session is bound to a context: keep this thread's alive with it
        self._ctx_ref = native.context_ref(device) if ctx is None else None
        _check(self.lib.liecl_b200_session_create_dense(ctx if ctx is not None else self._ctx_ref.ptr,
                                                        C.c_int32(d), C.c_int32(int(keep_original)), C.byref(cfg),
                                                        C.byref(self.ptr)))

    def set_loop_shards(self, nranks: int, rank: int, nccl_id: bytes | None = None, reduce=None):
        """D-shard the closure loop of this (fresh) session: operators stay whole
        on every rank, the projection GEMMs cover loop_shard_range(d, nranks,
        rank) only and their partial sums (and each accepted vector's slices)
        are summed over ranks through NCCL or `reduce` (as set_shards)."""
        self._set_shards(self.lib.liecl_b200_session_set_loop_shards, nranks, rank, nccl_id, reduce)

    def run_closure(self, gens) -> dict:
        """The whole closure from `gens` ((ngens, d*d) complex128, full operators):
        generator loop, then every cursor pair (liecl_b200_session_run_closure)."""
        gens = np.ascontiguousarray(gens, np.complex128)
        st = native.Stats()
        _check(self.lib.liecl_b200_session_run_closure(self.ptr, _dp(gens.view(np.float64)), C.c_int32(len(gens)),
                                                       C.byref(st)))
        return st.as_dict()

    def comm_bytes(self) -> int:
        """Bytes this rank has summed over ranks so far (D-sharded sessions)."""
        b = C.c_uint64()
        _check(self.lib.liecl_b200_session_comm_bytes(self.ptr, C.byref(b)))
        return b.value

    def warnings(self) -> list:
        buf = C.create_string_buffer(1 << 20)
        _check(self.lib.liecl_b200_session_warnings(self.ptr, buf, C.c_int64(len(buf))))
        return _parse_warnings(buf.value)

    def set_shards(self, nranks: int, rank: int, nccl_id: bytes | None = None, reduce=None):
        self._set_shards(self.lib.liecl_b200_session_set_shards, nranks, rank, nccl_id, reduce)
        lo, hi = shard_range(self.d, nranks, rank)
        self.width = hi - lo

    def _set_shards(self, fn, nranks: int, rank: int, nccl_id: bytes | None = None, reduce=None):
        """D-shard this (fresh) session: it then holds elements shard_range(d, nranks, rank)
        of every operator; overlaps and squared norms are summed over ranks through
        NCCL (`nccl_id` from nccl_unique_id(), shared by the caller) or through
        `reduce(values: np.ndarray)`, which must replace `values` in place by the
        sum over ranks with identical bits on every rank."""
        if nccl_id is not None:
            if len(nccl_id) != 128:
                raise InvalidInputError("an NCCL unique id is 128 bytes")
            _resident_nccl()
            buf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
            _check(fn(self.ptr, C.c_int32(nranks), C.c_int32(rank), buf, native.ReduceFn(), None))
        elif reduce is not None:
            def trampoline(values, count, _user):
                try:
                    reduce(np.ctypeslib.as_array(values, shape=(count,)))
                    return 0
                except Exception:  # reported as a failed reduction by the engine
                    return 1
            self._reduce = native.ReduceFn(trampoline)  # keep alive as long as the session
            _check(fn(self.ptr, C.c_int32(nranks), C.c_int32(rank), None, self._reduce, None))
        else:
            raise InvalidInputError("set_shards needs nccl_id or reduce")

    def close(self):
        if self.ptr:
            self.lib.liecl_b200_session_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_basis(self, V, on_device: bool = False, n: int | None = None):
        """V: (n, width) complex128 host array, or a pointer (int; device memory
        with on_device, else host -- e.g. pinned memory a prefetch_basis started)."""
        if (on_device or isinstance(V, int)) and n is None:
            raise InvalidInputError("set_basis with a pointer needs the basis size n")
        if on_device or isinstance(V, int):
            _check(self.lib.liecl_b200_session_set_basis(self.ptr, C.cast(C.c_void_p(V), C.POINTER(C.c_double)),
                                                         C.c_int64(n), C.c_int32(int(on_device))))
        else:
            V = np.ascontiguousarray(V, np.complex128)
            _check(self.lib.liecl_b200_session_set_basis(self.ptr, _dp(V.view(np.float64)), C.c_int64(len(V)),
                                                         C.c_int32(0)))

    def prefetch_basis(self, V_ptr: int, n: int):
        """Start the async H2D copy of the host basis at V_ptr (pinned, (n, width)
        complex128) for the next set_basis(V_ptr, n=n) -- overlaps the current work."""
        _check(self.lib.liecl_b200_session_prefetch_basis(self.ptr, C.cast(C.c_void_p(V_ptr), C.POINTER(C.c_double)),
                                                          C.c_int64(n)))

    def prefetch_candidates(self, cands_ptr: int, n: int):
        """Start the async H2D copy of n host candidates at cands_ptr (pinned,
        (n, width) complex128); the next check_candidates(cands_ptr, n=n) reads
        the device copy. Up to two copies in flight (the next step's while the
        current one is checked); the host memory must stay unchanged until then."""
        _check(self.lib.liecl_b200_session_prefetch_candidates(
            self.ptr, C.cast(C.c_void_p(cands_ptr), C.POINTER(C.c_double)), C.c_int64(n)))

    def run_pairs(self, g_begin: int, g_end: int) -> dict:
        st = native.Stats()
        _check(self.lib.liecl_b200_session_run_pairs(self.ptr, C.c_int64(g_begin), C.c_int64(g_end), C.byref(st)))
        return st.as_dict()

    def run_rows(self, row_begin: int, row_end: int) -> dict:
        st = native.Stats()
        _check(self.lib.liecl_b200_session_run_rows(self.ptr, C.c_int64(row_begin), C.c_int64(row_end),
                                                    C.byref(st)))
        return st.as_dict()

    def screen_pairs(self, g_begin: int, g_end: int):
        """(null flags, pass-1 residual norms) of pairs [g_begin, g_end); no state change."""
        cnt = max(g_end - g_begin, 0)
        nul = np.zeros(max(cnt, 1), np.int32)
        rn = np.zeros(max(cnt, 1))
        _check(self.lib.liecl_b200_session_screen_pairs(self.ptr, C.c_int64(g_begin), C.c_int64(g_end),
                                                        nul.ctypes.data_as(C.POINTER(C.c_int32)), _dp(rn)))
        return nul[:cnt], rn[:cnt]

    def size(self) -> int:
        n = C.c_int64()
        _check(self.lib.liecl_b200_session_size(self.ptr, C.byref(n)))
        return n.value

    def field(self) -> str:
        f = C.c_int32()
        _check(self.lib.liecl_b200_session_field(self.ptr, C.byref(f)))
        return {0: "unset", 1: "complex", 2: "antihermitian_packed"}[f.value]

    def basis(self, ortho: bool = False) -> np.ndarray:
        """The commutator basis (host copy); ortho=True: the orthonormal tuple
        (they differ for Alg. 3 sessions, keep_original)."""
        n = self.size()
        out = np.zeros((n, self.width), np.complex128)
        if ortho:
            _check(self.lib.liecl_b200_session_get_vectors(self.ptr, C.c_int64(0), C.c_int64(n),
                                                           _dp(out.view(np.float64)), C.c_int32(0), C.c_int32(1)))
        else:
            _check(self.lib.liecl_b200_session_get_basis(self.ptr, _dp(out.view(np.float64)), C.c_int64(n)))
        return out

    def vectors_to(self, first: int, count: int, out_ptr: int, on_device: bool = True, ortho: bool = False):
        """Copy basis elements [first, first+count) into caller memory (e.g. a torch tensor's data_ptr())."""
        _check(self.lib.liecl_b200_session_get_vectors(self.ptr, C.c_int64(first), C.c_int64(count),
                                                       C.cast(C.c_void_p(out_ptr), C.POINTER(C.c_double)),
                                                       C.c_int32(int(on_device)), C.c_int32(int(ortho))))

    def log(self) -> np.ndarray:
        n = C.c_int64()
        _check(self.lib.liecl_b200_session_get_log(self.ptr, None, C.c_int64(0), C.byref(n)))
        out = np.zeros(max(n.value, 1), DECISION_DTYPE)
        _check(self.lib.liecl_b200_session_get_log(self.ptr, out.ctypes.data_as(C.c_void_p), C.c_int64(n.value),
                                                   C.byref(n)))
        return out[: n.value]

    def check_candidates(self, cands, on_device: bool = False, n: int | None = None):
        """cands: (n, width) complex128 host array, or a pointer (int; device memory
        with on_device, else host -- e.g. pinned) with the count n."""
        if on_device or isinstance(cands, int):
            if n is None:
                raise InvalidInputError("check_candidates with a pointer needs the candidate count n")
            ptr = C.cast(C.c_void_p(cands), C.POINTER(C.c_double))
        else:
            cands = np.ascontiguousarray(cands, np.complex128)
            ptr = _dp(cands.view(np.float64))
            n = len(cands)
        ind = np.zeros(n, np.int32)
        rn = np.zeros(n)
        st = native.Stats()
        _check(self.lib.liecl_b200_session_check_candidates(self.ptr, ptr, C.c_int64(n), C.c_int32(int(on_device)),
                                                            ind.ctypes.data_as(C.POINTER(C.c_int32)), _dp(rn),
                                                            C.byref(st)))
        return ind, rn, st.as_dict()
