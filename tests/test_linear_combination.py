"""linear_combination (R:src/operator.cpp:137-182) against the reference
build: the Pauli branch (SumEngine merges) and the dense branch (GPU kernel),
bit for bit; null / empty-base fallbacks; argument errors (raised before any
device work, so they run on CPU)."""
import ctypes as C

import numpy as np
import pytest

from paper_2506_01120_b200 import liecl


def _rand_sum(rng, n, k):
    # built with the host recipe (test infrastructure); the product's from_terms runs on the device
    from paper_2506_01120_b200 import workloads as w
    raw = [((int(rng.integers(0, 1 << n)), int(rng.integers(0, 1 << n))), complex(*rng.standard_normal(2)))
           for _ in range(k)]
    b = w.PauliSumSpec.from_terms(n, raw)
    return liecl.PauliSum(n, [(liecl.PauliString(int(x), int(z), n), c) for x, z, c in zip(b.x, b.z, b.coef)])


def _ref_lc_pauli(ref, base, bc, tup, coeffs, n):
    ops = [base] + list(tup)
    offs, xs, zs, cs, nul = [0], [], [], [], []
    for o in ops:
        nul.append(1 if o is None else 0)
        for s, c in ([] if o is None else o.terms):
            xs.append(s.x); zs.append(s.z); cs.append((c.real, c.imag))
        offs.append(len(xs))
    off = np.array(offs, np.int64); x = np.array(xs or [0], np.uint64); z = np.array(zs or [0], np.uint64)
    c = np.array(cs or [(0.0, 0.0)], np.float64); nul = np.array(nul, np.int32)
    cf = np.array([[complex(v).real, complex(v).imag] for v in coeffs] or [[0.0, 0.0]], np.float64)
    cap = 1 << 16
    oo = np.zeros(2, np.int64); ox = np.zeros(cap, np.uint64); oz = np.zeros(cap, np.uint64); oc = np.zeros((cap, 2))
    onull = C.c_int()
    i64, u64, dp, ip = (C.POINTER(C.c_int64), C.POINTER(C.c_uint64), C.POINTER(C.c_double), C.POINTER(C.c_int))
    st = ref.lib.liecl_ref_linear_combination_pauli(
        off.ctypes.data_as(i64), x.ctypes.data_as(u64), z.ctypes.data_as(u64), c.ctypes.data_as(dp),
        C.c_int64(len(tup)), C.c_uint(n), nul.ctypes.data_as(ip), C.c_double(complex(bc).real),
        C.c_double(complex(bc).imag), cf.ctypes.data_as(dp), oo.ctypes.data_as(i64), ox.ctypes.data_as(u64),
        oz.ctypes.data_as(u64), oc.ctypes.data_as(dp), C.c_int64(cap), C.byref(onull))
    assert st == 0
    if onull.value:
        return None
    k = int(oo[1])
    return [(int(ox[i]), int(oz[i]), oc[i, 0], oc[i, 1]) for i in range(k)]


def _mine(s):
    return None if s is None else [(t.x, t.z, c.real, c.imag) for t, c in s.terms]


def _bits(v):
    return None if v is None else [(a, b, np.float64(c).view(np.uint64), np.float64(d).view(np.uint64)) for a, b, c, d in v]


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(6))
def test_pauli_branch_bit_exact(ref_exact, seed):
    rng = np.random.default_rng(50 + seed)
    n = int(rng.integers(1, 5))
    base = _rand_sum(rng, n, int(rng.integers(1, 6)))
    tup = [_rand_sum(rng, n, int(rng.integers(1, 6))) for _ in range(int(rng.integers(0, 5)))]
    if seed % 3 == 1 and tup:
        tup[0] = None  # null entries are skipped
    coeffs = [complex(*rng.standard_normal(2)) for _ in tup]
    bc = complex(*rng.standard_normal(2))
    if seed % 3 == 2:
        base = None  # chained-addition fallback
    elif seed == 3:
        base = liecl.PauliSum(n, [])  # empty base: also the fallback
    got = liecl.linear_combination(base, bc, tup, coeffs)
    want = _ref_lc_pauli(ref_exact, base, bc, tup, coeffs, n)
    assert _bits(_mine(got)) == _bits(want)


def test_errors():
    a = liecl.PauliSum.single(liecl.PauliString(1, 0, 1), 1.0)
    with pytest.raises(liecl.InvalidInputError, match="lengths differ"):
        liecl.linear_combination(a, 1.0, [a], [])
    b = liecl.PauliSum.single(liecl.PauliString(1, 0, 2), 1.0)
    with pytest.raises(liecl.InvalidInputError):
        liecl.linear_combination(a, 1.0, [b], [1.0])


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["plain", "null_entry", "null_base", "all_null"])
def test_dense_branch_matches_reference(ref_exact, case):
    rng = np.random.default_rng(7)
    d, n = 8, 5
    mk = lambda: liecl.DenseOperator.from_vec(rng.standard_normal(d * d) + 1j * rng.standard_normal(d * d), d)
    base = mk()
    tup = [mk() for _ in range(n)]
    coeffs = [complex(*rng.standard_normal(2)) for _ in range(n)]
    bc = complex(*rng.standard_normal(2))
    if case == "null_entry":
        tup[2] = None
    if case in ("null_base", "all_null"):
        base = None
    if case == "all_null":
        tup = [None] * n
    got = liecl.linear_combination(base, bc, tup, coeffs)
    if case == "all_null":
        assert got is None
        return
    # reference: dense branch, or the chained fallback from the first non-null
    live = [(o, c) for o, c in zip(tup, coeffs) if o is not None]
    if base is None:
        b0, c0 = live[0]
        rest = live[1:]
    else:
        b0, c0, rest = base, bc, live
    T = np.stack([o.vec() for o, _ in rest]) if rest else np.zeros((1, d * d), complex)
    cf = np.array([[c.real, c.imag] for _, c in rest] or [[0.0, 0.0]])
    out = np.zeros(d * d, complex)
    dp = C.POINTER(C.c_double)
    bv = np.ascontiguousarray(b0.vec())
    assert ref_exact.lib.liecl_ref_linear_combination_dense(
        bv.ctypes.data_as(dp), C.c_double(c0.real), C.c_double(c0.imag), T.ctypes.data_as(dp), cf.ctypes.data_as(dp),
        C.c_int64(len(rest)), C.c_int(d), out.ctypes.data_as(dp)) == 0
    assert np.array_equal(got.vec().view(np.uint64), out.view(np.uint64))


@pytest.mark.gpu
def test_pauli_norm_inner_product_axpy_dot_and_helpers():
    rng = np.random.default_rng(9)
    a, b = _rand_sum(rng, 3, 5), _rand_sum(rng, 3, 5)
    ka = {(s.z, s.x): c for s, c in a.terms}
    want = sum((np.conj(ka[(s.z, s.x)]) * c for s, c in b.terms if (s.z, s.x) in ka), 0j)
    assert abs(liecl.inner_product(a, b) - want) < 1e-15
    assert liecl.inner_product(None, b) == 0 and liecl.norm(None) == 0.0
    assert abs(liecl.norm(a) - np.sqrt(sum(abs(c) ** 2 for _, c in a.terms))) < 1e-15
    assert liecl.axpy_dot([], []) is None
    with pytest.raises(liecl.InvalidInputError, match="lengths differ"):
        liecl.axpy_dot([a], [])
    assert _mine(liecl.axpy_dot([a, b], [2.0, 1j])) == _mine(liecl.linear_combination(a, 2.0, [b], [1j]))
    u = liecl.normalized(a)
    assert abs(liecl.norm(u) - 1.0) < 1e-15
    assert liecl.is_zero(None, 0.0) and not liecl.is_zero(a, 1e-3)
    with pytest.raises(liecl.InvalidInputError):
        liecl.is_zero(a, -1.0)
    with pytest.raises(liecl.InvalidInputError, match="null operator"):
        liecl.normalized(liecl.PauliSum(3, []))


@pytest.mark.gpu
def test_dense_normalized_and_axpy_dot():
    rng = np.random.default_rng(10)
    d = 4
    mk = lambda: liecl.DenseOperator.from_vec(rng.standard_normal(d * d) + 1j * rng.standard_normal(d * d), d)
    a, b = mk(), mk()
    u = liecl.normalized(a)
    assert abs(liecl.norm(u) - 1.0) < 1e-14
    s = liecl.axpy_dot([a, b], [1.5, -2j])
    assert np.allclose(s.vec(), 1.5 * a.vec() - 2j * b.vec(), rtol=0, atol=1e-13)
