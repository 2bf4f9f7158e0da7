"""input expansion and result listings.

CPU: the Python mirror's from_terms / format_pauli_sum / format_operator
against the reference build. GPU: the device from_pauli, bit for bit."""
import numpy as np
import pytest

from paper_2506_01120_b200 import liecl
from paper_2506_01120_b200 import workloads as w


def random_sum(rng, n, k):
    # built with the host recipe (test infrastructure); liecl.pauli_sum_from_terms runs on the device
    raw = []
    for _ in range(k):
        c = complex(rng.standard_normal(), rng.standard_normal() if rng.random() < 0.5 else 0.0)
        raw.append(((int(rng.integers(0, 1 << n)), int(rng.integers(0, 1 << n))), c))
    b = w.PauliSumSpec.from_terms(n, raw)
    return liecl.PauliSum(n, [(liecl.PauliString(int(x), int(z), n), c) for x, z, c in zip(b.x, b.z, b.coef)])


def arrays(s):
    x = np.array([t[0].x for t in s.terms], np.uint64)
    z = np.array([t[0].z for t in s.terms], np.uint64)
    c = np.array([[complex(t[1]).real, complex(t[1]).imag] for t in s.terms]).reshape(-1, 2)
    return x, z, c


@pytest.mark.gpu
def test_from_terms_matches_workload_recipe():
    rng = np.random.default_rng(1)
    for _ in range(20):
        n = int(rng.integers(1, 5))
        raw = [((int(rng.integers(0, 1 << n)), int(rng.integers(0, 1 << n))), complex(*rng.standard_normal(2)))
               for _ in range(int(rng.integers(1, 8)))]
        a = liecl.pauli_sum_from_terms(n, [(liecl.PauliString(x, z, n), c) for (x, z), c in raw])
        b = w.PauliSumSpec.from_terms(n, raw)
        assert [(t[0].x, t[0].z) for t in a.terms] == list(zip(b.x, b.z))
        assert [t[1] for t in a.terms] == b.coef


def test_format_pauli_sum_matches_reference(ref):
    rng = np.random.default_rng(2)
    for _ in range(30):
        n = int(rng.integers(1, 6))
        s = random_sum(rng, n, int(rng.integers(1, 6)))
        x, z, c = arrays(s)
        assert liecl.format_pauli_sum(s) == ref.format_pauli(x, z, c, n)
    assert liecl.format_pauli_sum(liecl.PauliSum(3, [])) == "0 III"


def test_format_dense_matches_reference(ref):
    cfg = w.config0()
    for g in cfg.generators:
        op = liecl.DenseOperator.from_vec(g, cfg.d)
        assert liecl.format_operator(op) == ref.format_dense(g, cfg.d)


@pytest.mark.gpu
def test_device_from_pauli_bit_exact(ref):
    rng = np.random.default_rng(3)
    for n in (1, 2, 3, 5, 6):
        sums = [random_sum(rng, n, int(rng.integers(1, 9))) for _ in range(4)]
        dense = liecl.from_pauli(sums)
        for s, op in zip(sums, dense):
            x, z, c = arrays(s)
            assert np.array_equal(op.vec().view(np.uint64), ref.from_pauli(x, z, c, n).view(np.uint64))
    # the BASELINE generators: same bytes as the host recipe
    for cfg in (w.config0(), w.config1(), w.config2()):
        sums = [liecl.PauliSum(s.qubits, [(liecl.PauliString(x, z, s.qubits), c) for x, z, c in zip(s.x, s.z, s.coef)])
                for s in cfg.sums]
        got = np.stack([op.vec() for op in liecl.from_pauli(sums)])
        assert np.array_equal(got.view(np.uint64), cfg.generators.view(np.uint64))
    with pytest.raises(liecl.CapacityError):
        liecl.from_pauli(liecl.PauliSum(13, [(liecl.PauliString(1, 0, 13), 1.0)]))


PARSE_CASES = [
    ("1.5 XIZ - (0,2) YYI + 0.25 XIZ", 3),
    ("  -2e-3 ZZ\n+ (1e2, -3.5E+1)   XY - 1 II ", 2),
    ("3 X", 1),
    ("(0.5,0.5) IXYZ - (0.5,0.5) IXYZ + 1 ZZZZ", 4),  # an exact cancellation drops the term
    ("1e-20 XX + 1 ZZ", 2),  # below the 1e-14 relative drop floor
    ("", 2), ("   ", 2), ("1.5", 2), ("1.5XX", 2), ("1.5 XQ", 2), ("1.5 XXX", 2), ("1.5 X", 2),
    ("1 XX * 2 ZZ", 2), ("(1 2) XX", 2), ("(1,2 XX", 2), ("1..2 XX", 2), ("1 XX +", 2), ("1 XX\n - e ZZ", 2),
    ("+ 1 XX", 2), ("1 XX - - 2 ZZ", 2),
]


@pytest.mark.gpu
@pytest.mark.parametrize("text,qubits", PARSE_CASES)
def test_parse_pauli_sum_matches_reference(ref_exact, text, qubits):
    """parse_pauli_sum (R:src/pauli.cpp:230-395): the same terms, bit for bit,
    or the same ParseError (message, line, column)."""
    want = ref_exact.parse_pauli_sum(text, qubits)
    if isinstance(want[0], str):
        with pytest.raises(liecl.ParseError) as e:
            liecl.parse_pauli_sum(text, qubits)
        assert str(e.value) == want[1] and (e.value.line, e.value.column) == (want[2], want[3])
        return
    got = liecl.parse_pauli_sum(text, qubits)
    x, z, c = want
    assert [(s.x, s.z) for s, _ in got.terms] == list(zip(x.tolist(), z.tolist()))
    mine = np.array([[v.real, v.imag] for _, v in got.terms]).reshape(-1, 2)
    assert np.array_equal(mine.view(np.uint64), c.view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("family,n", [("hea", 3), ("spin_glass_hva", 4), ("xxz_hva", 4), ("tfim_hva_open", 5)])
def test_realize_generators_matches_reference(ref_exact, family, n):
    """realize_generators (R:src/generators.cpp:171-194) through the C-ABI:
    the Pauli backend term for term and bit for bit, the dense backend
    (device from_pauli) bit for bit, and the xxz zero-magnetization
    restriction (C(n, n/2) submatrix) equal to the reference's B^H A B."""
    off, x, z, c = ref_exact.build_generators(family, n)
    got = liecl.realize_generators(family, n)
    assert len(got) == len(off) - 1
    for i, s_ in enumerate(got):
        assert [(t.x, t.z) for t, _ in s_.terms] == list(zip(x[off[i]:off[i + 1]].tolist(),
                                                             z[off[i]:off[i + 1]].tolist()))
        mine = np.array([[v.real, v.imag] for _, v in s_.terms]).reshape(-1, 2)
        assert np.array_equal(mine.view(np.uint64), c[off[i]:off[i + 1]].view(np.uint64))
    dense = liecl.realize_generators(family, n, backend=liecl.Backend.dense)
    want, m = ref_exact.realize_generators_dense(family, n)
    assert m == 1 << n and all(np.array_equal(a.vec(), b) for a, b in zip(dense, want))
    if family == "xxz_hva":
        sub = liecl.realize_generators(family, n, restrict_zero_magnetization=True)
        want, m = ref_exact.realize_generators_dense(family, n, restrict=True)
        assert m == 6 and all(np.array_equal(a.vec(), b) for a, b in zip(sub, want))


def test_pauli_single_list_is_a_lazy_sequence():
    """result.basis of a single-string closure (liecl.PauliSingleList): built on
    access from the (x, z, coef) arrays, equal to the eager list of sums."""
    import numpy as np
    x = np.array([1, 2, 3], np.uint64)
    z = np.array([0, 2, 1], np.uint64)
    c = np.array([[0.0, 1.0], [0.5, -0.5], [-1.0, 0.0]])
    lst = liecl.PauliSingleList(x, z, c, 2)
    eager = [liecl.PauliSum.single(liecl.PauliString(int(x[i]), int(z[i]), 2), complex(c[i, 0], c[i, 1]))
             for i in range(3)]
    assert len(lst) == 3 and lst == eager and list(lst) == eager
    assert lst[-1] == eager[-1] and lst[0:2] == eager[0:2]
    assert liecl.format_pauli_sum(lst[1]) == liecl.format_pauli_sum(eager[1])
    try:
        lst[3]
        raise AssertionError("index past the end must raise")
    except IndexError:
        pass


def test_pauli_sum_list_is_a_lazy_sequence():
    """result.basis of a multi-term closure (liecl.PauliSumList) built on access."""
    import numpy as np
    off = np.array([0, 2, 2, 3], np.int64)
    x = np.array([1, 2, 3], np.uint64)
    z = np.array([0, 2, 1], np.uint64)
    c = np.array([[0.0, 1.0], [0.5, -0.5], [-1.0, 0.0]])
    lst = liecl.PauliSumList(off, x, z, c, 2)
    assert len(lst) == 3
    assert [len(s.terms) for s in lst] == [2, 0, 1]
    assert lst[0].terms[1] == (liecl.PauliString(2, 2, 2), complex(0.5, -0.5))
    assert lst[-1] == lst[2] and lst[0:2] == [lst[0], lst[1]]
