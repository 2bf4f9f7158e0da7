"""Single-string Pauli closures on up to 64 qubits (128-bit string keys) and
the persistent one-CTA frontier loop. Needs a B200.

The reference keeps strings as two uint64 masks and accepts 1..64 qubits
(R:src/pauli.cpp:383-391, R:src/generators.cpp:32). Its default dimension
cap (2^q)^2 (R:src/closure.cpp:369-371, R:src/operator.cpp:42-44) overflows
from q = 32 on, so these cases pass max_dim explicitly, as a reference user
must.
"""
import numpy as np
import pytest

from paper_2506_01120_b200 import liecl
from paper_2506_01120_b200 import workloads as w

pytestmark = pytest.mark.gpu

ALL = (1 << 64) - 1


def ring_case(pos, all_ones=True, seed=5):
    """c4-style ring (X X, Y Y, Z) on the qubit positions `pos` of 64, plus Y^64
    (x = z = all ones: the empty-slot marker of the string tables)."""
    n = len(pos)
    xs, zs = [], []
    for j in range(n):
        b = (1 << pos[j]) | (1 << pos[(j + 1) % n])
        xs.append(b), zs.append(0)
    for j in range(n):
        b = (1 << pos[j]) | (1 << pos[(j + 1) % n])
        xs.append(b), zs.append(b)
    for j in range(n):
        xs.append(0), zs.append(1 << pos[j])
    if all_ones:
        xs.append(ALL), zs.append(ALL)
    coef = np.random.default_rng(seed).normal(size=(len(xs), 2))
    return np.array(xs, np.uint64), np.array(zs, np.uint64), coef


@pytest.mark.parametrize("method", [liecl.Method.orthonorm_dimonly, liecl.Method.orthonorm],
                         ids=["dimonly", "orthonorm"])
def test_64_qubit_closure_matches_reference(ref_exact, method):
    x, z, c = ring_case([0, 31, 32, 63])
    keep = method == liecl.Method.orthonorm
    r = ref_exact.decision_log_pauli(np.arange(len(x) + 1), x, z, c, 64, keep_original=keep, tol=1e-10,
                                     basis_cap=4096, term_cap=1 << 14)
    assert r.dimension == 126
    res = liecl.closure_pauli_arrays(x, z, c, 64, method,
                                     liecl.ClosureConfig(tolerance=1e-10, record_log=True, max_dim=4096))
    assert res.dimension == r.dimension
    off, rx, rz, rc = r.basis
    assert np.array_equal(off, np.arange(r.dimension + 1))  # single strings stay single strings
    bx, bz, bc = res.basis_array
    assert np.array_equal(bx, rx) and np.array_equal(bz, rz)
    assert np.array_equal(bc.view(np.uint64), rc.view(np.uint64))
    assert (bx == np.uint64(ALL)).any()  # Y^64 is in the basis (the special slot)
    log, rl = res.decision_log, r.log
    assert len(log) == len(rl)
    for k in ("l", "m", "null_cand", "independent"):
        assert np.array_equal(log[k], rl[k]), k
    assert np.array_equal(log["residual_norm"].view(np.uint64), rl["residual_norm"].view(np.uint64))


def test_embedded_ring_equals_the_10_qubit_closure():
    """Config 4's ring relabelled onto qubits spread over all 64 bit positions:
    the same algebra, so the same verdicts, dimension and coefficient bits."""
    p = w.config4()
    pos = [0, 7, 19, 31, 32, 40, 47, 55, 62, 63]

    def embed(m):
        out = 0
        for j in range(p.qubits):
            if (int(m) >> j) & 1:
                out |= 1 << pos[j]
        return out
    ex = np.array([embed(v) for v in p.x], np.uint64)
    ez = np.array([embed(v) for v in p.z], np.uint64)
    cfg = liecl.ClosureConfig(tolerance=p.tol, record_log=True, max_dim=4096)
    small = liecl.closure_pauli_arrays(p.x, p.z, p.coef, p.qubits, config=cfg)
    big = liecl.closure_pauli_arrays(ex, ez, p.coef, 64, config=cfg)
    assert small.dimension == big.dimension == 380
    sx, sz, sc = small.basis_array
    bx, bz, bc = big.basis_array
    assert np.array_equal(bx, [embed(v) for v in sx]) and np.array_equal(bz, [embed(v) for v in sz])
    assert np.array_equal(bc.view(np.uint64), sc.view(np.uint64))
    for k in ("l", "m", "null_cand", "independent"):
        assert np.array_equal(small.decision_log[k], big.decision_log[k])


@pytest.mark.parametrize("wide", ["0", "1000", "100000000"], ids=["multi_cta", "mixed", "persistent"])
@pytest.mark.parametrize("method", [liecl.Method.orthonorm_dimonly, liecl.Method.orthonorm],
                         ids=["dimonly", "orthonorm"])
def test_frontier_paths_match_golden(golden, wide, method, monkeypatch):
    """LIECL_B200_PAULI_WIDE moves the hand-over between the one-CTA frontier
    loop and the multi-CTA batches; every split gives the golden bits."""
    monkeypatch.setenv("LIECL_B200_PAULI_WIDE", wide)
    p = w.config4()
    meta, g = golden(f"{p.name}_{liecl.to_string(method)}")
    res = liecl.closure_pauli_arrays(p.x, p.z, p.coef, p.qubits, method,
                                     liecl.ClosureConfig(tolerance=p.tol, record_log=True))
    assert res.dimension == meta["dimension"] == 380
    for k in ("commutators_evaluated", "independence_checks", "accepted"):
        assert getattr(res.stats, k) == meta["stats"][k]
    bx, bz, bc = res.basis_array
    assert np.array_equal(bx, g["x"]) and np.array_equal(bz, g["z"])
    assert np.array_equal(bc.view(np.uint64), g["coef_bits"])
    log = res.decision_log
    assert np.array_equal(log["independent"], g["log_indep"])
    assert np.array_equal(log["residual_norm"].view(np.uint64), g["log_rn_bits"])


def test_frontier_grows_basis_buffers_mid_loop(port, monkeypatch):
    """HEA n=5 sparse (dim 1023) on the one-CTA loop only: the basis buffers
    start at 1024 slots and the table at 4096, so growth and relaunch happen
    inside the loop; the result equals the C restatement bit for bit."""
    monkeypatch.setenv("LIECL_B200_PAULI_WIDE", "100000000")
    n = 5
    x = np.array([1 << i for i in range(n)] + [0] * n + [0] * (n - 1), np.uint64)
    z = np.array([0] * n + [1 << i for i in range(n)] + [(1 << i) | (1 << (i + 1)) for i in range(n - 1)], np.uint64)
    c = np.tile([1.0, 0.0], (3 * n - 1, 1))
    res = liecl.closure_pauli_arrays(x, z, c, n, config=liecl.ClosureConfig(tolerance=1e-10, record_log=True))
    assert res.stats.engine["batches"] > 1
    po = port.closure_pauli_single(x, z, c, n, tol=1e-10)
    assert res.dimension == po.dimension == 1023
    bx, bz, bc = res.basis_array
    assert np.array_equal(bx, po.basis[0]) and np.array_equal(bz, po.basis[1])
    assert np.array_equal(bc.view(np.uint64), po.basis[2].view(np.uint64))


def test_capacity_error_inside_the_frontier_loop():
    p = w.config4()
    with pytest.raises(liecl.CapacityError):
        liecl.closure_pauli_arrays(p.x, p.z, p.coef, p.qubits,
                                   config=liecl.ClosureConfig(tolerance=p.tol, max_dim=200))


def test_qubit_range():
    x = np.array([1], np.uint64)
    z = np.array([0], np.uint64)
    c = np.array([[0.0, 1.0]])
    with pytest.raises(liecl.InvalidInputError):
        liecl.closure_pauli_arrays(x, z, c, 65, config=liecl.ClosureConfig(max_dim=8))
    r = liecl.closure_pauli_arrays(np.array([ALL], np.uint64), np.array([ALL], np.uint64), c, 64,
                                   config=liecl.ClosureConfig(max_dim=8))
    assert r.dimension == 1 and int(r.basis_array[0][0]) == ALL
    # max_dim = 0 on 40 qubits: no cap (the reference's d^2 default overflows)
    p = w.config4()
    r = liecl.closure_pauli_arrays(p.x << np.uint64(30), p.z << np.uint64(30), p.coef, 40,
                                   config=liecl.ClosureConfig(tolerance=p.tol))
    assert r.dimension == 380


# ---- multi-term sums on 32..63 qubits (SumEngineT<WKey>: 128-bit keys) ------

def embed_masks(a, pos):
    out = np.zeros(len(a), np.uint64)
    for i, m in enumerate(a):
        v = 0
        for j, p in enumerate(pos):
            if (int(m) >> j) & 1:
                v |= 1 << p
        out[i] = v
    return out


WIDE = [("tfim_hva_open", 4, 16, 48, [3, 31, 40, 47]), ("xxz_hva", 4, 10, 63, [0, 33, 34, 62]),
        ("spin_glass_hva", 3, 63, 40, [5, 32, 39])]


@pytest.mark.parametrize("method", [liecl.Method.orthonorm_dimonly, liecl.Method.orthonorm],
                         ids=["dimonly", "orthonorm"])
@pytest.mark.parametrize("family,n,dim,q,pos", WIDE, ids=[w_[0] for w_ in WIDE])
def test_wide_sums_match_reference(ref_exact, family, n, dim, q, pos, method):
    """The reference's catalog generators relabelled onto qubits past 31: the
    wide-key engine against the reference build, bit for bit (basis terms,
    coefficient bits, statistics, decision log residual bits)."""
    off, x, z, c = ref_exact.build_generators(family, n)
    ex, ez = embed_masks(x, pos), embed_masks(z, pos)
    keep = method == liecl.Method.orthonorm
    res = liecl.closure_pauli_sums_arrays(off, ex, ez, c, q, method,
                                          liecl.ClosureConfig(tolerance=1e-10, record_log=True, max_dim=4096))
    o = ref_exact.closure_pauli(off, ex, ez, c, q, method=liecl.to_string(method), tol=1e-10, threads=4,
                                max_dim=4096, basis_cap=4096)
    assert res.dimension == o.dimension == dim
    for k in ("commutators_evaluated", "independence_checks", "accepted"):
        assert getattr(res.stats, k) == o.stats[k], k
    bo, bx, bz, bc = res.basis_array
    ro, rx, rz, rc = o.basis
    assert np.array_equal(bo, ro) and np.array_equal(bx, rx) and np.array_equal(bz, rz)
    assert np.array_equal(bc.view(np.uint64), rc.view(np.uint64))
    assert int(max(bx.max(), bz.max())) >> 32  # genuinely past 32 bits
    lg = ref_exact.decision_log_pauli(off, ex, ez, c, q, keep_original=keep, tol=1e-10, basis_cap=4096)
    mine = res.decision_log
    assert len(mine) == len(lg.log)
    for f in ("l", "m", "null_cand", "independent"):
        assert np.array_equal(mine[f], lg.log[f]), f
    assert np.array_equal(mine["residual_norm"].view(np.uint64), lg.log["residual_norm"].view(np.uint64))


def test_wide_sums_equal_narrow_relabelled(ref_exact, monkeypatch):
    """Narrow (31-qubit) and wide keys on the same algebra: identical bits
    once relabelled; also with the fused single-CTA check switched off."""
    off, x, z, c = ref_exact.build_generators("tfim_hva_open", 6)
    pos = [1, 20, 32, 44, 50, 61]
    cfg = liecl.ClosureConfig(tolerance=1e-10, record_log=True, max_dim=4096)
    small = liecl.closure_pauli_sums_arrays(off, x, z, c, 6, config=cfg)
    for fused in ("1", "0"):
        monkeypatch.setenv("LIECL_B200_SUMS_FUSED", fused)
        big = liecl.closure_pauli_sums_arrays(off, embed_masks(x, pos), embed_masks(z, pos), c, 62, config=cfg)
        so, sx, sz, sc = small.basis_array
        bo, bx, bz, bc = big.basis_array
        assert big.dimension == small.dimension == 36
        assert np.array_equal(bo, so)
        assert np.array_equal(bx, embed_masks(sx, pos)) and np.array_equal(bz, embed_masks(sz, pos))
        assert np.array_equal(bc.view(np.uint64), sc.view(np.uint64))
        assert np.array_equal(big.decision_log["residual_norm"].view(np.uint64),
                              small.decision_log["residual_norm"].view(np.uint64))


@pytest.mark.parametrize("q,pos", [(30, [0, 7, 13, 21, 26, 29]), (31, [2, 9, 16, 23, 28, 30]), (29, [1, 5, 11, 19, 24, 28])],
                         ids=["q30", "q31", "q29"])
def test_narrow_sums_past_64_composite_bits(ref_exact, q, pos, monkeypatch):
    """Narrow 64-bit keys on 29..31 qubits: segment | marker | 2q string bits no
    longer fit one 64-bit sort word, so the merge sorts by the key and then by
    the segment (sum_engine.cuh merge, sort.cuh). Against the 6-qubit closure
    relabelled (identical bits) and, for the decisions, the reference build."""
    monkeypatch.setenv("LIECL_B200_SUMS_FUSED", "0")  # every check through the merge pipelines
    off, x, z, c = ref_exact.build_generators("tfim_hva_open", 6)
    cfg = liecl.ClosureConfig(tolerance=1e-10, record_log=True, max_dim=4096)
    small = liecl.closure_pauli_sums_arrays(off, x, z, c, 6, config=cfg)
    ex, ez = embed_masks(x, pos), embed_masks(z, pos)
    big = liecl.closure_pauli_sums_arrays(off, ex, ez, c, q, config=cfg)
    so, sx, sz, sc = small.basis_array
    bo, bx, bz, bc = big.basis_array
    assert big.dimension == small.dimension == 36
    assert np.array_equal(bo, so)
    assert np.array_equal(bx, embed_masks(sx, pos)) and np.array_equal(bz, embed_masks(sz, pos))
    assert np.array_equal(bc.view(np.uint64), sc.view(np.uint64))
    assert np.array_equal(big.decision_log["residual_norm"].view(np.uint64),
                          small.decision_log["residual_norm"].view(np.uint64))
    o = ref_exact.closure_pauli(off, ex, ez, c, q, method="orthonorm-dimonly", tol=1e-10, threads=4, max_dim=4096,
                                basis_cap=4096)
    assert o.dimension == 36
    ro, rx, rz, rc = o.basis
    assert np.array_equal(bo, ro) and np.array_equal(bx, rx) and np.array_equal(bz, rz)
    assert np.array_equal(bc.view(np.uint64), rc.view(np.uint64))


def test_wide_parse_matches_reference(ref_exact):
    """parse_pauli_sum (the reference grammar; from_terms on the device, wide
    keys) on 40 qubits against the reference build."""
    q = 40
    text = "1.5 " + "X" * 33 + "Z" + "I" * 6 + " - (0,2) " + "I" * 39 + "Y" + " + 0.25 " + "X" * 33 + "Z" + "I" * 6
    got = liecl.parse_pauli_sum(text, q)
    rx, rz, rc = ref_exact.parse_pauli_sum(text, q)
    assert [(t[0].x, t[0].z) for t in got.terms] == list(zip(map(int, rx), map(int, rz)))
    assert np.array_equal(np.array([[t[1].real, t[1].imag] for t in got.terms]).view(np.uint64), rc.view(np.uint64))
    # 64 qubits parse too; only the string Y^64 (all ones: the key marker) is refused
    got = liecl.parse_pauli_sum("1.0 " + "X" * 64 + " + 2 " + "Y" * 63 + "Z", 64)
    rx, rz, rc = ref_exact.parse_pauli_sum("1.0 " + "X" * 64 + " + 2 " + "Y" * 63 + "Z", 64)
    assert [(t[0].x, t[0].z) for t in got.terms] == list(zip(map(int, rx), map(int, rz)))
    with pytest.raises(liecl.InvalidInputError):
        liecl.parse_pauli_sum("1.0 " + "Y" * 64, 64)


def test_64_qubit_sums_match_reference(ref_exact):
    """Multi-term sums on all 64 qubits (the reference's limit, R:src/pauli.cpp:391):
    the catalog's spin-glass generators relabelled onto qubits 0, 31, 63, against
    the reference build bit for bit."""
    off, x, z, c = ref_exact.build_generators("spin_glass_hva", 3)
    pos = [0, 31, 63]
    ex, ez = embed_masks(x, pos), embed_masks(z, pos)
    res = liecl.closure_pauli_sums_arrays(off, ex, ez, c, 64, liecl.Method.orthonorm_dimonly,
                                          liecl.ClosureConfig(tolerance=1e-10, record_log=True, max_dim=4096))
    o = ref_exact.closure_pauli(off, ex, ez, c, 64, method="orthonorm-dimonly", tol=1e-10, threads=4, max_dim=4096,
                                basis_cap=4096)
    assert res.dimension == o.dimension == 63
    for k in ("commutators_evaluated", "independence_checks", "accepted"):
        assert getattr(res.stats, k) == o.stats[k], k
    bo, bx, bz, bc = res.basis_array
    ro, rx, rz, rc = o.basis
    assert np.array_equal(bo, ro) and np.array_equal(bx, rx) and np.array_equal(bz, rz)
    assert np.array_equal(bc.view(np.uint64), rc.view(np.uint64))
    assert int(bx.max()) >> 63 or int(bz.max()) >> 63  # bit 63 is in use


def test_64_qubit_sums_refuse_only_y64():
    """Y^64 is the key arrays' marker: as an input term, or as the product of a
    bracket, it raises InvalidInputError instead of giving a wrong result."""
    one = np.array([1.0, 0.0])
    off = np.array([0, 1], np.int64)
    with pytest.raises(liecl.InvalidInputError):  # an input term
        liecl.closure_pauli_sums_arrays(off, np.array([ALL], np.uint64), np.array([ALL], np.uint64), one.reshape(1, 2),
                                        64, liecl.Method.orthonorm_dimonly, liecl.ClosureConfig(max_dim=16))
    # a product: P = X on every qubit with Z on qubit 0 too (Y_0 X_1..X_63), Q = Z on qubits 1..63:
    # P Q has x = all ones, z = all ones, and they anticommute (63 positions with X against Z)
    px, pz = ALL, 1
    qx, qz = 0, ALL & ~1
    off2 = np.array([0, 1, 2], np.int64)
    with pytest.raises(liecl.InvalidInputError):
        liecl.closure_pauli_sums_arrays(off2, np.array([px, qx], np.uint64), np.array([pz, qz], np.uint64),
                                        np.array([[1.0, 0.0], [1.0, 0.0]]), 64, liecl.Method.orthonorm_dimonly,
                                        liecl.ClosureConfig(max_dim=16))
    # an anticommuting pair one qubit narrower closes normally: dimension 3
    m63 = (1 << 63) - 1
    r = liecl.closure_pauli_sums_arrays(off2, np.array([m63, 0], np.uint64), np.array([1, m63], np.uint64),
                                        np.array([[1.0, 0.0], [1.0, 0.0]]), 63, liecl.Method.orthonorm_dimonly,
                                        liecl.ClosureConfig(max_dim=16))
    assert r.dimension == 3
