"""The C++ drop-in: a liecl consumer (reference headers + reference pauli/dense/
operator/generators objects) linked with closure_b200.cpp instead of
R:src/closure.cpp, calling liecl::run_closure / project_residual on the GPU."""
import hashlib
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "paper_2506_01120_b200", "lib", "dropin", "liecl_dropin_demo")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def demo():
    if not os.path.exists(DEMO):
        pytest.skip("drop-in demo not built (needs the reference headers at build time)")
    out = subprocess.run([DEMO], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    res = json.loads(out.stdout)
    # the binary must come from the sources in this tree (build() runs `make dropin`)
    h = hashlib.sha256()
    for f in ("closure_b200.cpp", "dropin_demo.cpp"):
        with open(os.path.join(ROOT, "paper_2506_01120_b200", "csrc", "dropin", f), "rb") as fh:
            h.update(fh.read())
    assert res["src_sha"] == h.hexdigest()[:16], "stale drop-in demo: rebuild with `make -C paper_2506_01120_b200/csrc dropin`"
    return res


@pytest.mark.parametrize("method", ["orthonorm-dimonly", "orthonorm"])
def test_dropin_dense_closure(demo, golden, method):
    meta, g = golden(f"c0_tfim_n3_{method}")
    r = demo[f"c0_{method}"]
    assert r["dimension"] == meta["dimension"] == 9
    for k in ("commutators_evaluated", "independence_checks", "accepted"):
        assert r[k] == meta["stats"][k]
    # demo prints each basis matrix row-major by Eigen linear index = column-major vec
    basis = np.array(r["basis"]).reshape(9, -1, 2)
    basis = basis[..., 0] + 1j * basis[..., 1]
    assert np.abs(basis - g["basis"]).max() < 1e-10


def test_dropin_pauli_closure(demo, golden):
    meta, g = golden("c4_pauli_ring_n10_orthonorm-dimonly")
    r = demo["c4"]
    assert r["dimension"] == 380
    for k in ("commutators_evaluated", "independence_checks", "accepted"):
        assert r[k] == meta["stats"][k]
    s = np.array(r["strings"])
    assert np.array_equal(s[:, 0].astype(np.uint64), g["x"]) and np.array_equal(s[:, 1].astype(np.uint64), g["z"])
    coef = g["coef_bits"].view(np.float64)
    assert np.array_equal(s[:, 2:], coef)  # values equal (signed zeros may normalise)


def test_dropin_project_residual_and_errors(demo):
    pr = demo["project_residual"]
    assert pr["coeff"] == [1.0, 0.0] and pr["residual_err"] < 1e-14
    assert demo["capacity_error"] is True


def test_dropin_matrix_inversion(demo, ref):
    from paper_2506_01120_b200 import workloads as w
    cfg = w.config0()
    theirs = ref.closure_dense(cfg.generators, cfg.d, method="matrix-inversion", tol=cfg.tol)
    r = demo["c0_matrix-inversion"]
    assert r["dimension"] == theirs.dimension == 9
    assert r["commutators_evaluated"] == theirs.stats["commutators_evaluated"]
    assert r["independence_checks"] == theirs.stats["independence_checks"]
    assert r["gram_size"] == 9 and r["inverse_error"] < 1e-10


@pytest.mark.parametrize("method", ["orthonorm-dimonly", "orthonorm"])
def test_dropin_multi_term_pauli_closure(demo, ref_exact, method):
    # run_closure over multi-term sums through the drop-in: every term's
    # string and coefficient value equal to the reference build's
    off, x, z, c = ref_exact.build_generators("tfim_hva_open", 6)
    o = ref_exact.closure_pauli(off, x, z, c, 6, method=method, tol=1e-10)
    r = demo[f"tfim6_{method}"]
    assert r["dimension"] == o.dimension == 36
    for k in ("commutators_evaluated", "independence_checks", "accepted"):
        assert r[k] == o.stats[k]
    ro, rx, rz, rc = o.basis
    got = [np.array(s_) for s_ in r["sums"]]
    assert [len(s_) for s_ in got] == np.diff(ro).tolist()
    allt = np.concatenate(got)
    assert np.array_equal(allt[:, 0].astype(np.uint64), rx) and np.array_equal(allt[:, 1].astype(np.uint64), rz)
    assert np.array_equal(allt[:, 2:], rc)


def test_dropin_rank_method(demo, ref):
    # close_standard (Alg. 1) through the drop-in: same closure as the reference
    from paper_2506_01120_b200 import workloads as w
    cfg = w.config0()
    theirs = ref.closure_dense(cfg.generators, cfg.d, method="standard-rank", tol=cfg.tol)
    r = demo["c0_standard-rank"]
    assert r["dimension"] == theirs.dimension == 9
    for k in ("commutators_evaluated", "independence_checks", "accepted"):
        assert r[k] == theirs.stats[k]
    basis = np.array(r["basis"]).reshape(9, -1, 2)
    assert np.abs(basis[..., 0] + 1j * basis[..., 1] - theirs.basis).max() < 1e-10


def test_dropin_concurrent_callers(demo):
    """liecl::run_closure from four threads at once (one device context per
    calling thread): every result bit-identical to the serial run."""
    assert demo["concurrent_identical"] is True


def _sum_arrays(sums):
    offs, xs, zs, cs = [0], [], [], []
    for s_ in sums:
        for x, z, c in s_:
            xs.append(x); zs.append(z); cs.append(c)
        offs.append(len(xs))
    return (np.array(offs, np.int64), np.array(xs, np.uint64), np.array(zs, np.uint64),
            np.array(cs, np.float64).reshape(-1, 2))


def _split(off, x, z, c):
    return [[(int(x[t]), int(z[t]), (c[t, 0], c[t, 1])) for t in range(off[i], off[i + 1])]
            for i in range(len(off) - 1)]


def test_dropin_pauli_matrix_inversion(demo, ref_exact):
    """close_matrix_inversion on Pauli generators through the drop-in (single
    strings: HEA n = 3; multi-term sums: TFIM HVA n = 4) against the reference."""
    off, x, z, c = ref_exact.build_generators("hea", 3)
    o = ref_exact.closure_pauli(off, x, z, c, 3, method="matrix-inversion", tol=1e-10)
    r = demo["hea3_matrix-inversion"]
    assert r["dimension"] == o.dimension == 63 and r["gram_size"] == 63 and r["inverse_error"] == 0.0
    for k in ("commutators_evaluated", "independence_checks", "accepted"):
        assert r[k] == o.stats[k]
    off, x, z, c = ref_exact.build_generators("tfim_hva_open", 4)
    o = ref_exact.closure_pauli(off, x, z, c, 4, method="matrix-inversion", tol=1e-10)
    r = demo["tfim4_matrix-inversion"]
    assert r["dimension"] == o.dimension and r["gram_size"] == o.dimension and r["inverse_error"] < 1e-10
    for k in ("commutators_evaluated", "independence_checks", "accepted"):
        assert r[k] == o.stats[k]
    ro, rx, rz, rc = o.basis
    allt = np.concatenate([np.array(s_) for s_ in r["sums"]])
    assert np.array_equal(allt[:, 0].astype(np.uint64), rx) and np.array_equal(allt[:, 1].astype(np.uint64), rz)
    assert np.array_equal(allt[:, 2:], rc)


def test_dropin_pauli_project_residual_and_check(demo, ref_exact):
    import ctypes as C
    off, x, z, c = ref_exact.build_generators("tfim_hva_open", 4)
    gens = _split(off, x, z, c)
    o = ref_exact.closure_pauli(off, x, z, c, 4, method="orthonorm-dimonly", tol=1e-10)
    basis = _split(*o.basis)
    # h = [gens[0], basis[7]] through the reference
    ao, ax, az, ac = _sum_arrays([gens[0], basis[7]])
    cap = 1 << 12
    ho, hx, hz, hc = np.zeros(2, np.int64), np.zeros(cap, np.uint64), np.zeros(cap, np.uint64), np.zeros((cap, 2))
    i64, u64, dp = C.POINTER(C.c_int64), C.POINTER(C.c_uint64), C.POINTER(C.c_double)
    assert ref_exact.lib.liecl_ref_sum_commutator(
        ao.ctypes.data_as(i64), ax.ctypes.data_as(u64), az.ctypes.data_as(u64), ac.ctypes.data_as(dp), C.c_uint(4),
        ho.ctypes.data_as(i64), hx.ctypes.data_as(u64), hz.ctypes.data_as(u64), hc.ctypes.data_as(dp),
        C.c_int64(cap)) == 0
    h = [(int(hx[t]), int(hz[t]), (hc[t, 0], hc[t, 1])) for t in range(int(ho[1]))]
    po, px, pz, pc = _sum_arrays(basis[:6] + [h])
    (rx, rz, rcf), coeffs = ref_exact.project_residual_pauli(po, px, pz, pc, 6, 4)
    acc = 0.0
    for re, im in rcf:
        acc += re * re + im * im
    pr = demo["pauli_project_residual"]
    assert pr["terms"] == len(rx)
    assert pr["norm_bits"] == format(np.float64(np.sqrt(acc)).view(np.uint64), "016x")
    assert pr["coeff0"] == [coeffs[0].real, coeffs[0].imag]
    ck = demo["pauli_check_matrix_inversion"]
    assert ck["member_independent"] is False and abs(ck["beta2"][0] - 1.0) < 1e-14 and ck["beta2"][1] == 0.0


def test_dropin_gram_state_and_large_dense(demo):
    g = demo["gram_state"]
    assert g["schur"] == 0.75 and abs(g["inv01"] + 2.0 / 3.0) < 1e-15 and g["err"] < 1e-15
    assert demo["d128"]["dimension"] == 3


def _relabel(a, pos):
    out = np.zeros(len(a), np.uint64)
    for i, m in enumerate(a):
        v = 0
        for j, p in enumerate(pos):
            if (int(m) >> j) & 1:
                v |= 1 << p
        out[i] = v
    return out


def test_dropin_48_qubit_strings(demo, golden):
    """Config 4's ring relabelled onto 48 qubits through the C++ drop-in (the
    128-bit string keys): config 4's golden strings relabelled, same bits."""
    meta, g = golden("c4_pauli_ring_n10_orthonorm-dimonly")
    r = demo["c4_q48"]
    assert r["dimension"] == 380
    for k in ("commutators_evaluated", "independence_checks", "accepted"):
        assert r[k] == meta["stats"][k]
    pos = [0, 5, 11, 17, 23, 29, 35, 41, 44, 47]
    xs = np.array([int(t[0]) for t in r["strings"]], np.uint64)
    zs = np.array([int(t[1]) for t in r["strings"]], np.uint64)
    assert np.array_equal(xs, _relabel(g["x"], pos)) and np.array_equal(zs, _relabel(g["z"], pos))
    coef = np.array([t[2:] for t in r["strings"]])
    assert np.array_equal(coef, g["coef_bits"].view(np.float64))


def test_dropin_48_qubit_sums(demo, ref_exact):
    """The reference's TFIM-open n = 4 generators on 48 qubits through the C++
    drop-in (SumEngineT<WKey>) against the reference build on the same input."""
    off, x, z, c = ref_exact.build_generators("tfim_hva_open", 4)
    pos = [3, 31, 40, 47]
    ex, ez = _relabel(x, pos), _relabel(z, pos)
    o = ref_exact.closure_pauli(off, ex, ez, c, 48, method="orthonorm-dimonly", tol=1e-10, max_dim=4096,
                                basis_cap=4096)
    r = demo["tfim4_q48"]
    assert r["dimension"] == o.dimension == 16
    for k in ("commutators_evaluated", "independence_checks", "accepted"):
        assert r[k] == o.stats[k]
    ro, rx, rz, rc = o.basis
    allt = [t for s_ in r["sums"] for t in s_]
    assert [len(s_) for s_ in r["sums"]] == np.diff(ro).tolist()
    assert np.array_equal(np.array([int(t[0]) for t in allt], np.uint64), rx)
    assert np.array_equal(np.array([int(t[1]) for t in allt], np.uint64), rz)
    assert np.array_equal(np.array([t[2:] for t in allt]), rc)
