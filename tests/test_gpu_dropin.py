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
