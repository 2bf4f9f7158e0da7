"""Concurrent callers from Python threads: each thread gets its own device
context (include/liecl_b200.h: one context per device and caller thread), so
closures may run concurrently and give the serial results bit for bit."""
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from paper_2506_01120_b200 import liecl, native
from paper_2506_01120_b200 import workloads as w

pytestmark = pytest.mark.gpu


def _dense():
    cfg = w.config1()
    r = liecl.closure_dense_arrays(cfg.generators, cfg.d, liecl.Method.orthonorm_dimonly,
                                   liecl.ClosureConfig(tolerance=cfg.tol))
    return r.dimension, r.basis_array.tobytes()


def _pauli():
    cfg = w.config4()
    x, z, c, n = cfg.x, cfg.z, cfg.coef, cfg.qubits
    r = liecl.closure_pauli_arrays(x, z, c, n, liecl.Method.orthonorm_dimonly, liecl.ClosureConfig(tolerance=1e-10))
    return r.dimension, b"".join(np.asarray(a).tobytes() for a in r.basis_array)


def _sums():
    off, x, z, c = w.sum_arrays(w.tfim_hva_open(8))
    r = liecl.closure_pauli_sums_arrays(off, x, z, c, 8, liecl.Method.orthonorm_dimonly,
                                        liecl.ClosureConfig(tolerance=1e-10))
    return r.dimension, b"".join(np.asarray(a).tobytes() for a in r.basis_array)


@pytest.mark.parametrize("job", [_dense, _pauli, _sums])
def test_concurrent_closures_match_serial(job):
    want = job()
    with ThreadPoolExecutor(max_workers=4) as ex:
        got = list(ex.map(lambda _: job(), range(8)))
    assert all(g == want for g in got)


def test_contexts_are_per_thread():
    main = native.context(0).value
    seen = []
    t = threading.Thread(target=lambda: seen.append(native.context(0).value))
    t.start(); t.join()
    assert seen and seen[0] != main
    assert native.context(0).value == main  # stable within a thread


def test_session_keeps_its_context_alive():
    """A session created on a worker thread stays usable after that thread
    exits (the session holds its context)."""
    holder = {}

    def make():
        s = liecl.ClosureSession(4)
        X = np.array([[0, 1], [1, 0]], complex); Z = np.diag([1.0, -1.0]).astype(complex)
        b = np.stack([np.kron(X, np.eye(2)).ravel(order="F") * 1j, np.kron(Z, np.eye(2)).ravel(order="F") * 1j])
        s.set_basis(b)
        holder["s"] = s

    t = threading.Thread(target=make)
    t.start(); t.join()
    s = holder["s"]
    cand = (np.kron(np.eye(2), np.array([[0, 1], [1, 0]], complex)) * 1j).ravel(order="F")[None]
    res = s.check_candidates(cand)
    assert res is not None
