"""Parity of the CUDA path (through the C-ABI) with the oracle and the golden
fixtures generated from the reference. Needs a B200.

Bars (north_star): same closure dimension and accept/reject sequence as the
reference; basis elements within 1e-10 relative; Pauli path bit-exact.
"""
import numpy as np
import pytest

from paper_2506_01120_b200 import liecl, native
from paper_2506_01120_b200 import workloads as w

pytestmark = pytest.mark.gpu

VERDICT = ["l", "m", "null_cand", "independent"]
BASIS_RTOL = 1e-10


def rel_err(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


FIELDS = ["auto", "complex"]  # auto = packed anti-Hermitian path for these i*H generators


@pytest.mark.parametrize("field", FIELDS)
@pytest.mark.parametrize("make", [w.config0, w.config1], ids=["c0", "c1"])
@pytest.mark.parametrize("method", [liecl.Method.orthonorm_dimonly, liecl.Method.orthonorm],
                         ids=["dimonly", "orthonorm"])
def test_dense_closure_matches_golden(golden, make, method, field):
    cfg = make()
    meta, g = golden(f"{cfg.name}_{liecl.to_string(method)}")
    assert meta["digest"] == cfg.digest()
    res = liecl.closure_dense_arrays(cfg.generators, cfg.d, method,
                                     liecl.ClosureConfig(tolerance=cfg.tol, record_log=True, field=field))
    assert res.dimension == meta["dimension"]
    assert res.stats.commutators_evaluated == meta["stats"]["commutators_evaluated"]
    assert res.stats.independence_checks == meta["stats"]["independence_checks"]
    assert res.stats.accepted == meta["stats"]["accepted"]
    log = res.decision_log
    assert np.array_equal(log["l"], g["log_l"]) and np.array_equal(log["m"], g["log_m"])
    assert np.array_equal(log["null_cand"], g["log_null"])
    assert np.array_equal(log["independent"], g["log_indep"])  # the accept/reject sequence
    acc = g["log_indep"] == 1
    assert np.abs(log["residual_norm"][acc] - g["log_rn"][acc]).max() < 1e-12
    rej = (g["log_indep"] == 0) & (g["log_null"] == 0)
    if rej.any():
        assert log["residual_norm"][rej].max() < 1e-12
    assert rel_err(res.basis_array, g["basis"]) < BASIS_RTOL
    assert rel_err(res.ortho_array, g["ortho"]) < BASIS_RTOL
    assert res.stats.warnings == [] and meta["warnings"] == ""


@pytest.mark.parametrize("method", [liecl.Method.orthonorm_dimonly, liecl.Method.orthonorm],
                         ids=["dimonly", "orthonorm"])
def test_pauli_closure_bit_exact(golden, method):
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
    assert np.array_equal(log["l"], g["log_l"]) and np.array_equal(log["m"], g["log_m"])
    assert np.array_equal(log["null_cand"], g["log_null"])
    assert np.array_equal(log["independent"], g["log_indep"])
    assert np.array_equal(log["residual_norm"].view(np.uint64), g["log_rn_bits"])


def test_pauli_general_coefficients_bit_exact(port):
    rng = np.random.default_rng(11)
    for trial in range(6):
        n = int(rng.integers(2, 6))
        k = int(rng.integers(2, 6))
        x = rng.integers(0, 1 << n, k).astype(np.uint64)
        z = rng.integers(0, 1 << n, k).astype(np.uint64)
        coef = rng.standard_normal((k, 2))
        if trial == 0:
            x[1], z[1], coef[1] = x[0], z[0], 2.0 * coef[0]  # duplicate generator string
        for keep in (False, True):
            method = liecl.Method.orthonorm if keep else liecl.Method.orthonorm_dimonly
            res = liecl.closure_pauli_arrays(x, z, coef, n, method, liecl.ClosureConfig(tolerance=1e-10))
            o = port.closure_pauli_single(x, z, coef, n, keep_original=keep, tol=1e-10)
            assert res.dimension == o.dimension
            bx, bz, bc = res.basis_array
            assert np.array_equal(bx, o.basis[0]) and np.array_equal(bz, o.basis[1])
            assert np.array_equal(bc.view(np.uint64), o.basis[2].view(np.uint64))
            assert res.stats.independence_checks == o.stats["independence_checks"]


def test_hea_paper_dims_pauli(ref):
    for n, dim in ((2, 15), (3, 63), (4, 255), (5, 1023)):
        off, x, z, c = ref.build_generators("hea", n)
        res = liecl.closure_pauli_arrays(x, z, c, n, liecl.Method.orthonorm_dimonly,
                                         liecl.ClosureConfig(tolerance=1e-10))
        assert res.dimension == dim
        assert res.stats.commutators_evaluated == dim * (dim - 1) // 2


@pytest.mark.parametrize("d", [8, 16, 32, 64])
def test_primitives_vs_oracle(port, d):
    rng = np.random.default_rng(d)
    a = rng.standard_normal(d * d) + 1j * rng.standard_normal(d * d)
    b = rng.standard_normal(d * d) + 1j * rng.standard_normal(d * d)
    A, B = liecl.DenseOperator.from_vec(a, d), liecl.DenseOperator.from_vec(b, d)
    c = liecl.commutator(A, B).vec()
    assert rel_err(c, port.commutator_dense(a, b, d)) < 1e-13
    assert abs(liecl.inner_product(A, B) - port.inner_product_dense(a, b, d)) < 1e-12 * d
    assert abs(liecl.norm(A) - port.norm_dense(a, d)) < 1e-12
    q, _ = np.linalg.qr(rng.standard_normal((d * d, 7)) + 1j * rng.standard_normal((d * d, 7)))
    V = (q.T * np.sqrt(d)).copy()
    r, co = liecl.project_residual([liecl.DenseOperator.from_vec(v, d) for v in V], A)
    rp, cp = port.project_residual_dense(V, a, d)
    assert rel_err(r.vec(), rp) < 1e-12
    assert rel_err(np.array(co), cp) < 1e-12


def test_window_saturated_basis_all_rejects(port):
    # a saturated orthonormal basis of all traceless d x d matrices: every
    # bracket is dependent (d=8: 63 vectors)
    d = 8
    rng = np.random.default_rng(5)
    M = rng.standard_normal((d * d, d * d - 1)) + 1j * rng.standard_normal((d * d, d * d - 1))
    ident = np.eye(d).ravel(order="F")
    M -= np.outer(ident, ident.conj() @ M) / d  # remove the trace component
    q, _ = np.linalg.qr(M)
    V = (q.T * np.sqrt(d)).copy()
    s = liecl.ClosureSession(d, config=liecl.ClosureConfig(tolerance=1e-10, record_log=True))
    s.set_basis(V)
    st = s.run_rows(1, len(V))
    log = s.log()
    nul, ind, rn = port.bracket_window_dense(V, d, 1, len(V), tol=1e-10)
    assert st["commutators_evaluated"] == len(V) * (len(V) - 1) // 2 == len(log)
    assert np.array_equal(log["null_cand"], nul) and np.array_equal(log["independent"], ind)
    assert ind.sum() == 0 and s.size() == len(V)


def test_ordered_check_candidates_vs_oracle(port):
    # config-3 semantics at a size the oracle finishes in seconds:
    # N=256 orthonormal basis of D=1024 (d=32), 64 candidates, even Gaussian,
    # odd combinations + 1e-14 noise
    d, N, K = 32, 256, 64
    rng = np.random.default_rng(9)
    G = rng.standard_normal((d * d, N)) + 1j * rng.standard_normal((d * d, N))
    q, _ = np.linalg.qr(G)
    V = (q.T * np.sqrt(d)).copy()
    cands = np.empty((K, d * d), np.complex128)
    for k in range(K):
        if k % 2 == 0:
            cands[k] = rng.standard_normal(d * d) + 1j * rng.standard_normal(d * d)
        else:
            a = rng.standard_normal(N) + 1j * rng.standard_normal(N)
            cands[k] = a @ V + 1e-14 * (rng.standard_normal(d * d) + 1j * rng.standard_normal(d * d))
    s = liecl.ClosureSession(d, config=liecl.ClosureConfig(tolerance=1e-10, max_dim=N + K))
    s.set_basis(V)
    ind, rn, st = s.check_candidates(cands)
    oind, orn, room = port.check_sequence_dense(V, cands, d, tol=1e-10, append=True)
    assert np.array_equal(ind, oind)
    assert ind.sum() == K // 2
    assert np.abs(rn[ind == 1] - orn[oind == 1]).max() < 1e-12
    assert rn[ind == 0].max() < 1e-12
    assert rel_err(s.basis(), room) < BASIS_RTOL


def test_capacity_and_timeout_errors():
    cfg = w.config1()
    with pytest.raises(liecl.CapacityError):
        liecl.closure_dense_arrays(cfg.generators, cfg.d, liecl.Method.orthonorm_dimonly,
                                   liecl.ClosureConfig(tolerance=1e-10, max_dim=10))
    import time
    with pytest.raises(liecl.TimeoutError):
        liecl.closure_dense_arrays(w.config2().generators, 64, liecl.Method.orthonorm_dimonly,
                                   liecl.ClosureConfig(tolerance=1e-10, deadline=time.monotonic() + 0.5))


def test_null_generator_warning_and_kernels_launched():
    cfg = w.config0()
    gens = np.concatenate([np.zeros((1, 64), np.complex128), cfg.generators])
    k0 = native.kernel_count(0)
    res = liecl.closure_dense_arrays(gens, 8, liecl.Method.orthonorm_dimonly, liecl.ClosureConfig(tolerance=1e-10))
    assert res.dimension == 9
    assert [wr.kind for wr in res.stats.warnings] == ["null_generator"]
    assert res.stats.warnings[0].detail == "generator 0 has norm 0.000000 and was skipped"
    assert native.kernel_count(0) > k0


@pytest.mark.parametrize("field", FIELDS)
def test_c2_growth_phase_matches_reference(golden, field):
    """Config 2 (n=6, d=64): the growth phase (rows 1..99, every accept of the
    closure happens here) decision for decision against the reference's own
    run (tests/golden, generated by tests/golden/make_golden.py --c2)."""
    meta, g = golden("c2_random_sums_n6_s0_orthonorm-dimonly_rows100")
    cfg = w.config2()
    assert meta["digest"] == cfg.digest()
    s = liecl.ClosureSession(64, config=liecl.ClosureConfig(tolerance=cfg.tol, record_log=True, field=field))
    ind, rn, st = s.check_candidates(cfg.generators)
    gen = g["log_m"] < 0
    assert np.array_equal(ind, g["log_indep"][gen])
    s.run_rows(1, meta["rows"])
    log = s.log()
    pairs = ~gen
    assert s.size() == meta["dimension"] == 4095
    assert np.array_equal(log["l"], g["log_l"][pairs]) and np.array_equal(log["m"], g["log_m"][pairs])
    assert np.array_equal(log["null_cand"], g["log_null"][pairs])
    assert np.array_equal(log["independent"], g["log_indep"][pairs])  # 4092 accepts, same order
    acc = g["log_indep"][pairs] == 1
    assert np.abs(log["residual_norm"][acc] - g["log_rn"][pairs][acc]).max() < 1e-9
    V = s.basis()
    rows = g["basis_rows"]
    assert rel_err(V[rows], g["basis"]) < BASIS_RTOL
    rng = np.random.default_rng(1234)
    wts = rng.standard_normal(4096) + 1j * rng.standard_normal(4096)
    assert rel_err(V @ wts, g["basis_checksum"]) < BASIS_RTOL


@pytest.mark.parametrize("d", [2, 6, 12, 128])
def test_generic_dimensions_vs_oracle(port, d):
    # off the DMMA-templated sizes (e.g. subspace-restricted operators): the
    # generic commutator kernel + the same projection GEMMs
    rng = np.random.default_rng(d)
    a = rng.standard_normal(d * d) + 1j * rng.standard_normal(d * d)
    b = rng.standard_normal(d * d) + 1j * rng.standard_normal(d * d)
    A, B = liecl.DenseOperator.from_vec(a, d), liecl.DenseOperator.from_vec(b, d)
    assert rel_err(liecl.commutator(A, B).vec(), port.commutator_dense(a, b, d)) < 1e-13
    if d <= 12:
        gens = np.stack([a - a.reshape(d, d, order="F").conj().T.ravel(order="F"),
                         b - b.reshape(d, d, order="F").conj().T.ravel(order="F")])  # anti-Hermitian
        res = liecl.closure_dense_arrays(gens, d, liecl.Method.orthonorm_dimonly,
                                         liecl.ClosureConfig(tolerance=1e-10, record_log=True))
        o = port.closure_dense(gens, d, tol=1e-10)
        assert res.dimension == o.dimension
        assert np.array_equal(res.decision_log["independent"], o.log["independent"])
        assert rel_err(res.basis_array, o.basis) < BASIS_RTOL


def antiherm_saturated_basis(d, seed=3):
    """Orthonormal basis of the traceless anti-Hermitian d x d matrices (su(d)),
    vec layout, orthonormal under <a,b> = vdot(a,b)/d."""
    rng = np.random.default_rng(seed)
    n = d * d - 1
    mats = []
    for _ in range(n):
        a = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
        a = a - a.conj().T
        a -= np.trace(a) / d * np.eye(d)
        mats.append(a.ravel(order="F"))
    M = np.array(mats).T  # D x n, every column anti-Hermitian
    # Gram-Schmidt with the real part of the inner product keeps real
    # combinations only (the span of anti-Hermitian matrices over R)
    Q = np.zeros_like(M)
    for k in range(n):
        v = M[:, k].copy()
        for _ in range(2):
            coef = (Q[:, :k].conj().T @ v).real
            v -= Q[:, :k] @ coef
        Q[:, k] = v / np.linalg.norm(v)
    V = (Q.T * np.sqrt(d)).copy()
    for k in range(n):  # exact anti-Hermitian bits
        m = V[k].reshape(d, d, order="F")
        m = 0.5 * (m - m.conj().T)
        V[k] = m.ravel(order="F")
    return V


@pytest.mark.parametrize("field", FIELDS)
def test_window_antihermitian_saturated_basis(port, field):
    d = 8
    V = antiherm_saturated_basis(d)
    s = liecl.ClosureSession(d, config=liecl.ClosureConfig(tolerance=1e-10, record_log=True, field=field))
    s.set_basis(V)
    st = s.run_rows(1, len(V))
    log = s.log()
    nul, ind, rn = port.bracket_window_dense(V, d, 1, len(V), tol=1e-10)
    assert st["commutators_evaluated"] == len(V) * (len(V) - 1) // 2 == len(log)
    assert np.array_equal(log["null_cand"], nul) and np.array_equal(log["independent"], ind)
    assert ind.sum() == 0 and s.size() == len(V)
    assert rel_err(s.basis(), V) < 1e-15  # packed round trip is exact up to the diagonal's real part


def test_antihermitian_then_general_promotes(port):
    """A session that starts on the packed path and then receives a general
    complex candidate promotes itself (unpacking the basis)."""
    cfg = w.config0()
    rng = np.random.default_rng(2)
    s = liecl.ClosureSession(8, config=liecl.ClosureConfig(tolerance=1e-10))
    ind1, _, _ = s.check_candidates(cfg.generators)
    extra = rng.standard_normal((2, 64)) + 1j * rng.standard_normal((2, 64))
    ind2, rn2, _ = s.check_candidates(extra)
    o1, _, room = port.check_sequence_dense(np.zeros((0, 64)), np.concatenate([cfg.generators, extra]), 8,
                                            append=True)
    assert np.array_equal(np.concatenate([ind1, ind2]), o1)
    assert rel_err(s.basis(), room) < BASIS_RTOL


def test_distributed_driver_single_rank_matches_session():
    """The multi-GPU driver (screen -> all-reduce -> replicate on survivors)
    at world size 1 on the real session equals the plain engine."""
    from paper_2506_01120_b200.distributed import DistributedClosure
    cfg = w.config2()
    a = liecl.ClosureSession(64, config=liecl.ClosureConfig(tolerance=cfg.tol))
    a.check_candidates(cfg.generators)
    st = DistributedClosure(a, cfg.tol, batch_max=2048).run_rows(1, 160)
    b = liecl.ClosureSession(64, config=liecl.ClosureConfig(tolerance=cfg.tol))
    b.check_candidates(cfg.generators)
    stb = b.run_rows(1, 160)
    assert a.size() == b.size() == 4095
    assert st.commutators_evaluated == stb["commutators_evaluated"] == 160 * 159 // 2
    assert st.independence_checks == stb["independence_checks"]
    assert st.accepted == stb["accepted"] == 4092
    assert st.batches_sharded > 0 and st.batches_replicated > 0
    assert rel_err(a.basis(), b.basis()) < BASIS_RTOL


@pytest.mark.parametrize("keep", [False, True], ids=["dimonly", "orthonorm"])
def test_tiny_kernel_hands_over_to_batched_engine(ref, port, keep):
    """HEA n=4 as dense operators (d = 16, closure dimension 255): the
    device-resident small-closure kernel runs the first 128 elements, the
    batched engine the rest; verdicts must equal the oracle's throughout."""
    off, x, z, c = ref.build_generators("hea", 4)
    gens = np.stack([1j * ref.from_pauli(x[off[i]:off[i + 1]], z[off[i]:off[i + 1]], c[off[i]:off[i + 1]], 4)
                     for i in range(len(off) - 1)])
    method = liecl.Method.orthonorm if keep else liecl.Method.orthonorm_dimonly
    res = liecl.closure_dense_arrays(gens, 16, method, liecl.ClosureConfig(tolerance=1e-10, record_log=True))
    o = port.closure_dense(gens, 16, keep_original=keep, tol=1e-10, threads=8, log_cap=1 << 16)
    assert res.dimension == o.dimension == 255
    assert res.stats.commutators_evaluated == o.stats["commutators_evaluated"] == 255 * 254 // 2
    assert res.stats.independence_checks == o.stats["independence_checks"]
    assert np.array_equal(res.decision_log["independent"], o.log["independent"])
    assert np.array_equal(res.decision_log["null_cand"], o.log["null_cand"])
    assert rel_err(res.basis_array, o.basis) < BASIS_RTOL


@pytest.mark.parametrize("n", [6])
def test_sparse_hea_paper_table(port, n):
    """PAPER.md §4.2 sparse-Pauli HEA (n = 6: dimension 4095 = 4^n - 1): the
    single-string path, bit-exact against the oracle (8.4M brackets)."""
    xs = [1 << i for i in range(n)] + [0] * n + [0] * (n - 1)
    zs = [0] * n + [1 << i for i in range(n)] + [(1 << i) | (1 << (i + 1)) for i in range(n - 1)]
    coef = np.tile([1.0, 0.0], (3 * n - 1, 1))
    x, z = np.array(xs, np.uint64), np.array(zs, np.uint64)
    res = liecl.closure_pauli_arrays(x, z, coef, n, liecl.Method.orthonorm_dimonly,
                                     liecl.ClosureConfig(tolerance=1e-10))
    o = port.closure_pauli_single(x, z, coef, n, tol=1e-10, log_cap=1)
    dim = 4 ** n - 1
    assert res.dimension == o.dimension == dim
    assert res.stats.commutators_evaluated == o.stats["commutators_evaluated"] == dim * (dim - 1) // 2
    assert res.stats.independence_checks == o.stats["independence_checks"]
    bx, bz, bc = res.basis_array
    assert np.array_equal(bx, o.basis[0]) and np.array_equal(bz, o.basis[1])
    assert np.array_equal(bc.view(np.uint64), o.basis[2].view(np.uint64))


def test_prefetch_basis_matches_plain_upload():
    import torch
    cfg = w.config0()
    full = liecl.closure_dense_arrays(cfg.generators, cfg.d, liecl.Method.orthonorm_dimonly,
                                      liecl.ClosureConfig(tolerance=cfg.tol))
    B = full.basis_array
    a = torch.from_numpy(B.copy()).pin_memory()
    b = torch.from_numpy(B[::-1].copy()).pin_memory()
    s = liecl.ClosureSession(cfg.d, config=liecl.ClosureConfig(tolerance=cfg.tol))
    s.set_basis(a.data_ptr(), n=len(B))  # host pointer, plain upload
    assert np.array_equal(s.basis(), B)
    s.prefetch_basis(b.data_ptr(), len(B))  # consumed by the matching set_basis
    s.set_basis(b.data_ptr(), n=len(B))
    assert np.array_equal(s.basis(), B[::-1])
    s.prefetch_basis(a.data_ptr(), len(B))  # superseded: a different pointer is uploaded normally
    s.set_basis(B[:5])
    assert np.array_equal(s.basis(), B[:5])
    st = s.run_rows(1, 5)
    assert st["commutators_evaluated"] == 10


def test_session_accepts_host_pointers():
    # pinned host buffers passed as pointers (the e2e pattern) = numpy arrays
    import torch
    cfg = w.config1()
    full = liecl.closure_dense_arrays(cfg.generators, cfg.d, liecl.Method.orthonorm_dimonly,
                                      liecl.ClosureConfig(tolerance=cfg.tol))
    B = full.basis_array[:10]
    cands = full.basis_array[10:20] + 0.5 * full.basis_array[:10]
    s = liecl.ClosureSession(cfg.d, config=liecl.ClosureConfig(tolerance=cfg.tol))
    s.set_basis(B)
    ind_a, rn_a, _ = s.check_candidates(cands)
    hb, hc = torch.from_numpy(B.copy()).pin_memory(), torch.from_numpy(cands.copy()).pin_memory()
    s.set_basis(hb.data_ptr(), n=len(B))
    ind_b, rn_b, _ = s.check_candidates(hc.data_ptr(), n=len(cands))
    assert np.array_equal(ind_a, ind_b) and np.array_equal(rn_a, rn_b) and ind_a.sum() == 10
    with pytest.raises(liecl.InvalidInputError):
        s.check_candidates(hc.data_ptr())


def test_candidate_prefetch_matches_direct_checks():
    """prefetch_candidates: the next stream's H2D on a side stream, consumed by
    the matching check_candidates; two copies in flight (alternating pinned
    buffers) give the same verdicts and norms as direct host checks."""
    import torch
    rng = np.random.default_rng(21)
    d = 8
    D = d * d
    V = []
    while len(V) < 20:  # orthonormal (1/d inner product) complex basis
        v = rng.standard_normal(D) + 1j * rng.standard_normal(D)
        for u in V:
            v = v - (np.vdot(u, v) / d) * u
        V.append(v / np.sqrt(np.vdot(v, v).real / d))
    V = np.array(V)
    streams = []
    for s in range(4):
        c = rng.standard_normal((30, D)) + 1j * rng.standard_normal((30, D))
        c[::3] = rng.standard_normal((10, 20)) @ V  # in-span rows
        streams.append(c)
    ref = liecl.ClosureSession(d, config=liecl.ClosureConfig(tolerance=1e-10))
    ses = liecl.ClosureSession(d, config=liecl.ClosureConfig(tolerance=1e-10))
    bufs = [torch.empty((30, D), dtype=torch.complex128, pin_memory=True) for _ in range(2)]
    bufs[0].numpy()[:] = streams[0]
    for k in range(4):
        ref.set_basis(V)
        ses.set_basis(V)
        if k + 1 < 4:
            bufs[(k + 1) % 2].numpy()[:] = streams[k + 1]
            ses.prefetch_candidates(bufs[(k + 1) % 2].data_ptr(), 30)
        want = ref.check_candidates(streams[k])
        got = ses.check_candidates(bufs[k % 2].data_ptr(), n=30)
        assert np.array_equal(got[0], want[0])
        assert np.allclose(got[1], want[1], rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("make", [w.config0, w.config1], ids=["c0", "c1"])
def test_reject_norms_are_pass1_bounds(golden, make):
    """A certified reject (pass-1 residual <= tol/20) reports its pass-1 norm,
    not the reference's second-pass norm (R:src/closure.cpp:277-280): an upper
    bound of it up to O(eps), and both are far below tol."""
    cfg = make()
    method = liecl.Method.orthonorm_dimonly
    meta, g = golden(f"{cfg.name}_{liecl.to_string(method)}")
    res = liecl.closure_dense_arrays(cfg.generators, cfg.d, method,
                                     liecl.ClosureConfig(tolerance=cfg.tol, record_log=True))
    rej = (g["log_indep"] == 0) & (g["log_null"] == 0)
    assert rej.any()
    rn, ref = res.decision_log["residual_norm"][rej], g["log_rn"][rej]
    assert (rn <= cfg.tol / 20 + 1e-14).all() and (ref <= cfg.tol / 20 + 1e-14).all()
    assert (rn >= ref - 1e-14).all()
