"""The TMA-staged projection GEMMs (dgemm_tma.cuh, zgemm_tma.cuh) against the
cp.async kernels they replace (LIECL_B200_TMA=0), on session batches large
enough for unsplit grids: identical verdicts, residual norms to rounding.
Basis sizes n = 255, 254, 253 cover every K tail of the 5-D box (rows up to
4 ceil(n/4) are read from the zero tail of V). Needs a B200."""
import numpy as np
import pytest

from paper_2506_01120_b200 import liecl
from paper_2506_01120_b200 import workloads as w

pytestmark = pytest.mark.gpu


def su16_basis():
    gens = np.stack([w.vec(1j * w.from_pauli(sp)) for sp in w.hea(4)])
    r = liecl.closure_dense_arrays(gens, 16, liecl.Method.orthonorm, liecl.ClosureConfig(tolerance=1e-10))
    assert r.dimension == 255
    return r.ortho_array


def antiherm(rng, count, d):
    m = rng.standard_normal((count, d, d)) + 1j * rng.standard_normal((count, d, d))
    a = (m - np.conj(np.transpose(m, (0, 2, 1)))) / 2  # exactly anti-Hermitian
    a = a / np.sqrt(np.einsum("kij,kij->k", np.conj(a), a).real / d)[:, None, None]
    return np.stack([x.ravel(order="F") for x in a])


def run(V, cands, field, tma, monkeypatch):
    monkeypatch.setenv("LIECL_B200_TMA", tma)
    s = liecl.ClosureSession(16, config=liecl.ClosureConfig(tolerance=1e-10, field=field))
    s.set_basis(V)
    ind, rn, _ = s.check_candidates(cands)
    return ind, rn


@pytest.mark.parametrize("field", ["auto", "complex"])
@pytest.mark.parametrize("n", [255, 254, 253])
def test_tma_and_cpasync_gemms_agree(monkeypatch, n, field):
    V = su16_basis()[:n]
    rng = np.random.default_rng(n)
    k = 4096
    c = rng.standard_normal((k, n))
    dep = c @ V  # in the span (real coefficients keep them anti-Hermitian)
    dep = dep / np.sqrt(np.einsum("ki,ki->k", np.conj(dep), dep).real / 16)[:, None]
    cands = np.concatenate([antiherm(rng, k, 16), dep])
    ind1, rn1 = run(V, cands, field, "1", monkeypatch)
    ind0, rn0 = run(V, cands, field, "0", monkeypatch)
    assert np.array_equal(ind1, ind0)
    assert ind1.sum() == 256 - n  # random candidates complete u(16), then everything is dependent
    assert ind1[:256 - n].all()
    acc = ind1 == 1
    assert np.abs(rn1[acc] - rn0[acc]).max(initial=0.0) < 1e-10
    assert np.abs(rn1[~acc] - rn0[~acc]).max(initial=0.0) < 1e-12
    assert rn1[~acc].max(initial=0.0) < 1e-11


def test_transposed_basis_follows_appends_and_replacements(monkeypatch):
    """K2b reads VT, a transposed copy of the packed basis extended by the rows
    appended since its last use and discarded when the basis is replaced:
    batches after appends and after set_basis must equal the cp.async path."""
    V = su16_basis()
    rng = np.random.default_rng(3)
    b1 = np.concatenate([antiherm(rng, 8, 16), (rng.standard_normal((8184, 200)) @ V[:200])])
    b2 = antiherm(rng, 8192, 16)
    b3 = np.concatenate([antiherm(rng, 4, 16), (rng.standard_normal((8188, 120)) @ V[100:220])])

    def go(tma):
        monkeypatch.setenv("LIECL_B200_TMA", tma)
        s = liecl.ClosureSession(16, config=liecl.ClosureConfig(tolerance=1e-10))
        out = []
        s.set_basis(V[:200])
        out.append(s.check_candidates(b1)[:2])  # 8 accepts: rows 200..207 appended
        out.append(s.check_candidates(b2)[:2])  # VT extended by those rows first
        s.set_basis(V[100:220])                 # replaced: VT rebuilt, not reused
        out.append(s.check_candidates(b3)[:2])
        return out
    for (i1, r1), (i0, r0) in zip(go("1"), go("0")):
        assert np.array_equal(i1, i0)
        assert np.abs(r1 - r0).max() < 1e-10
