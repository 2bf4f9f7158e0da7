"""Parity pins against the reference build for the configurations whose full
size the reference cannot finish in a test (VERDICT r01 "what's
weak" 1):

* config 3's ordered check-and-append, on exactly reproducible inputs
  (workloads.Config3Exact) against a golden the reference produced
  (tests/golden/make_golden.py --c3-golden);
* config 3 at full size: the first 64 candidates against the same 17 GB
  basis bytes, the reference build (oracle/_ref, travels with the repo) run on
  the box's host cores;
* config 2 under Alg. 3 (orthonorm, keep_original): the growth phase against
  the reference's decision log (make_golden.py --c2-orthonorm);
* a saturated config-2 window: per-pair verdicts and residual norms against
  the reference on the same basis bytes (ref_harness.cpp
  liecl_ref_bracket_window_log_dense).

Rejected candidates: the engine reports its pass-1 residual (a certified
reject, rn1 <= tol/20), the reference its CGS2 (pass-2) residual; both sit at
rounding level, so the pin is |rn_gpu - rn_ref| < 1e-13 with both <= tol/20.
"""
import os

import numpy as np
import pytest

from paper_2506_01120_b200 import liecl
from paper_2506_01120_b200 import workloads as w

pytestmark = pytest.mark.gpu

BASIS_RTOL = 1e-10


def rel_err(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def check_norms(ind, rn, ref_ind, ref_rn, tol):
    assert np.array_equal(np.asarray(ind, np.int32), np.asarray(ref_ind, np.int32))
    acc = np.asarray(ref_ind) == 1
    if acc.any():
        assert np.abs(rn[acc] - ref_rn[acc]).max() < 1e-12 * max(1.0, np.abs(ref_rn[acc]).max())
    rej = ~acc
    if rej.any():
        assert rn[rej].max() <= tol / 20 and ref_rn[rej].max() <= tol / 20
        assert np.abs(rn[rej] - ref_rn[rej]).max() < 1e-13


def test_c3_exact_ordered_check_matches_reference_golden(golden):
    c = w.Config3Exact()
    meta, g = golden(c.name)
    V, cands = c.generate_numpy()
    assert c.digest(V, cands) == meta["input_digest"], "inputs did not regenerate bit for bit"
    s = liecl.ClosureSession(c.d, config=liecl.ClosureConfig(tolerance=c.tol, max_dim=c.n + c.ncand))
    s.set_basis(V)
    ind, rn, st = s.check_candidates(cands)
    assert int(ind.sum()) == meta["accepted"] == c.ncand // 2
    assert st["independence_checks"] == c.ncand
    check_norms(ind, rn, g["independent"], g["residual_norm"], c.tol)
    assert s.size() == c.n + meta["accepted"]
    s.close()


@pytest.mark.slow
def test_c3_full_size_first_64_candidates_same_bytes_as_reference(ref):
    """Full config 3 (N = 16384, D = 65536): candidates 0..63 one at a time
    against the fixed initial basis (the reference's project_residual on 16+
    host threads, ~40 s), verdicts and residual norms."""
    import torch
    dev = torch.device("cuda", 0)
    c3 = w.Config3()
    V, cands = c3.generate(torch, dev)
    torch.cuda.synchronize(dev)  # the context's stream does not order against torch's
    k = 64
    s = liecl.ClosureSession(c3.d, config=liecl.ClosureConfig(tolerance=c3.tol, max_dim=c3.n + 1))
    ind = np.zeros(k, np.int32)
    rn = np.zeros(k)
    for j in range(k):  # fixed basis: reset before every candidate
        s.set_basis(V.data_ptr(), on_device=True, n=c3.n)
        i1, r1, _ = s.check_candidates(cands[j:j + 1].data_ptr(), on_device=True, n=1)
        ind[j], rn[j] = i1[0], r1[0]
    Vh = V.cpu().numpy()
    ch = cands[:k].cpu().numpy()
    del V, cands
    s.close()
    torch.cuda.empty_cache()
    ref_ind, ref_rn, _ = ref.check_sequence_dense(Vh, ch, c3.d, tol=c3.tol, append=False,
                                                  threads=os.cpu_count() or 1)
    assert ind[0::2].all() and not ind[1::2].any()
    check_norms(ind, rn, ref_ind, ref_rn, c3.tol)


@pytest.mark.slow
@pytest.mark.parametrize("field", ["auto", "complex"])
def test_c2_growth_phase_alg3_matches_reference(golden, field):
    """Config 2 under Alg. 3 (keep_original: the commutator basis is the
    original brackets, R:src/closure.cpp:272-303): rows 1..99 decision for
    decision against the reference's own run."""
    meta, g = golden("c2_random_sums_n6_s0_orthonorm_rows100")
    cfg = w.config2()
    assert meta["digest"] == cfg.digest()
    s = liecl.ClosureSession(64, keep_original=True,
                             config=liecl.ClosureConfig(tolerance=cfg.tol, record_log=True, field=field))
    ind, rn, st = s.check_candidates(cfg.generators)
    gen = g["log_m"] < 0
    assert np.array_equal(ind, g["log_indep"][gen])
    s.run_rows(1, meta["rows"])
    log = s.log()
    pairs = ~gen
    assert s.size() == meta["dimension"]
    assert np.array_equal(log["l"], g["log_l"][pairs]) and np.array_equal(log["m"], g["log_m"][pairs])
    assert np.array_equal(log["null_cand"], g["log_null"][pairs])
    assert np.array_equal(log["independent"], g["log_indep"][pairs])
    acc = g["log_indep"][pairs] == 1
    assert np.abs(log["residual_norm"][acc] - g["log_rn"][pairs][acc]).max() < 1e-9
    rows = g["basis_rows"]
    B = s.basis()
    O = s.basis(ortho=True)
    assert rel_err(B[rows], g["basis"]) < BASIS_RTOL
    assert rel_err(O[rows], g["ortho"]) < BASIS_RTOL
    rng = np.random.default_rng(1234)
    wts = rng.standard_normal(4096) + 1j * rng.standard_normal(4096)
    assert rel_err(B @ wts, g["basis_checksum"]) < BASIS_RTOL
    assert rel_err(O @ wts, g["ortho_checksum"]) < BASIS_RTOL
    s.close()


@pytest.mark.slow
def test_c2_saturated_window_matches_reference_same_bytes(ref):
    """A saturated config-2 window (row 2000, pairs m = 0..767) on the grown
    basis: every pair's null flag, verdict and residual norm against the
    reference on the same basis bytes."""
    cfg = w.config2()
    s = liecl.ClosureSession(64, config=liecl.ClosureConfig(tolerance=cfg.tol, record_log=True))
    s.check_candidates(cfg.generators)
    s.run_rows(1, 100)
    assert s.size() == 4095
    V = s.basis()
    row, npairs = 2000, 768
    g0 = row * (row - 1) // 2
    s.set_basis(V)
    s.run_pairs(g0, g0 + npairs)
    log = s.log()
    assert np.array_equal(log["l"], np.full(npairs, row)) and np.array_equal(log["m"], np.arange(npairs))
    nul, ind, rn = ref.bracket_window_log_dense(V, 64, row, row + 1, tol=cfg.tol, max_pairs=npairs,
                                                threads=os.cpu_count() or 1)
    assert np.array_equal(log["null_cand"], nul)
    assert not ind.any() and not log["independent"].any()
    live = nul == 0
    check_norms(log["independent"][live], log["residual_norm"][live], ind[live], rn[live], cfg.tol)
    s.close()
