"""Rounding-sensitivity of a dense closure (TEST INFRASTRUCTURE: used only by
tests/ and tools/probe; never by the product path).

The reference's verdict for a candidate is `residual_norm > tol`
(R:proj/core/src/closure.cpp:277-280). For some inputs that comparison is
decided by rounding rather than by the algebra, and then any two correct
implementations - the reference built with and without FMA contraction, the
C restatement, the GPU path - may legitimately disagree:

  * a residual lands within 10x of tol: the reference's own
    "borderline_residual" warning (closure.cpp:325-336);
  * error amplification: an accepted residual rho is normalised by 1/rho
    (closure.cpp:283), so the new basis vector carries ~eps/rho of rounding
    error; a later bracket h of norm |h| is normalised by 1/|h|
    (closure.cpp:419-421), so its residual carries ~eps_basis/|h| of noise.
    When that a-priori noise reaches tol/10 the verdict is a coin toss;
  * Alg. 2: the Gram system A x = beta amplifies rounding by cond(A)
    (closure.cpp:109-130), and the Schur complement 1 - beta^H A^{-1} beta
    (closure.cpp:44-53) cannot resolve residual^2 below ~eps.

`sensitivity()` walks the reference's decision log with the reference's own
basis and reports the largest a-priori noise-to-tolerance ratio, so the
differential tests can compare verdicts exactly where they are defined and
fall back to the reference's error contract elsewhere.
"""
from __future__ import annotations

import numpy as np

EPS = np.finfo(np.float64).eps


def dense_sensitivity(log, basis, d: int, tol: float) -> dict:
    """Walk a reference decision log (orthonormal methods; DECISION_DTYPE) over
    the commutator basis `basis` ((n, d*d) vec layout, the reference's own
    output). Returns {"band": residuals within 10x of tol, "noise_ratio":
    max a-priori residual noise / tol, "sensitive": bool}."""
    B = [np.asarray(b).reshape(d, d, order="F") for b in basis]
    # error carried by the basis: each accepted residual rho adds eps / rho
    basis_err = EPS * d
    worst, band = 0.0, 0
    for e in log:
        r = float(e["residual_norm"])
        if not e["null_cand"] and tol / 10 <= r <= 10 * tol:
            band += 1
        l, m = int(e["l"]), int(e["m"])
        if l >= 0 and m >= 0 and l < len(B) and m < len(B) and not e["null_cand"]:
            h = B[l] @ B[m] - B[m] @ B[l]
            hn = np.linalg.norm(h) / np.sqrt(d)
            if hn > 0:
                worst = max(worst, basis_err * d / hn / tol)
        if e["independent"] and r > 0:
            basis_err = max(basis_err, EPS * d / r + basis_err / r * EPS * d)
    return {"band": band, "noise_ratio": worst, "sensitive": band > 0 or worst > 0.1}


def gram_sensitivity(basis, d: int, tol: float) -> dict:
    """Alg. 2: rounding noise of a dependent residual ~ eps * cond(A) * d."""
    if len(basis) == 0:
        return {"cond": 1.0, "noise_ratio": 0.0, "sensitive": False}
    V = np.asarray(basis).reshape(len(basis), d * d)
    A = V.conj() @ V.T / d
    ev = np.linalg.eigvalsh(A)
    cond = float(ev.max() / max(ev.min(), 1e-300))
    ratio = EPS * cond * d / tol
    return {"cond": cond, "noise_ratio": ratio, "sensitive": ratio > 0.1}
