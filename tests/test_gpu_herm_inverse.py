"""GramState::refresh's inverse on the device (R:src/closure.cpp:89-95, the
reference's A.ldlt().solve(I)): the hand-written blocked Gauss-Jordan
(gram_engine.cuh HermInverse, 64-wide pivot blocks on the DMMA GEMMs) on
Hermitian positive definite Gram matrices across the block edges, and its
pivoted fallback on matrices that are not positive definite. Checked against
numpy's inverse (a plain fp64 reference) and through A A^-1 = I."""
import numpy as np
import pytest

from paper_2506_01120_b200 import liecl

pytestmark = pytest.mark.gpu


def gram_of_unit_vectors(rng, n, dim):
    B = rng.standard_normal((n, dim)) + 1j * rng.standard_normal((n, dim))
    B /= np.linalg.norm(B, axis=1)[:, None]
    return B.conj() @ B.T  # A[l, m] = <b_l, b_m>, unit diagonal, Hermitian positive definite


def refresh(A):
    st = liecl.GramState(gram=A, inverse=np.zeros_like(A))
    st.refresh()
    return st.inverse


@pytest.mark.parametrize("n", [1, 2, 5, 63, 64, 65, 127, 128, 129, 300, 777])
def test_blocked_inverse_of_gram_matrices(n):
    rng = np.random.default_rng(n)
    A = gram_of_unit_vectors(rng, n, max(2 * n, 8))
    Ai = refresh(A)
    ref = np.linalg.inv(A)
    cond = np.linalg.cond(A)
    assert np.abs(Ai - ref).max() <= 1e-13 * cond * max(1.0, np.abs(ref).max())
    assert np.abs(A @ Ai - np.eye(n)).max() <= 1e-13 * cond


def test_ill_conditioned_gram_matrix():
    """Nearly dependent elements (Schur complements down to ~1e-8): the regime
    the Schur-complement refresh rule (s < 1e-4) sends here."""
    rng = np.random.default_rng(5)
    n, dim = 200, 400
    B = rng.standard_normal((n, dim)) + 1j * rng.standard_normal((n, dim))
    B[1::7] = B[0:-1:7][: len(B[1::7])] + 1e-4 * B[1::7]
    B /= np.linalg.norm(B, axis=1)[:, None]
    A = B.conj() @ B.T
    Ai = refresh(A)
    ref = np.linalg.inv(A)
    cond = np.linalg.cond(A)
    assert cond > 1e6
    assert np.abs(Ai - ref).max() <= 1e-14 * cond * np.abs(ref).max()


@pytest.mark.parametrize("n", [3, 70, 150])
def test_not_positive_definite_takes_the_pivoted_path(n):
    """An indefinite Hermitian matrix (a negative pivot) and one with a zero
    leading pivot: the reference's LDL^T still returns an inverse, so does
    the pivoted Gauss-Jordan fallback."""
    rng = np.random.default_rng(100 + n)
    H = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    H = H + H.conj().T
    for A in (H, H - np.diag(np.diag(H)) * 1.0 + np.diag(np.r_[0.0, np.ones(n - 1)])):
        Ai = refresh(A)
        ref = np.linalg.inv(A)
        cond = np.linalg.cond(A)
        assert np.abs(Ai - ref).max() <= 1e-12 * cond * np.abs(ref).max()


def test_singular_gram_matrix_raises():
    """A zero row and column: Cholesky stops at the zero diagonal and the
    pivoted path finds no pivot. (A matrix that is singular only up to
    rounding factors with a tiny positive pivot and returns a huge inverse,
    like the reference's LDL^T solve.)"""
    rng = np.random.default_rng(9)
    A = gram_of_unit_vectors(rng, 5, 16)
    A[2, :] = 0.0
    A[:, 2] = 0.0
    with pytest.raises(liecl.DegeneracyError):
        refresh(A)
    with pytest.raises(liecl.DegeneracyError):
        refresh(np.zeros((3, 3), np.complex128))
