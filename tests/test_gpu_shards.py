"""D-sharded independence check (BASELINE configs[3] "sharded
across GPUs").

On one GPU, P shards run as P threads, each with its own context, stream and
session holding a column slice of every vector; the engine's cross-rank sums
go through a host callback that adds the P partials in rank order. This is the
same engine path the NCCL reducer drives on P GPUs, with only the transport
swapped. Verdicts must equal the unsharded session's and the reference
restatement's; residual norms and the basis agree to rounding (the
partial sums regroup the additions)."""
import threading

import numpy as np
import pytest

from paper_2506_01120_b200 import liecl, native
from paper_2506_01120_b200.distributed import ShardedCheck, shard_bounds


def workload(d=16, n=40, ncand=96, seed=7):
    """Orthonormal basis (reference norm) + candidates: Gaussians, near-span
    combinations, exact zeros, and combinations of earlier candidates (in-batch
    dependence: only a re-check against in-batch accepts rejects them)."""
    rng = np.random.default_rng(seed)
    D = d * d
    G = rng.standard_normal((D, n)) + 1j * rng.standard_normal((D, n))
    Q, _ = np.linalg.qr(G)
    V = np.ascontiguousarray((Q.T * np.sqrt(d)).astype(np.complex128))
    C = np.zeros((ncand, D), np.complex128)
    for k in range(ncand):
        kind = k % 4
        if kind == 0:
            C[k] = rng.standard_normal(D) + 1j * rng.standard_normal(D)
        elif kind == 1:
            a = rng.standard_normal(n) + 1j * rng.standard_normal(n)
            C[k] = a @ V + 1e-13 * (rng.standard_normal(D) + 1j * rng.standard_normal(D))
        elif kind == 2:
            C[k] = 0.0 if k % 8 == 2 else (rng.standard_normal(n) + 1j * rng.standard_normal(n)) @ V
        else:
            C[k] = (0.5 - 2j) * C[k - 3] + 3.0 * V[k % n]  # depends on the Gaussian 3 back
    return d, V, C


class ThreadSum:
    """Sum over P threads in rank order: identical bits on every rank."""

    def __init__(self, P):
        self.P = P
        self.parts = [None] * P
        self.bar = threading.Barrier(P, timeout=120)

    def reducer(self, rank):
        def reduce(values):
            self.parts[rank] = values.copy()
            self.bar.wait()
            total = self.parts[0].copy()
            for r in range(1, self.P):
                total += self.parts[r]
            self.bar.wait()
            values[:] = total
        return reduce


def run_sharded_threads(d, V, C, P, tol=1e-10):
    sums = ThreadSum(P)
    out = [None] * P
    errs = []

    def rank_main(r):
        ctx = native.new_context(0)
        try:
            s = liecl.ClosureSession(d, config=liecl.ClosureConfig(tolerance=tol, max_dim=len(V) + len(C)), ctx=ctx)
            s.set_shards(P, r, reduce=sums.reducer(r))
            lo, hi = liecl.shard_range(d, P, r)
            assert (lo, hi) == shard_bounds(d, P, r)
            s.set_basis(np.ascontiguousarray(V[:, lo:hi]))
            ind, rn, st = s.check_candidates(np.ascontiguousarray(C[:, lo:hi]))
            out[r] = (ind, rn, st, s.basis(), lo, hi)
            s.close()
        except Exception as e:  # surfaced in the main thread
            errs.append(e)
            sums.bar.abort()
        finally:
            native.destroy_context(ctx)

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 3])
def test_sharded_check_matches_unsharded_and_port(P, port):
    d, V, C = workload()
    tol = 1e-10
    s = liecl.ClosureSession(d, config=liecl.ClosureConfig(tolerance=tol, max_dim=len(V) + len(C)))
    s.set_basis(V)
    ind0, rn0, st0 = s.check_candidates(C)
    B0 = s.basis()
    ind_p, _ = port.check_sequence_dense(V, C, d, tol=tol, append=True)[:2]
    assert np.array_equal(ind0, ind_p)
    assert 0 < ind0.sum() < len(C)
    out = run_sharded_threads(d, V, C, P, tol)
    for ind, rn, st, B, lo, hi in out:
        assert np.array_equal(ind, ind0)
        assert np.array_equal(rn, out[0][1])  # every rank, same bits
        np.testing.assert_allclose(rn, rn0, rtol=1e-11, atol=1e-14)
        assert st["accepted"] == st0["accepted"] and st["rechecks"] > 0
        np.testing.assert_allclose(B, B0[:, lo:hi], atol=1e-11)
    assert sum(o[5] - o[4] for o in out) == d * d


@pytest.mark.gpu
def test_sharded_check_nccl_single_rank():
    d, V, C = workload(seed=11)
    tol = 1e-10
    s = liecl.ClosureSession(d, config=liecl.ClosureConfig(tolerance=tol, max_dim=len(V) + len(C)))
    s.set_basis(V)
    ind0, rn0, _ = s.check_candidates(C)
    sc = ShardedCheck(d, config=liecl.ClosureConfig(tolerance=tol, max_dim=len(V) + len(C)))
    sc.set_basis(V)
    ind, rn, _ = sc.check_candidates(C)
    assert np.array_equal(ind, ind0)
    np.testing.assert_allclose(rn, rn0, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(sc.basis_slice(), s.basis(), atol=1e-12)


@pytest.mark.gpu
def test_sharded_session_refuses_commutators():
    s = liecl.ClosureSession(4)
    s.set_shards(2, 0, reduce=lambda v: None)
    rng = np.random.default_rng(0)
    s.set_basis(rng.standard_normal((3, 8)) + 0j)
    with pytest.raises(liecl.InvalidInputError, match="whole operators"):
        s.run_pairs(0, 3)
    with pytest.raises(liecl.InvalidInputError, match="fresh session"):
        s.set_shards(2, 1, reduce=lambda v: None)


@pytest.mark.gpu
def test_failed_reduction_is_reported():
    s = liecl.ClosureSession(4)
    s.set_shards(2, 0, reduce=lambda v: 1 / 0)
    with pytest.raises(liecl.Error, match="reduction"):
        s.check_candidates(np.ones((2, 8), np.complex128))
