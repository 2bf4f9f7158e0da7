"""Host logic of the multi-GPU closure (paper_2506_01120_b200/distributed.py)
on CPU: world_size 2 over gloo, each rank driving a numpy stand-in of the
device session with the engine's contract (screen_pairs / run_pairs). The
sharded run must reproduce the single-process run exactly: same verdicts,
same statistics, same basis."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_01120_b200 import workloads as w
from paper_2506_01120_b200.distributed import DistributedClosure, TorchComm, pair_index, split


class NumpySession:
    """numpy model of a dimension-only ClosureSession (reference semantics:
    CGS2 against the current basis, R:src/closure.cpp:142-162, 276-286)."""

    def __init__(self, d, tol):
        self.d, self.tol = d, tol
        self.V = []

    def _ip(self, a, b):
        return np.vdot(a, b) / self.d

    def _norm(self, a):
        return np.linalg.norm(a) / np.sqrt(self.d)

    def _project(self, h, passes):
        r = h.copy()
        for _ in range(passes):
            beta = [self._ip(v, r) for v in self.V]
            for b, v in zip(beta, self.V):
                r = r - b * v
        return r

    def add_generators(self, gens):
        for g in gens:
            n = self._norm(g)
            if n <= self.tol:
                continue
            r = self._project(g / n, 2)
            rn = self._norm(r)
            if rn > self.tol:
                self.V.append(r / rn)

    def size(self):
        return len(self.V)

    def _bracket(self, g):
        l = int((1 + np.sqrt(1 + 8 * g)) // 2)
        while l * (l - 1) // 2 > g:
            l -= 1
        while (l + 1) * l // 2 <= g:
            l += 1
        m = g - l * (l - 1) // 2
        A = self.V[l].reshape(self.d, self.d, order="F")
        B = self.V[m].reshape(self.d, self.d, order="F")
        return (A @ B - B @ A).ravel(order="F")

    def screen_pairs(self, g0, g1):
        nul = np.zeros(g1 - g0, np.int32)
        rn = np.zeros(g1 - g0)
        for k, g in enumerate(range(g0, g1)):
            h = self._bracket(g)
            hn = self._norm(h)
            if not hn > self.tol:
                nul[k] = 1
                continue
            rn[k] = self._norm(self._project(h / hn, 1))
        return nul, rn

    def run_pairs(self, g0, g1):
        st = {"commutators_evaluated": 0, "independence_checks": 0, "accepted": 0}
        for g in range(g0, g1):
            h = self._bracket(g)
            st["commutators_evaluated"] += 1
            hn = self._norm(h)
            if not hn > self.tol:
                continue
            st["independence_checks"] += 1
            r = self._project(h / hn, 2)
            rn = self._norm(r)
            if rn > self.tol:
                self.V.append(r / rn)
                st["accepted"] += 1
        return st


def _problem():
    cfg = w.config0()  # su-type closure, d = 8, dimension 9
    return cfg.generators, cfg.d


def _single(batch_max):
    gens, d = _problem()
    s = NumpySession(d, 1e-10)
    s.add_generators(gens)
    st = DistributedClosure(s, 1e-10, batch_max=batch_max).run_closure()
    return st, np.array(s.V)


def _worker(rank, world, port, batch_max, out_dir):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    gens, d = _problem()
    s = NumpySession(d, 1e-10)
    s.add_generators(gens)
    dc = DistributedClosure(s, 1e-10, comm=TorchComm(), batch_max=batch_max)
    st = dc.run_closure()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), V=np.array(s.V),
             stats=np.array([st.commutators_evaluated, st.independence_checks, st.accepted,
                             st.batches_sharded, st.batches_replicated]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def test_split_covers_range():
    for count in (0, 1, 7, 64, 1000):
        for world in (1, 2, 3, 8):
            parts = [split(count, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == count
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    assert pair_index(4094, 4093) == 8382464


@pytest.mark.parametrize("batch_max", [2, 16])
def test_two_ranks_match_single_process(tmp_path, batch_max):
    ref_stats, ref_V = _single(batch_max)
    assert ref_stats.accepted == 9 - 2 and ref_stats.commutators_evaluated == 36
    port = _free_port()
    mp.spawn(_worker, args=(2, port, batch_max, str(tmp_path)), nprocs=2, join=True)
    for rank in range(2):
        got = np.load(tmp_path / f"rank{rank}.npz")
        st = got["stats"]
        assert st[0] == ref_stats.commutators_evaluated
        assert st[1] == ref_stats.independence_checks
        assert st[2] == ref_stats.accepted
        assert np.array_equal(got["V"], ref_V)  # replicas identical, bit for bit
    assert got["stats"][3] > 0  # some batches were sharded (saturated tail)


# ---- D-sharded independence check (ShardedCheck / set_shards protocol) ----

def sharded_check_model(Vloc, Cloc, d, tol, reduce):
    """numpy model of the engine's D-sharded check: each rank holds column
    slices; every inner product and squared norm is a partial sum completed by
    `reduce` (in place, over ranks) -- the only cross-rank data."""
    V = [v.copy() for v in Vloc]
    ind, rns = [], []

    def gnorm(x):
        s = np.array([np.vdot(x, x).real])
        reduce(s)
        return np.sqrt(s[0]) / np.sqrt(d)

    def gproject(r):
        if not V:
            return r
        b = (np.array([np.vdot(v, r) for v in V]) / d).view(np.float64).copy()
        reduce(b)
        beta = b.view(np.complex128)
        return r - np.tensordot(beta, np.array(V), axes=1)

    for c in Cloc:
        hn = gnorm(c)
        if not hn > tol:
            ind.append(0)
            rns.append(0.0)
            continue
        r = gproject(gproject(c / hn))
        rn = gnorm(r)
        ind.append(int(rn > tol))
        rns.append(rn)
        if rn > tol:
            V.append(r / rn)
    return np.array(ind), np.array(rns), np.array(V)


def _sharded_problem():
    rng = np.random.default_rng(5)
    d, n = 4, 5
    D = d * d
    Q, _ = np.linalg.qr(rng.standard_normal((D, n)) + 1j * rng.standard_normal((D, n)))
    V = (Q.T * np.sqrt(d)).astype(np.complex128)
    C = [rng.standard_normal(D) + 1j * rng.standard_normal(D), (1 - 2j) * V[1] + V[3], np.zeros(D)]
    C.append(2.0 * C[0] - V[0])  # dependent on an in-stream accept
    C.append(rng.standard_normal(D) + 0j)
    return d, V, np.array(C)


def _sharded_worker(rank, world, port, out_dir):
    from paper_2506_01120_b200.distributed import shard_bounds
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    comm = TorchComm()
    token = comm.broadcast_bytes(bytes(range(128)) if rank == 0 else None)  # the NCCL-id handoff
    d, V, C = _sharded_problem()
    lo, hi = shard_bounds(d, world, rank)
    ind, rn, B = sharded_check_model(V[:, lo:hi], C[:, lo:hi], d, 1e-10, comm.sum_doubles)
    np.savez(os.path.join(out_dir, f"shard{rank}.npz"), ind=ind, rn=rn, B=B, lo=lo, hi=hi,
             token=np.frombuffer(token, np.uint8))
    dist.barrier()
    dist.destroy_process_group()


def test_two_d_shards_match_unsharded(tmp_path):
    d, V, C = _sharded_problem()
    ind0, rn0, B0 = sharded_check_model(V, C, d, 1e-10, lambda v: None)
    assert ind0.tolist() == [1, 0, 0, 0, 1]
    mp.spawn(_sharded_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    got = [np.load(tmp_path / f"shard{r}.npz") for r in range(2)]
    for g in got:
        assert np.array_equal(g["ind"], ind0)
        assert np.array_equal(g["rn"], got[0]["rn"])  # every rank, same bits
        np.testing.assert_allclose(g["rn"], rn0, rtol=1e-13, atol=1e-15)
        np.testing.assert_allclose(g["B"], B0[:, int(g["lo"]):int(g["hi"])], atol=1e-13)
        assert bytes(g["token"]) == bytes(range(128))
    assert int(got[0]["hi"]) == int(got[1]["lo"]) and int(got[1]["hi"]) == d * d


# ---- D-sharded closure loop (ShardedClosure / set_loop_shards protocol) ----

def loop_shard_model(gens, d, tol, lo, hi, reduce):
    """numpy model of the engine's D-sharded closure loop: whole operators on
    every rank (commutators, norms and normalisation computed locally, same
    bits everywhere); inner products and residual norms over the slice
    [lo, hi) completed by `reduce`; an accepted vector rebuilt from the
    ranks' slices by a sum. Cursor order as R:src/closure.cpp:412-460."""
    V = []

    def ip_slice(a, b):
        return np.vdot(a[lo:hi], b[lo:hi]) / d

    def project(r):
        if not V:
            return r
        b = np.array([ip_slice(v, r) for v in V]).view(np.float64).copy()
        reduce(b)
        return r - np.tensordot(b.view(np.complex128), np.array(V), axes=1)

    def rnorm(r):
        s = np.array([np.vdot(r[lo:hi], r[lo:hi]).real])
        reduce(s)
        return np.sqrt(s[0]) / np.sqrt(d)

    def check_append(h):
        r = project(project(h))
        rn = rnorm(r)
        if rn > tol:
            full = np.zeros_like(r)
            full[lo:hi] = r[lo:hi] / rn
            fv = full.view(np.float64).copy()
            reduce(fv)  # the other ranks' slices
            V.append(fv.view(np.complex128))
        return int(rn > tol)

    log = []
    for g in gens:
        n = np.linalg.norm(g) / np.sqrt(d)
        log.append(check_append(g / n) if n > tol else -1)
    l = 1
    while l < len(V):
        row_start = len(V)
        for m in range(l):
            A = V[l].reshape(d, d, order="F")
            B = V[m].reshape(d, d, order="F")
            h = (A @ B - B @ A).ravel(order="F")
            hn = np.linalg.norm(h) / np.sqrt(d)
            log.append(check_append(h / hn) if hn > tol else -1)
        assert len(V) >= row_start
        l += 1
    return np.array(log), np.array(V)


def _loop_problem():
    rng = np.random.default_rng(9)
    d = 4
    mats = []
    for _ in range(2):
        H = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
        mats.append((1j * (H + H.conj().T)).ravel(order="F"))
    return d, np.array(mats)


def _loop_worker(rank, world, port, out_dir):
    from paper_2506_01120_b200 import liecl
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    comm = TorchComm()
    d, gens = _loop_problem()
    lo, hi = liecl.loop_shard_range(d, world, rank)  # the engine's bounds (no device call)
    log, V = loop_shard_model(gens, d, 1e-10, lo, hi, comm.sum_doubles)
    np.savez(os.path.join(out_dir, f"loop{rank}.npz"), log=log, V=V, lo=lo, hi=hi)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_loop_matches_unsharded(tmp_path):
    d, gens = _loop_problem()
    log0, V0 = loop_shard_model(gens, d, 1e-10, 0, d * d, lambda v: None)
    assert len(V0) == d * d  # two random i*H generate u(4)
    mp.spawn(_loop_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    got = [np.load(tmp_path / f"loop{r}.npz") for r in range(2)]
    assert int(got[0]["lo"]) == 0 and int(got[0]["hi"]) == int(got[1]["lo"]) and int(got[1]["hi"]) == d * d
    assert int(got[0]["hi"]) % 2 == 0  # 16-byte aligned packed rows
    for g in got:
        assert np.array_equal(g["log"], log0)  # same verdict sequence
        np.testing.assert_allclose(g["V"], V0, atol=1e-12)
    assert np.array_equal(got[0]["V"].view(np.uint64), got[1]["V"].view(np.uint64))  # identical replicas
