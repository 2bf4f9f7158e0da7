"""The D-sharded closure loop (north star: "basis rows sharded per
GPU, only partial overlap sums all-reduced, the ordered accept/append stays
ordered so the result matches the reference exactly").

On one GPU, P ranks run as P threads (each with its own context and stream)
or as P processes over gloo, every rank with whole operators and projections
over its element slice; the engine's cross-rank sums go through a host
callback instead of NCCL (NCCL refuses two ranks on one device). The kernels
of different ranks never wait on each other: the ranks meet on the host.
Verdicts, statistics and the basis must equal the single-GPU run and the
reference golden fixtures."""
import os
import threading

import numpy as np
import pytest

from paper_2506_01120_b200 import liecl, native
from paper_2506_01120_b200 import workloads as w

pytestmark = pytest.mark.gpu


class ThreadSum:
    """Sum over P threads in rank order: identical bits on every rank."""

    def __init__(self, P):
        self.P = P
        self.parts = [None] * P
        self.bar = threading.Barrier(P, timeout=300)
        self.calls = [0] * P

    def reducer(self, rank):
        def reduce(values):
            self.calls[rank] += 1
            self.parts[rank] = values.copy()
            self.bar.wait()
            total = self.parts[0].copy()
            for r in range(1, self.P):
                total += self.parts[r]
            self.bar.wait()
            values[:] = total
        return reduce


def run_threads(P, d, job, keep=False, field="auto", tol=1e-10):
    sums = ThreadSum(P)
    out = [None] * P
    errs = []

    def rank_main(r):
        ctx = native.new_context(0)
        try:
            cfg = liecl.ClosureConfig(tolerance=tol, record_log=True, field=field)
            s = liecl.ClosureSession(d, keep_original=keep, config=cfg, ctx=ctx)
            s.set_loop_shards(P, r, reduce=sums.reducer(r))
            out[r] = job(s)
            s.close()
        except Exception as e:  # surfaced in the main thread
            errs.append(e)
            sums.bar.abort()
        finally:
            native.destroy_context(ctx)
    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return out, sums


def closure_job(gens):
    def job(s):
        st = s.run_closure(gens)
        return st, s.log(), s.basis(), s.basis(ortho=True), [wr.kind for wr in s.warnings()]
    return job


def test_loop_shard_ranges_partition_and_align():
    for d in (2, 8, 32, 64, 256):
        D = d * d
        for P in range(1, 9):
            b = [liecl.loop_shard_range(d, P, r) for r in range(P)]
            assert b[0][0] == 0 and b[-1][1] == D
            assert all(x[1] == y[0] for x, y in zip(b, b[1:]))
            assert all(lo % 2 == 0 for lo, _ in b)  # 16-byte aligned packed rows
            if D // P >= 256:  # wide slices sit on the GEMM tiles: every bound within half a tile of D r / P
                assert all(lo % 128 == 0 for lo, _ in b)
                assert max(hi - lo for lo, hi in b) <= D / P + 128


@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("field", ["auto", "complex"])
@pytest.mark.parametrize("method", ["orthonorm-dimonly", "orthonorm"])
def test_sharded_closure_matches_single_gpu_and_golden(golden, P, field, method):
    cfg = w.config1()
    keep = method == "orthonorm"
    meta, g = golden(f"{cfg.name}_{method}")
    one = liecl.closure_dense_arrays(cfg.generators, cfg.d, liecl.method_from_string(method),
                                     liecl.ClosureConfig(tolerance=cfg.tol, record_log=True, field=field))
    out, sums = run_threads(P, cfg.d, closure_job(cfg.generators), keep=keep, field=field)
    for st, log, B, O, warns in out:
        assert st["dimension"] == one.dimension == meta["dimension"]
        for k in ("commutators_evaluated", "independence_checks", "accepted"):
            assert st[k] == meta["stats"][k]
        assert np.array_equal(log["l"], g["log_l"]) and np.array_equal(log["m"], g["log_m"])
        assert np.array_equal(log["independent"], g["log_indep"])  # the reference's accept sequence
        assert np.abs(B - one.basis_array).max() < 1e-12
        assert np.abs(O - one.ortho_array).max() < 1e-12
        assert warns == []
    # every rank holds the same bits
    for st, log, B, O, _ in out[1:]:
        assert np.array_equal(B.view(np.uint64), out[0][2].view(np.uint64))
        assert np.array_equal(log["residual_norm"].view(np.uint64), out[0][1]["residual_norm"].view(np.uint64))
    assert min(sums.calls) > 0 and len(set(sums.calls)) == 1  # same collective sequence on every rank


@pytest.mark.slow
def test_sharded_c2_growth_phase_matches_golden(golden):
    """Config 2 (d = 64, packed field) rows 1..99 -- all 4092 loop accepts --
    with P = 2 shards, decision for decision against the reference."""
    meta, g = golden("c2_random_sums_n6_s0_orthonorm-dimonly_rows100")
    cfg = w.config2()

    def job(s):
        ind, rn, _ = s.check_candidates(cfg.generators)
        s.run_rows(1, meta["rows"])
        return ind, s.log(), s.size(), s.field()
    out, _ = run_threads(2, 64, job)
    gen = g["log_m"] < 0
    for ind, log, n, field in out:
        assert field == "antihermitian_packed"
        assert n == 4095
        assert np.array_equal(ind, g["log_indep"][gen])
        assert np.array_equal(log["independent"], g["log_indep"][~gen])
        acc = g["log_indep"][~gen] == 1
        assert np.abs(log["residual_norm"][acc] - g["log_rn"][~gen][acc]).max() < 1e-9


def _gloo_rank(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2506_01120_b200.distributed import ShardedClosure, TorchComm
        comm = TorchComm()
        cfg = w.config1()
        sc = ShardedClosure(cfg.d, config=liecl.ClosureConfig(tolerance=cfg.tol, record_log=True), comm=comm,
                            reduce=comm.sum_doubles)
        st = sc.run_closure(cfg.generators)
        q.put((rank, st["dimension"], st["commutators_evaluated"], st["independence_checks"],
               sc.session.log()["independent"].tolist(), sc.basis().view(np.uint64).tobytes()))
        sc.close()
        dist.destroy_process_group()
    except Exception as e:  # reported to the parent
        q.put((rank, "error", repr(e)))


def test_two_processes_over_gloo_match_golden(golden):
    """The real engine in two processes on one GPU, cross-rank sums over gloo
    (TorchComm.sum_doubles as the session's reduce callback)."""
    import multiprocessing as mp
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_gloo_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=600) for _ in ps], key=lambda t: t[0])
    for p in ps:
        p.join(timeout=60)
    for r in res:
        assert r[1] != "error", r
    cfg = w.config1()
    meta, g = golden(f"{cfg.name}_orthonorm-dimonly")
    for _, dim, comms, checks, indep, basis in res:
        assert dim == meta["dimension"]
        assert comms == meta["stats"]["commutators_evaluated"] and checks == meta["stats"]["independence_checks"]
        assert indep == g["log_indep"].tolist()
    assert res[0][5] == res[1][5]  # bit-identical replicas


@pytest.mark.parametrize("chunks", ["1", "4"])
def test_sharded_saturated_window_chunked_reductions(chunks, monkeypatch):
    """A saturated-window batch of 8,192 pairs on P = 2 thread ranks: with
    LIECL_B200_SHARD_CHUNKS = 4 the partial overlaps are reduced chunk by chunk
    on a side stream while the next chunks' GEMMs run; verdicts and norms equal
    the unsharded session's (and the unchunked sharded run's)."""
    from bench import random_saturated_basis
    monkeypatch.setenv("LIECL_B200_SHARD_CHUNKS", chunks)
    V = random_saturated_basis(64, 0)
    d = 64
    rows = (1024, 1032)  # ~8,200 pairs: full 8,192-pair batches

    def job(s):
        s.set_basis(V)
        st = s.run_rows(*rows)
        return st, s.log()
    out, sums = run_threads(2, d, job)
    solo = liecl.ClosureSession(d, config=liecl.ClosureConfig(tolerance=1e-10, record_log=True))
    solo.set_basis(V)
    st0 = solo.run_rows(*rows)
    log0 = solo.log()
    for st, log in out:
        assert st["accepted"] == st0["accepted"] == 0
        assert np.array_equal(log["independent"], log0["independent"])
        assert np.abs(log["residual_norm"] - log0["residual_norm"]).max() < 1e-12
    assert sums.calls[0] == sums.calls[1]


@pytest.mark.parametrize("P", [2, 4, 8])
def test_sharded_commutator_columns(P, monkeypatch):
    """d = 64 with slices on whole tile columns (P = 2, 4, 8): each rank forms
    only its columns of every bracket (commutator_ah_cols_kernel) and the
    brackets' norms are summed over ranks. Verdicts and residual norms equal
    the unsharded session's and the whole-operator kernel's
    (LIECL_B200_SHARD_COMM=0) on a saturated window; one more reduction per
    batch than with whole operators."""
    from bench import random_saturated_basis
    V = random_saturated_basis(64, 0)
    rows = (1024, 1028)

    def job(s):
        s.set_basis(V)
        st = s.run_rows(*rows)
        return st, s.log(), s.comm_bytes()
    out, sums = run_threads(P, 64, job)
    monkeypatch.setenv("LIECL_B200_SHARD_COMM", "0")
    # the gate is read once per process: compare against the unsharded session instead of a second sharded run
    solo = liecl.ClosureSession(64, config=liecl.ClosureConfig(tolerance=1e-10, record_log=True))
    solo.set_basis(V)
    st0 = solo.run_rows(*rows)
    log0 = solo.log()
    for st, log, _ in out:
        assert st["accepted"] == st0["accepted"] == 0
        assert st["commutators_evaluated"] == st0["commutators_evaluated"]
        assert np.array_equal(log["null_cand"], log0["null_cand"])
        assert np.array_equal(log["independent"], log0["independent"])
        assert np.abs(log["residual_norm"] - log0["residual_norm"]).max() < 1e-12
    assert len(set(sums.calls)) == 1  # every rank made the same reductions
    assert len({o[2] for o in out}) == 1


@pytest.mark.slow
@pytest.mark.parametrize("method", ["orthonorm-dimonly", "orthonorm"])
def test_sharded_commutator_columns_growth_phase(golden, method):
    """Config 2's growth phase (all 4092 loop accepts) on P = 4 ranks with
    column-sharded brackets, Alg. 4 and Alg. 3 (the accepted brackets' slices
    are summed into whole originals): the reference's accept sequence, the
    basis of the single-GPU run to 1e-11."""
    meta, g = golden(f"c2_random_sums_n6_s0_{method}_rows100")
    cfg = w.config2()
    keep = method == "orthonorm"

    def job(s):
        ind, rn, _ = s.check_candidates(cfg.generators)
        s.run_rows(1, meta["rows"])
        return ind, s.log(), s.size(), s.basis()
    out, _ = run_threads(4, 64, job, keep=keep)
    one = liecl.ClosureSession(64, keep_original=keep, config=liecl.ClosureConfig(tolerance=cfg.tol, record_log=True))
    one.check_candidates(cfg.generators)
    one.run_rows(1, meta["rows"])
    B1 = one.basis()
    gen = g["log_m"] < 0
    for ind, log, n, B in out:
        assert n == 4095
        assert np.array_equal(ind, g["log_indep"][gen])
        assert np.array_equal(log["independent"], g["log_indep"][~gen])
        assert np.abs(B - B1).max() < 1e-11
    assert np.array_equal(out[0][3].view(np.uint64), out[3][3].view(np.uint64))  # identical replicas
