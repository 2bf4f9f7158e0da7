"""Multi-GPU closure: one process per GPU.

`ShardedClosure` (the north star's layout) D-shards the closure
loop: every rank keeps whole operators and forms every commutator itself
(identical bits), the projection GEMMs -- 95 % of the work -- run on 1/P of
the elements of every vector, and the engine sums the partial overlaps beta,
the partial squared residual norms and each accepted vector's slices over the
ranks with NCCL. One batch of B candidates against n basis vectors moves
8 n B (packed field) + 8 B bytes per pass; every rank then takes the same
verdicts in cursor order, so the result equals the single-GPU run whatever P
(tests/test_gpu_loop_shards.py). A per-batch digest all-reduce turns any rank
divergence into an error.

`DistributedClosure` below is the alternative the survey asked to measure
beside it: basis replicated, candidates sharded.

The reference has no distributed execution; this is the B200
scale-out of its cursor loop (R:src/closure.cpp:412-460). Every rank holds the
whole basis (config 2: 268 MB; config 3: 19 GB -- both fit one B200), and each
device batch of cursor pairs is split into contiguous slices, one per rank:

  1. every rank *screens* its slice on its own GPU (commutator + first
     projection pass, `ClosureSession.screen_pairs`): per pair a null flag and
     the pass-1 residual norm;
  2. one all-reduce (sum) of the batch's survivor count, a survivor being a
     non-null pair with rn1 > tol/20 (the engine's certified-reject screen);
  3. no survivors -- the saturated phase, >99.9 % of config 2's brackets --
     means every verdict of the batch is a certified reject: the batch is done
     on every rank, nothing else crosses NVLink;
  4. survivors -- the growth phase -- every rank runs the batch through the
     single-GPU ordered apply (`run_pairs`): deterministic kernels on identical
     inputs, so all replicas accept the same candidates and append identical
     vectors in cursor order.

Verdicts, statistics and the final basis therefore equal the single-GPU run,
whatever the rank count. The collective is one 8-byte all-reduce per batch
(plus an all-gather of the per-pair verdict data when a decision log is
requested).

Config 3 (an independence check over a fixed basis, no commutators) is
sharded the other way, `ShardedCheck`: along D. Each rank holds a contiguous
slice of every vector (16384 x 65536 complex: 17 GB, 2.1 GB per rank at 8),
the projection GEMMs yield partial overlaps, and the engine sums beta and the
squared residual norms over ranks in place through NCCL (one all-reduce of
16 n B bytes per pass over a batch of B candidates against n vectors), so
every rank takes the same verdicts and appends its slice of the same vectors.
The closure loop cannot shard this way: a commutator needs whole operators.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def pair_index(l: int, m: int) -> int:
    return l * (l - 1) // 2 + m


def split(count: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of `count` items for `rank` (balanced)."""
    base, extra = divmod(count, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class _Solo:
    """Communicator stand-in for world_size 1 (no torch.distributed)."""
    rank, world = 0, 1

    def sum_int(self, x: int) -> int:
        return int(x)

    def gather_objects(self, obj):
        return [obj]

    def broadcast_bytes(self, data):
        return data

    def sum_doubles(self, values) -> None:
        pass


class TorchComm:
    """torch.distributed collectives (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group, self.device = torch, dist, group, device
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def sum_int(self, x: int) -> int:
        t = self.torch.tensor([int(x)], dtype=self.torch.int64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return int(t.item())

    def gather_objects(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def sum_doubles(self, values) -> None:
        """In-place sum over ranks of a float64 numpy array (identical bits on
        every rank); usable as ClosureSession.set_shards(reduce=...) where no
        NCCL communicator is wanted."""
        t = self.torch.from_numpy(np.ascontiguousarray(values)).to(self.device or "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        values[:] = t.cpu().numpy()

    def broadcast_bytes(self, data):
        """rank 0's `data` on every rank"""
        box = [data if self.rank == 0 else None]
        self.dist.broadcast_object_list(box, src=0, group=self.group)
        return box[0]


@dataclass
class DistStats:
    commutators_evaluated: int = 0
    independence_checks: int = 0
    accepted: int = 0
    batches_sharded: int = 0
    batches_replicated: int = 0
    log: list = field(default_factory=list)


class DistributedClosure:
    """Sharded cursor loop over a replicated basis.

    `session` exposes size(), screen_pairs(g0, g1) -> (null, rn1) and
    run_pairs(g0, g1) -> stats dict (liecl.ClosureSession does); `comm` exposes
    rank, world, sum_int and gather_objects (TorchComm, or None for one rank).
    """

    def __init__(self, session, tol: float, comm=None, batch_max: int = 8192, record: bool = False):
        self.s = session
        self.tol = tol
        self.screen = tol / 20.0
        self.comm = comm or _Solo()
        self.batch_max = batch_max * self.comm.world
        self.batch = min(512 * self.comm.world, self.batch_max)
        self.record = record
        self.stats = DistStats()

    def _batch(self, g0: int, cnt: int) -> int:
        """One batch of pairs [g0, g0+cnt); returns the number accepted."""
        lo, hi = split(cnt, self.comm.rank, self.comm.world)
        nul, rn = self.s.screen_pairs(g0 + lo, g0 + hi)
        survivors = int(np.count_nonzero((nul == 0) & (rn > self.screen)))
        if self.comm.sum_int(survivors) == 0:
            nonnull = self.comm.sum_int(int(np.count_nonzero(nul == 0)))
            self.stats.commutators_evaluated += cnt
            self.stats.independence_checks += nonnull
            self.stats.batches_sharded += 1
            if self.record:
                parts = self.comm.gather_objects((nul.tolist(), rn.tolist()))
                g = g0
                for pn, pr in parts:
                    for k, (n_, r_) in enumerate(zip(pn, pr)):
                        self.stats.log.append((g + k, int(n_), 0, float(r_) if not n_ else 0.0))
                    g += len(pn)
            return 0
        st = self.s.run_pairs(g0, g0 + cnt)  # every rank, identical inputs and kernels
        self.stats.commutators_evaluated += st["commutators_evaluated"]
        self.stats.independence_checks += st["independence_checks"]
        self.stats.accepted += st["accepted"]
        self.stats.batches_replicated += 1
        if self.record and hasattr(self.s, "log"):
            for rec in self.s.log():
                g = pair_index(int(rec["l"]), int(rec["m"]))
                self.stats.log.append((g, int(rec["null_cand"]), int(rec["independent"]),
                                       float(rec["residual_norm"])))
        return st["accepted"]

    def _adapt(self, acc: int, cnt: int) -> None:
        if acc == 0:
            self.batch = min(2 * self.batch, self.batch_max)
        elif acc * 4 > cnt:
            self.batch = max(64, self.batch // 2)

    def run_pairs(self, g_begin: int, g_end: int) -> DistStats:
        g = g_begin
        while g < g_end:
            nb = self.s.size()
            avail = nb * (nb - 1) // 2
            if g >= avail:
                raise ValueError(f"cursor pair {g} refers to a basis element that does not exist yet")
            cnt = min(self.batch, avail - g, g_end - g)
            self._adapt(self._batch(g, cnt), cnt)
            g += cnt
        return self.stats

    def run_rows(self, row_begin: int, row_end: int) -> DistStats:
        return self.run_pairs(pair_index(max(row_begin, 1), 0), pair_index(max(row_end, 1), 0))

    def run_closure(self) -> DistStats:
        """All cursor pairs until the basis stops growing (after the generator loop)."""
        g = 0
        while True:
            nb = self.s.size()
            avail = nb * (nb - 1) // 2
            if g >= avail:
                return self.stats
            cnt = min(self.batch, avail - g)
            self._adapt(self._batch(g, cnt), cnt)
            g += cnt


class ShardedClosure:
    """The D-sharded closure loop over the ranks of `comm` (one process per
    GPU). Every rank passes the same FULL generators; NCCL carries the
    engine's cross-rank sums (an id from rank 0, broadcast through `comm`),
    or `reduce` (an in-place float64 sum over ranks, e.g. TorchComm over gloo
    for tests on one device). Results are identical on every rank."""

    def __init__(self, d: int, keep_original: bool = False, config=None, comm=None, device: int = 0,
                 nccl_id: bytes | None = None, reduce=None):
        from . import liecl
        self.comm = comm or _Solo()
        self.d = d
        self.session = liecl.ClosureSession(d, keep_original=keep_original, config=config, device=device)
        self.lo, self.hi = liecl.loop_shard_range(d, self.comm.world, self.comm.rank)
        if reduce is None and nccl_id is None:
            nccl_id = self.comm.broadcast_bytes(liecl.nccl_unique_id() if self.comm.rank == 0 else None)
        self.session.set_loop_shards(self.comm.world, self.comm.rank, nccl_id=nccl_id, reduce=reduce)

    def run_closure(self, gens) -> dict:
        return self.session.run_closure(gens)

    def set_basis(self, V):
        self.session.set_basis(V)

    def run_rows(self, row_begin: int, row_end: int) -> dict:
        return self.session.run_rows(row_begin, row_end)

    def basis(self):
        return self.session.basis()

    def close(self):
        self.session.close()


def shard_bounds(d: int, world: int, rank: int) -> tuple[int, int]:
    """Elements [lo, hi) of a d*d operator held by D-shard `rank` (the engine's
    shard_range, csrc/shard.cuh): floor(D r / P) .. floor(D (r+1) / P)."""
    D = d * d
    return D * rank // world, D * (rank + 1) // world


class ShardedCheck:
    """Config-3 independence check, D-sharded over the ranks of `comm`.

    Every rank passes the FULL-width basis / candidates (host arrays or torch
    tensors, (n, d*d)); only the rank's column slice [lo, hi) is handed to the
    engine. Verdicts and residual norms come back identical on every rank;
    `basis_slice()` is this rank's slice of the resulting basis.
    """

    def __init__(self, d: int, config=None, comm=None, device: int = 0, nccl_id: bytes | None = None):
        from . import liecl
        self.comm = comm or _Solo()
        self.d = d
        self.lo, self.hi = shard_bounds(d, self.comm.world, self.comm.rank)
        self.session = liecl.ClosureSession(d, config=config, device=device)
        if nccl_id is None:
            nccl_id = self.comm.broadcast_bytes(liecl.nccl_unique_id() if self.comm.rank == 0 else None)
        self.session.set_shards(self.comm.world, self.comm.rank, nccl_id=nccl_id)

    def local(self, X):
        """This rank's contiguous column slice of full-width rows."""
        return X[:, self.lo:self.hi]

    def set_basis(self, V):
        import numpy as _np
        if isinstance(V, _np.ndarray):
            self.session.set_basis(_np.ascontiguousarray(self.local(V)))
        else:  # torch tensor on this rank's device
            loc = self.local(V).contiguous()
            self.session.set_basis(loc.data_ptr(), on_device=True, n=loc.shape[0])
            return loc

    def check_candidates(self, C):
        import numpy as _np
        if isinstance(C, _np.ndarray):
            return self.session.check_candidates(_np.ascontiguousarray(self.local(C)))
        loc = self.local(C).contiguous()
        return self.session.check_candidates(loc.data_ptr(), on_device=True, n=loc.shape[0])

    def basis_slice(self):
        return self.session.basis()
