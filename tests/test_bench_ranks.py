"""bench.py's multi-rank bookkeeping on CPU (gloo, world size 2): per-rank
windows are disjoint rows of the saturated phase, and the whole-job count is
the SUM of per-rank counts while the time is the MAX over ranks."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_windows_disjoint_and_inside_the_saturated_phase(world):
    for step in range(6):
        spans = [bench.window_rows(step, r, world, 1024, 8) for r in range(world)]
        rows = [set(range(a, b)) for a, b in spans]
        for i in range(world):
            a, b = spans[i]
            assert 1024 <= a < b <= 4095 and b - a == 8
            for j in range(i):
                assert not rows[i] & rows[j]


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r0, r1 = bench.window_rows(0, rank, world, 1024, 8)
        mine = float(bench.brackets_in(r0, r1))
        total = bench.reduce_over_ranks(mine, "sum")
        slowest = bench.reduce_over_ranks(10.0 + rank, "max")
        out.put((rank, mine, total, slowest))
    finally:
        dist.destroy_process_group()


def test_sum_and_max_over_ranks_gloo():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    mine = [r[1] for r in res]
    assert mine[0] != mine[1]  # different rows -> different counts
    assert all(r[2] == sum(mine) for r in res)
    assert all(r[3] == 11.0 for r in res)
    assert bench.reduce_over_ranks(5.0, "sum") == 5.0  # no process group: identity
