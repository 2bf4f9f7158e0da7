"""The multi-GPU cursor loop over NCCL on the real engine (one rank: this
round's boxes have one GPU; world-2 coverage of the host logic is in
test_distributed_gloo.py), and bench.py launched by torchrun."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _nccl_worker(rank, port, out):
    import torch
    import torch.distributed as dist
    from paper_2506_01120_b200 import liecl, workloads as w
    from paper_2506_01120_b200.distributed import DistributedClosure, TorchComm
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=1,
                            device_id=torch.device("cuda", 0))
    cfg = w.config2()
    s = liecl.ClosureSession(64, config=liecl.ClosureConfig(tolerance=cfg.tol))
    s.check_candidates(cfg.generators)
    st = DistributedClosure(s, cfg.tol, comm=TorchComm(device=torch.device("cuda", 0)), batch_max=4096).run_rows(1, 200)
    np.savez(out, V=s.basis(), stats=np.array([st.commutators_evaluated, st.independence_checks, st.accepted,
                                               st.batches_sharded, st.batches_replicated]))
    dist.destroy_process_group()


def test_distributed_closure_over_nccl(tmp_path):
    import torch.multiprocessing as mp
    from paper_2506_01120_b200 import liecl, workloads as w
    out = str(tmp_path / "r0.npz")
    mp.spawn(_nccl_worker, args=(_free_port(), out), nprocs=1, join=True)
    got = np.load(out)
    cfg = w.config2()
    s = liecl.ClosureSession(64, config=liecl.ClosureConfig(tolerance=cfg.tol))
    s.check_candidates(cfg.generators)
    ref = s.run_rows(1, 200)
    assert got["stats"][0] == ref["commutators_evaluated"] == 200 * 199 // 2
    assert got["stats"][2] == ref["accepted"] == 4092
    assert got["stats"][3] > 0 and got["stats"][4] > 0
    V = s.basis()
    assert np.abs(got["V"] - V).max() / np.abs(V).max() < 1e-10


def test_bench_under_torchrun():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"), "--gpus", "1",
           "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-secondary", "--no-general", "--no-e2e"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["gpu_launches"] > 0


def test_bench_sharded_loop_under_torchrun():
    """bench.py's N > 1 path (the D-sharded closure loop over NCCL) at one
    rank: same windows, strong scaling, the sharded whole closure as secondary."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"), "--gpus", "1",
           "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-general", "--c2-mode", "sharded"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["scaling"] == "strong" and line["value"] > 0 and line["comm"]["allreduce_bytes_per_step"] > 0
    full = line["secondary"]["c2_full_closure_sharded"]
    assert full["dimension"] == 4095 and full["brackets"] == 8382465
    assert line["e2e"]["value"] > 0
