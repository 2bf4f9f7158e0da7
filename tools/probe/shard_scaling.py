"""Compute side of the D-sharded closure loop at P = 1, 2, 4, 8 ranks, measured
on ONE GPU: the P ranks run as threads (own context and stream each) through a
host reducer, and a turnstile lets only one rank use the device at a time, so
every rank's CUDA-event kernel totals are clean (no kernels of different ranks
overlap, none waits on another: the ranks meet on the host). Reported per P:
the slowest rank's kernel time per saturated config-2 window (commutator,
K2a, K2b, other), the bytes summed over ranks per window, and the step time a
node would see with those bytes all-reduced at an ASSUMED bus bandwidth
(a model, labelled as such: NCCL over more than one GPU cannot run here).
  python tools/probe/shard_scaling.py [steps]"""
import json, os, sys, threading, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2506_01120_b200 import liecl, native, workloads as w

STEPS = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ROW0, ROWS = 1024, int(os.environ.get("SHARD_ROWS", "64"))  # long windows: batch tails are negligible
BUSBW_GBS = 700.0  # assumed all-reduce bus bandwidth over NVLink 5 / NVSwitch (not measured here)


class Turnstile:
    """Host sums in rank order; the device belongs to one rank at a time."""

    def __init__(self, P):
        self.P, self.parts = P, [None] * P
        self.bar = threading.Barrier(P, timeout=900)
        self.device = threading.Lock()
        self.bytes = [0] * P

    def reducer(self, rank):
        def reduce(values):
            try:
                return body(values)
            except BaseException:
                import traceback
                traceback.print_exc()
                raise

        def body(values):
            self.bytes[rank] += values.nbytes
            self.parts[rank] = values.copy()
            self.device.release()  # this rank's device work up to here is done (values are on the host)
            self.bar.wait()
            total = self.parts[0].copy()
            for r in range(1, self.P):
                total += self.parts[r]
            self.bar.wait()
            values[:] = total
            self.device.acquire()
        return reduce


def run(P, cfg):
    ts = Turnstile(P)
    out, errs = [None] * P, []

    def rank_main(r):
        ts.device.acquire()
        try:
            s = liecl.ClosureSession(cfg.d, config=liecl.ClosureConfig(tolerance=cfg.tol))
            if P > 1:
                s.set_loop_shards(P, r, reduce=ts.reducer(r))
            s.check_candidates(cfg.generators)
            s.run_rows(1, 128)  # growth phase
            assert s.size() == 4095
            s.run_rows(ROW0 - ROWS, ROW0)  # warm-up window
            native.kernel_times(0)
            native.set_timing(True, 0)
            b0 = ts.bytes[r]
            t0 = time.perf_counter()
            acc = 0
            for k in range(STEPS):
                acc += s.run_rows(ROW0 + k * ROWS, ROW0 + (k + 1) * ROWS)["accepted"]
            wall = time.perf_counter() - t0
            native.set_timing(False, 0)
            out[r] = (native.kernel_times(0), ts.bytes[r] - b0, wall, acc)
            s.close()
        except Exception as e:
            errs.append(e)
            ts.bar.abort()
        finally:
            try:
                ts.device.release()
            except RuntimeError:
                pass
    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return out


def main():
    cfg = w.config2()
    brackets = sum((ROW0 + k * ROWS + i) for k in range(STEPS) for i in range(ROWS))
    base = None
    for P in [int(x) for x in os.environ.get("SHARD_RANKS", "1,2,4,8").split(",")]:
        res = run(P, cfg)
        assert all(r[3] == 0 for r in res)
        per = []
        for kt, nbytes, wall, _ in res:
            per.append({k: v["ms"] / STEPS for k, v in kt.items()})
        total = [sum(p.values()) for p in per]
        slow = int(np.argmax(total))
        kt = res[slow][0]
        gemm_ms = kt["zgemm_project"]["ms"] + kt["zgemm_subtract"]["ms"]
        gemm_tf = (kt["zgemm_project"]["flops"] + kt["zgemm_subtract"]["flops"]) / max(gemm_ms, 1e-9) / 1e9
        comm_bytes = res[0][1] / STEPS
        # ring all-reduce: 2 (P-1)/P of the payload crosses each link
        comm_ms = 0.0 if P == 1 else 2.0 * (P - 1) / P * comm_bytes / (BUSBW_GBS * 1e9) * 1e3
        compute_ms = total[slow]
        base = base or compute_ms
        line = {"ranks": P, "brackets_per_window": brackets / STEPS,
                "slowest_rank_kernel_ms_per_window": round(compute_ms, 3),
                "of_which": {k: round(v, 3) for k, v in per[slow].items()},
                "gemm_tflops_on_the_slice": round(gemm_tf, 2),
                "compute_speedup_vs_1_rank": round(base / compute_ms, 2),
                "allreduce_bytes_per_window": int(comm_bytes),
                "model": {"assumed_busbw_GBps": BUSBW_GBS, "allreduce_ms_unoverlapped": round(comm_ms, 3),
                          "brackets_per_s_if_fully_overlapped": round(brackets / STEPS / compute_ms * 1e3),
                          "brackets_per_s_if_not_overlapped": round(brackets / STEPS / (compute_ms + comm_ms) * 1e3)}}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
