"""Soak of the D-sharded closure loop: random anti-Hermitian generators at
d = 64 (column-sharded brackets at P = 2, 4, 8; whole brackets at P = 3, 5),
d = 32 and d = 16, both orthonormal methods, P thread ranks on one GPU through
the host reducer, against the single-GPU session: same verdict sequence,
basis within 1e-10 (orthonormal vectors: 1e-13 / the smallest accepted
residual norm), bit-identical replicas.
  python tools/probe/shard_soak.py [seed] [cases]"""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from paper_2506_01120_b200 import liecl
from test_gpu_loop_shards import run_threads

SEED = int(sys.argv[1]) if len(sys.argv) > 1 else 1
CASES = int(sys.argv[2]) if len(sys.argv) > 2 else 12
rng = np.random.default_rng(SEED)


def random_ah(d, k):
    m = rng.standard_normal((k, d, d)) + 1j * rng.standard_normal((k, d, d))
    return np.stack([(a - a.conj().T).ravel(order="F") for a in m])


fails, done = [], []
t0 = time.time()
for case in range(CASES):
    d = int(rng.choice([16, 32, 64, 64, 64]))
    P = int(rng.choice([2, 3, 4, 5, 8]))
    keep = bool(rng.integers(0, 2))
    rows = int(rng.integers(8, 40)) if d == 64 else int(rng.integers(20, 120))
    gens = random_ah(d, int(rng.integers(2, 4)))
    cfg = liecl.ClosureConfig(tolerance=1e-10, record_log=True)

    def job(s):
        s.check_candidates(gens)
        st = s.run_rows(1, rows)
        return st, s.log(), s.basis(), s.basis(ortho=True)
    try:
        out, sums = run_threads(P, d, job, keep=keep)
        one = liecl.ClosureSession(d, keep_original=keep, config=cfg)
        st1, log1, B1, O1 = job(one)
        one.close()
        for st, log, B, O in out:
            assert st["dimension"] == st1["dimension"], ("dimension", st["dimension"], st1["dimension"])
            if not np.array_equal(log["independent"], log1["independent"]):
                k = int(np.argmax(log["independent"] != log1["independent"]))
                raise AssertionError(("verdict", k, int(log["l"][k]), int(log["m"][k]), float(log["residual_norm"][k]),
                                      float(log1["residual_norm"][k])))
            assert np.array_equal(log["null_cand"], log1["null_cand"]), "null flags"
            assert np.abs(B - B1).max() < 1e-10, ("basis", float(np.abs(B - B1).max()))
            # an accepted residual of norm rn is normalised by 1/rn: rounding differences between the
            # sharded and the whole sums (~1e-15) show up in that orthonormal vector amplified by 1/rn
            acc = log1["residual_norm"][log1["independent"] == 1]
            tol_o = max(1e-10, 1e-13 / max(float(acc.min()) if len(acc) else 1.0, 1e-10))
            assert np.abs(O - O1).max() < tol_o, ("ortho", float(np.abs(O - O1).max()), tol_o)
        for r in range(1, P):
            assert np.array_equal(out[0][2].view(np.uint64), out[r][2].view(np.uint64)), ("replica basis", r)
            assert np.array_equal(out[0][3].view(np.uint64), out[r][3].view(np.uint64)), ("replica ortho", r)
        done.append({"d": d, "P": P, "keep": keep, "rows": rows, "dim": st1["dimension"]})
    except Exception as e:  # keep going: report every failure
        fails.append({"case": case, "d": d, "P": P, "keep": keep, "rows": rows, "error": repr(e)[:300]})
print(json.dumps({"seed": SEED, "cases": CASES, "passed": len(done), "failures": fails, "seconds": round(time.time() - t0, 1),
                  "shapes": done}))
