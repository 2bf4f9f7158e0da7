"""Wall time of single-string Pauli closures against the frontier hand-over
width LIECL_B200_PAULI_WIDE (one-CTA persistent loop below it, multi-CTA
batches above): config 4 and sparse HEA n = 5, 6, 7. Best of 5 warm calls."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2506_01120_b200 import liecl, workloads as w  # noqa: E402


def hea(n):
    x = np.array([1 << i for i in range(n)] + [0] * n + [0] * (n - 1), np.uint64)
    z = np.array([0] * n + [1 << i for i in range(n)] + [(1 << i) | (1 << (i + 1)) for i in range(n - 1)], np.uint64)
    return x, z, np.tile([1.0, 0.0], (3 * n - 1, 1)), n


def run(case, reps=5):
    x, z, c, q = case
    cfg = liecl.ClosureConfig(tolerance=1e-10, max_dim=1 << 16)
    liecl.closure_pauli_arrays(x, z, c, q, config=cfg)
    best, r = 1e30, None
    for _ in range(reps):
        t0 = time.perf_counter()
        r = liecl.closure_pauli_arrays(x, z, c, q, config=cfg)
        best = min(best, time.perf_counter() - t0)
    return {"dim": r.dimension, "wall_ms": best * 1e3, "engine_ms": r.stats.wall_seconds * 1e3,
            "kernels": r.stats.engine["kernels"], "batches": r.stats.engine["batches"]}


p = w.config4()
cases = {"c4": (p.x, p.z, p.coef, p.qubits), "hea5": hea(5), "hea6": hea(6), "hea7": hea(7)}
for wide in sys.argv[1:] or ["0", "16384", "65536", "262144", "100000000"]:
    os.environ["LIECL_B200_PAULI_WIDE"] = wide
    for name, case in cases.items():
        if name == "hea7" and wide == "100000000":
            continue
        print(json.dumps({"wide": int(wide), "case": name, **run(case)}), flush=True)
