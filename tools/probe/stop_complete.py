"""Spin-glass n = 5 / 6 with and without stop_when_complete (the paper's rows,
BASELINE.md:31, imply an early stop)."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2506_01120_b200 import liecl, workloads as w
os.environ["LIECL_B200_TRACE"] = "1"
for n in (5, 6):
    gens = np.stack([w.vec(1j * w.from_pauli(sp)) for sp in w.spin_glass_hva(n)])
    for stop in (True, False):
        t = time.perf_counter()
        r = liecl.closure_dense_arrays(gens, 1 << n, liecl.Method.orthonorm_dimonly,
                                       liecl.ClosureConfig(tolerance=1e-10, stop_when_complete=stop))
        print(json.dumps({"n": n, "stop_when_complete": stop, "dimension": r.dimension,
                          "seconds": round(time.perf_counter() - t, 3), "brackets": r.stats.commutators_evaluated,
                          "paper_s": {5: 1.0, 6: 8.0}[n]}), flush=True)
