import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2506_01120_b200 import liecl, workloads as w
n = 8
gens = np.stack([w.vec(1j * w.from_pauli(sp)) for sp in w.xxz_hva(n)])
for field in sys.argv[1:] or ["auto"]:
    t = time.perf_counter()
    try:
        r = liecl.closure_dense_arrays(gens, 1 << n, liecl.Method.orthonorm_dimonly,
                                       liecl.ClosureConfig(tolerance=1e-10, field=field, max_dim=2000, record_log=False,
                                                           deadline=time.monotonic() + 150))
        print(field, os.environ.get("LIECL_B200_LARGE_COMM_MIN_D", "128"), "dim", r.dimension, "warnings", len(r.stats.warnings),
              r.stats.commutators_evaluated, round(time.perf_counter() - t, 2), flush=True)
    except Exception as e:
        print(field, os.environ.get("LIECL_B200_LARGE_COMM_MIN_D", "128"), "EXC", repr(e)[:120], round(time.perf_counter() - t, 2), flush=True)
