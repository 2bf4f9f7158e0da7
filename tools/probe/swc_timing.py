"""stop_when_complete closure of config 2: first call vs cached engine."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2506_01120_b200 import liecl  # noqa: E402
from paper_2506_01120_b200 import workloads as w  # noqa: E402

cfg = w.config2()
for rep in range(3):
    t0 = time.perf_counter()
    r = liecl.closure_dense_arrays(cfg.generators, 64, liecl.Method.orthonorm_dimonly,
                                   liecl.ClosureConfig(tolerance=cfg.tol, stop_when_complete=True))
    t1 = time.perf_counter()
    print("rep %d: %.3f s (engine wall %.3f s) dim %d brackets %d" % (rep, t1 - t0, r.stats.wall_seconds, r.dimension,
                                                                       r.stats.commutators_evaluated), r.stats.engine,
          flush=True)
