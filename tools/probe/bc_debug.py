"""Debug the Gram-block path: generator check of config 2 and the c1 closure."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2506_01120_b200 import liecl  # noqa: E402
from paper_2506_01120_b200 import workloads as w  # noqa: E402

cfg = w.config2()
s = liecl.ClosureSession(64, config=liecl.ClosureConfig(tolerance=cfg.tol, record_log=True))
ind, rn, st = s.check_candidates(cfg.generators)
print("gens", ind, rn, st, flush=True)
c1 = w.config1()
r = liecl.closure_dense_arrays(c1.generators, c1.d, liecl.Method.orthonorm_dimonly,
                               liecl.ClosureConfig(tolerance=c1.tol, record_log=True))
print("c1", r.dimension, r.stats, flush=True)
