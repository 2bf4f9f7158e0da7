"""c2 growth phase and the stop_when_complete closure: wall times per block
path (LIECL_B200_BLOCK_CHOL / LIECL_B200_BLOCK_GS), same basis check."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2506_01120_b200 import liecl  # noqa: E402
from paper_2506_01120_b200 import workloads as w  # noqa: E402

cfg = w.config2()
out = {}
for field in ("auto", "complex"):
    times = []
    for rep in range(3):
        s = liecl.ClosureSession(64, config=liecl.ClosureConfig(tolerance=cfg.tol, field=field))
        s.check_candidates(cfg.generators)
        t0 = time.perf_counter()
        st = s.run_rows(1, 128)
        times.append(time.perf_counter() - t0)
        V = s.basis()
        s.close()
    out[field] = (min(times), st["batches"], st["rechecks"], s and V.shape)
    print(field, "growth rows 1..127: best %.3f s" % min(times), times, st, flush=True)
t0 = time.perf_counter()
r = liecl.closure_dense_arrays(cfg.generators, 64, liecl.Method.orthonorm_dimonly,
                               liecl.ClosureConfig(tolerance=cfg.tol, stop_when_complete=True))
print("stop_when_complete closure: %.3f s dim %d" % (time.perf_counter() - t0, r.dimension), flush=True)
