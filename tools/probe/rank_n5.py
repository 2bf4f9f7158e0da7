import os, sys, time
sys.path.insert(0, os.getcwd())
os.environ["LIECL_B200_TRACE"] = "1"
import numpy as np
from paper_2506_01120_b200 import liecl, workloads as w
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5
gens = np.stack([w.vec(1j * w.from_pauli(sp)) for sp in w.spin_glass_hva(n)])
t = time.perf_counter()
try:
    r = liecl.closure_dense_arrays(gens, 1 << n, liecl.Method.standard_rank,
                                   liecl.ClosureConfig(tolerance=1e-10, deadline=time.monotonic() + 120))
    print("dim", r.dimension, r.stats.engine, time.perf_counter() - t, file=sys.stderr)
except Exception as e:
    print("EXC", repr(e)[:200], time.perf_counter() - t, file=sys.stderr)
