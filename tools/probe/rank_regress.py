import os, sys, time
sys.path.insert(0, os.getcwd())
os.environ["LIECL_B200_TRACE"] = "1"
import numpy as np
from paper_2506_01120_b200 import liecl, workloads as w
for fam, n in (("hea", 4), ("spin_glass_hva", 4), ("tfim_hva_open", 8)):
    gens = np.stack([w.vec(1j * w.from_pauli(sp)) for sp in getattr(w, fam)(n)])
    for rep in range(2):
        t = time.perf_counter()
        r = liecl.closure_dense_arrays(gens, 1 << n, liecl.Method.standard_rank, liecl.ClosureConfig(tolerance=1e-10))
        print(fam, n, "rep", rep, "dim", r.dimension, "s %.3f" % (time.perf_counter() - t), r.stats.engine, file=sys.stderr, flush=True)
