import os, sys
sys.path.insert(0, os.getcwd())
os.environ["LIECL_B200_TRACE"] = "1"
import numpy as np
from paper_2506_01120_b200 import liecl, workloads as w
gens = np.stack([w.vec(1j * w.from_pauli(sp)) for sp in w.spin_glass_hva(4)])
r = liecl.closure_dense_arrays(gens, 16, liecl.Method.standard_rank, liecl.ClosureConfig(tolerance=1e-10))
print("dim", r.dimension, r.stats.engine, file=sys.stderr)
