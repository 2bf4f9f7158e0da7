import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2506_01120_b200 import liecl
from oracle.oracle import Ref
ref = Ref()
off, x, z, c = ref.build_generators("spin_glass_hva", 3)
gens = np.stack([1j * ref.from_pauli(x[off[i]:off[i+1]], z[off[i]:off[i+1]], c[off[i]:off[i+1]], 3) for i in range(len(off) - 1)])
t = time.perf_counter()
r = liecl.closure_dense_arrays(gens, 8, liecl.Method.standard_rank, liecl.ClosureConfig(tolerance=1e-10))
print(r.dimension, time.perf_counter() - t, r.stats.independence_checks, r.stats.engine)
