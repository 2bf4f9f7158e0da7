"""Matrix-inversion (Alg. 2) closures: GPU vs the reference build (all host threads)."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2506_01120_b200 import liecl
from oracle.oracle import Ref
ref = Ref()
for fam, n in (("hea", 3), ("hea", 4), ("tfim_hva_open", 6)):
    off, x, z, c = ref.build_generators(fam, n)
    gens = np.stack([1j * ref.from_pauli(x[off[i]:off[i+1]], z[off[i]:off[i+1]], c[off[i]:off[i+1]], n) for i in range(len(off) - 1)])
    cfg = liecl.ClosureConfig(tolerance=1e-10)
    liecl.closure_dense_arrays(gens, 1 << n, liecl.Method.matrix_inversion, cfg)
    t = time.perf_counter()
    r = liecl.closure_dense_arrays(gens, 1 << n, liecl.Method.matrix_inversion, cfg)
    g = time.perf_counter() - t
    t = time.perf_counter()
    o = ref.closure_dense(gens, 1 << n, method="matrix-inversion", tol=1e-10, threads=os.cpu_count())
    print(json.dumps({"family": fam, "n": n, "dim": r.dimension, "ref_dim": o.dimension, "gpu_s": round(g, 3),
                      "ref_s": round(time.perf_counter() - t, 3), "threads": os.cpu_count(),
                      "engine": r.stats.engine}), flush=True)
