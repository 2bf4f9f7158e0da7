"""Rank method (Alg. 1): GPU vs the reference build (all host threads)."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2506_01120_b200 import liecl
from oracle.oracle import Ref
ref = Ref()
for fam, n in (("hea", 3), ("spin_glass_hva", 3), ("spin_glass_hva", 4)):
    off, x, z, c = ref.build_generators(fam, n)
    gens = np.stack([1j * ref.from_pauli(x[off[i]:off[i+1]], z[off[i]:off[i+1]], c[off[i]:off[i+1]], n) for i in range(len(off) - 1)])
    cfg = liecl.ClosureConfig(tolerance=1e-10)
    liecl.closure_dense_arrays(gens, 1 << n, liecl.Method.standard_rank, cfg) if n == 3 else None
    t = time.perf_counter()
    r = liecl.closure_dense_arrays(gens, 1 << n, liecl.Method.standard_rank, cfg)
    g = time.perf_counter() - t
    out = {"family": fam, "n": n, "dim": r.dimension, "gpu_s": round(g, 3), "checks": r.stats.independence_checks,
           "svd_candidates": r.stats.engine.get("survivors"), "screen": os.environ.get("LIECL_B200_RANK_SCREEN", "1")}
    if n == 3:
        t = time.perf_counter()
        o = ref.closure_dense(gens, 1 << n, method="standard-rank", tol=1e-10, threads=os.cpu_count())
        out.update(ref_s=round(time.perf_counter() - t, 3), ref_dim=o.dimension, threads=os.cpu_count())
    print(json.dumps(out), flush=True)
