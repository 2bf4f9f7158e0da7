import json, os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2506_01120_b200 import liecl, workloads as w
for n in (20, 24, 28):
    off, x, z, c = w.sum_arrays(w.tfim_hva_open(n))
    t = time.perf_counter()
    r = liecl.closure_pauli_sums_arrays(off, x, z, c, n, liecl.Method.orthonorm_dimonly, liecl.ClosureConfig(tolerance=1e-10))
    print(json.dumps({"family": "tfim_hva_open", "n": n, "dim": r.dimension, "seconds": round(time.perf_counter() - t, 2),
                      "brackets": r.stats.commutators_evaluated}), flush=True)
