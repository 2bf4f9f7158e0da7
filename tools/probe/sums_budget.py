import json, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2506_01120_b200 import liecl, workloads as w
for n in (20, 24, 28):
    off, x, z, c = w.sum_arrays(w.tfim_hva_open(n))
    base = None
    for b in (1 << 24, 1 << 26, 1 << 27):
        t = time.perf_counter()
        r = liecl.closure_pauli_sums_arrays(off, x, z, c, n, liecl.Method.orthonorm_dimonly,
                                            liecl.ClosureConfig(tolerance=1e-10, batch_max=b))
        dt = time.perf_counter() - t
        bits = [np.asarray(a).tobytes() for a in r.basis_array]
        same = base is None or bits == base
        base = base or bits
        print(json.dumps({"n": n, "budget_log2": b.bit_length() - 1, "seconds": round(dt, 2), "dim": r.dimension,
                          "batches": r.stats.engine.get("batches"), "identical_to_2^24": same}), flush=True)
