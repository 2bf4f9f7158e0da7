"""Multi-term PauliSum closures, engine wall time of whichever library
LIECL_B200_LIB names (A/B of the hand-written sorts against the CUB build)."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2506_01120_b200 import liecl, workloads as w
cases = [("tfim_hva_open", int(a)) for a in sys.argv[1:]] or [("tfim_hva_open", n) for n in (8, 12, 16, 20, 24)]
for fam, n in cases:
    off, x, z, c = w.sum_arrays(w.tfim_hva_open(n))
    best = None
    for _ in range(3 if n <= 20 else 1):
        t = time.perf_counter()
        r = liecl.closure_pauli_sums_arrays(off, x, z, c, n, liecl.Method.orthonorm_dimonly,
                                            liecl.ClosureConfig(tolerance=1e-10))
        s = time.perf_counter() - t
        best = s if best is None else min(best, s)
    print(json.dumps({"lib": os.path.basename(os.environ.get("LIECL_B200_LIB", "default")), "family": fam, "n": n,
                      "dim": r.dimension, "seconds": round(best, 4), "engine_s": round(r.stats.wall_seconds, 4)}),
          flush=True)
