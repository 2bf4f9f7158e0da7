"""Per-stage trace of the multi-term engine (LIECL_B200_TRACE=1) on given families."""
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2506_01120_b200 import liecl, workloads as w
for arg in sys.argv[1:] or ["tfim_hva_open:12"]:
    fam, n = arg.split(":")
    n = int(n)
    off, x, z, c = w.sum_arrays(getattr(w, fam)(n))
    t = time.perf_counter()
    res = liecl.closure_pauli_sums_arrays(off, x, z, c, n, liecl.Method.orthonorm_dimonly, liecl.ClosureConfig(tolerance=1e-10))
    print(fam, n, res.dimension, "python %.3f s" % (time.perf_counter() - t), "engine %.3f s" % res.stats.wall_seconds, flush=True)
