import os, sys, time
sys.path.insert(0, os.getcwd())
os.environ["LIECL_B200_TRACE"] = "1"
from paper_2506_01120_b200 import liecl, workloads as w
n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
off, x, z, c = w.sum_arrays(w.tfim_hva_open(n))
t = time.perf_counter()
r = liecl.closure_pauli_sums_arrays(off, x, z, c, n, liecl.Method.orthonorm_dimonly, liecl.ClosureConfig(tolerance=1e-10))
print("n", n, "dim", r.dimension, "seconds", round(time.perf_counter() - t, 2), r.stats.engine, file=sys.stderr)
