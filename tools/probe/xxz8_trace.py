import os, sys, time
sys.path.insert(0, os.getcwd())
os.environ["LIECL_B200_TRACE"] = "1"
from paper_2506_01120_b200 import liecl, workloads as w
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
off, x, z, c = w.sum_arrays(w.xxz_hva(n))
t = time.perf_counter()
try:
    r = liecl.closure_pauli_sums_arrays(off, x, z, c, n, liecl.Method.orthonorm_dimonly,
                                        liecl.ClosureConfig(tolerance=1e-10, deadline=time.monotonic() + 60))
    print("dim", r.dimension, r.stats.engine, "terms", int(r.basis_array[0][-1]) if False else "", time.perf_counter() - t, file=sys.stderr)
except Exception as e:
    print("EXC", repr(e)[:150], time.perf_counter() - t, file=sys.stderr)
