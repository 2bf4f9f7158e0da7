"""Dense (i*H) closure dimension against the bit-exact Pauli-sum closure for
the reference catalog families; wall times."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2506_01120_b200 import liecl, workloads as w
for fam, n, field in (("xxz_hva", 6, "auto"), ("xxz_hva", 7, "auto"), ("tfim_hva_open", 8, "auto"), ("xxz_hva", 7, "complex")):
    specs = getattr(w, fam)(n)
    gens = np.stack([w.vec(1j * w.from_pauli(sp)) for sp in specs])
    t = time.perf_counter()
    try:
        r = liecl.closure_dense_arrays(gens, 1 << n, liecl.Method.orthonorm_dimonly,
                                       liecl.ClosureConfig(tolerance=1e-10, field=field, deadline=time.monotonic() + 120))
        dd, nw = r.dimension, len(r.stats.warnings)
    except Exception as e:
        dd, nw = repr(e)[:80], -1
    td = time.perf_counter() - t
    off, x, z, c = w.sum_arrays(specs)
    t = time.perf_counter()
    try:
        ps = liecl.closure_pauli_sums_arrays(off, x, z, c, n, liecl.Method.orthonorm_dimonly,
                                             liecl.ClosureConfig(tolerance=1e-10, deadline=time.monotonic() + 120))
        ds = ps.dimension
    except Exception as e:
        ds = repr(e)[:80]
    print(fam, n, field, "dense", dd, "warnings", nw, "%.2f s" % td, "| sums", ds, "%.2f s" % (time.perf_counter() - t), flush=True)
