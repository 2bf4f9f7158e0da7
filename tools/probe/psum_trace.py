import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2506_01120_b200 import liecl
from oracle.oracle import Ref, REF_EXACT_SO
ref = Ref(REF_EXACT_SO)
for fam, n in [("tfim_hva_open", 12), ("xxz_hva", 6), ("tfim_hva_open", 12)]:
    off, x, z, c = ref.build_generators(fam, n)
    t = time.perf_counter()
    res = liecl.closure_pauli_sums_arrays(off, x, z, c, n, liecl.Method.orthonorm_dimonly, liecl.ClosureConfig(tolerance=1e-10))
    print(fam, n, res.dimension, "python %.3f s" % (time.perf_counter() - t), "engine %.3f s" % res.stats.wall_seconds, flush=True)
