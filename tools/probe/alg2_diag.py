import numpy as np, sys
sys.path.insert(0, '.')
from oracle.oracle import Ref, REF_EXACT_SO
from paper_2506_01120_b200 import liecl
r = Ref(REF_EXACT_SO)
off, x, z, c = r.build_generators("tfim_hva_open", 5)
o = r.closure_pauli(off, x, z, c, 5, method="matrix-inversion", tol=1e-10)
print("ref warnings:", o.warnings)
for fld in (None,):
    res = liecl.closure_pauli_sums_arrays(off, x, z, c, 5, liecl.Method.matrix_inversion, liecl.ClosureConfig(tolerance=1e-10, record_log=True))
    lg = res.decision_log
    rej = (lg["null_cand"] == 0) & (lg["independent"] == 0)
    rn = lg["residual_norm"][rej]
    print("ours: rejects", rej.sum(), "max rn", rn.max(), "n>1e-11", (rn > 1e-11).sum(), "median", np.median(rn))
    for w in res.stats.warnings[:12]: print(w.detail)
    A, Ai = res.gram
    print("cond", np.linalg.cond(A), "inv err", np.abs(A @ Ai - np.eye(len(A))).max())
    Ar, Air = r.last_gram(res.dimension)
    print("ref inv err", np.abs(Ar @ Air - np.eye(len(Ar))).max(), "Ai diff", np.abs(Ai - Air).max())
