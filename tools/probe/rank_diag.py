"""Rank-engine divergence probe: first GPU basis column outside the
reference's span, with numpy's sigma ratio for that verdict."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2506_01120_b200 import liecl
from oracle.oracle import Ref
eps = np.finfo(float).eps
for f in ("soak_fail_8_221", "soak_fail_7_139"):
    gens = np.load(f"tools/probe/soak_cases/{f}.npy"); d = 8; D = 64
    o = Ref().closure_dense(gens, d, method="standard-rank", tol=1e-10)
    RB = np.asarray(o.basis).reshape(o.dimension, D).T
    for bs in (0, 1, 4):
        try:
            r = liecl.closure_dense_arrays(gens, d, liecl.Method.standard_rank,
                                           liecl.ClosureConfig(tolerance=1e-10, batch_max=bs, record_log=True))
        except Exception as e:
            print(f, bs, repr(e)[:200]); continue
        GB = np.asarray(r.basis_array).reshape(r.dimension, D).T
        first = None
        for k in range(GB.shape[1]):
            if k >= RB.shape[1] or np.abs(GB[:, k] - RB[:, k]).max() > 1e-8:
                first = k; break
        line = [f, "bs", bs, "gpu dim", r.dimension, "ref dim", o.dimension, "first differing column", first]
        if first is not None:
            S = GB[:, : first + 1]
            s = np.linalg.svd(S, compute_uv=False)
            line += ["numpy sigma ratio at that accept %.2e (thr %.2e)" % (s[-1] / s[0], eps * max(D, first + 1))]
            L = r.decision_log
            acc = np.nonzero(L["independent"] == 1)[0]
            e = L[acc[first]]
            line += ["pair", (int(e["l"]), int(e["m"])), "rechecked", int(e["rechecked"])]
        print(*line, flush=True)
