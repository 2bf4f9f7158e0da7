import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2506_01120_b200 import liecl, workloads as w
def run(make, field, method=liecl.Method.orthonorm_dimonly):
    cfg = make()
    return liecl.closure_dense_arrays(cfg.generators, cfg.d, method, liecl.ClosureConfig(tolerance=cfg.tol, record_log=True, field=field))
for f in ("auto", "complex"):
    run(w.config0, f)
r = run(w.config1, "auto")
log = r.decision_log
bad = np.nonzero(~np.isfinite(log["residual_norm"]))[0]
print("dim", r.dimension, "nan entries", len(bad), [(int(log["l"][i]), int(log["m"][i]), int(log["independent"][i]), int(log["rechecked"][i])) for i in bad[:12]], flush=True)
print("basis finite:", bool(np.isfinite(r.basis_array).all()))
