"""First-divergence analysis of the soak's dense failures: GPU decision log
against the reference build's, with the residuals on both sides. Logs come
from oracle/_ref (travels with the snapshot) - a diagnostic, not a test."""
import os, sys, glob
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2506_01120_b200 import liecl
from oracle.oracle import Ref
ref = Ref()
tol = 1e-10
for f in sorted(glob.glob("tools/probe/soak_cases/*.npy")):
    gens = np.load(f); d = int(round(np.sqrt(gens.shape[1])))
    if d != 16: continue
    rl = ref.decision_log_dense(gens, d, tol=tol).log
    for field in ("auto", "complex"):
        for bs in (0, 1, 16):
            try:
                r = liecl.closure_dense_arrays(gens, d, liecl.Method.orthonorm_dimonly,
                                               liecl.ClosureConfig(tolerance=tol, field=field, record_log=True, max_dim=400, batch_max=bs))
            except Exception as e:
                print(os.path.basename(f), field, bs, repr(e)[:200]); continue
            gl = r.decision_log
            n = min(len(gl), len(rl)); first = None
            for i in range(n):
                a, b = gl[i], rl[i]
                if (a["l"], a["m"]) != (b["l"], b["m"]) or a["null_cand"] != b["null_cand"] or a["independent"] != b["independent"]:
                    first = i; break
            if first is None:
                print(os.path.basename(f), field, bs, "dim", r.dimension, "no divergence in", n); continue
            a, b = gl[first], rl[first]
            print(os.path.basename(f), field, bs, "dim", r.dimension, "first divergence", first, "pair", (int(a["l"]), int(a["m"])),
                  "gpu null/ind/res", int(a["null_cand"]), int(a["independent"]), "%.3e" % a["residual_norm"],
                  "ref", int(b["null_cand"]), int(b["independent"]), "%.3e" % b["residual_norm"],
                  "in band:", any(tol / 10 <= x <= 10 * tol for x in (a["residual_norm"], b["residual_norm"])), flush=True)
