"""Multi-term sums closures against the fused-check batch limit
(LIECL_B200_SUMS_FUSED_BATCH): engine seconds, best of 3, per family/size."""
import json, os, subprocess, sys
CHILD = r'''
import os, sys, time, json
sys.path.insert(0, os.getcwd())
from paper_2506_01120_b200 import liecl, workloads as w
fam, n = sys.argv[1], int(sys.argv[2])
off, x, z, c = w.sum_arrays(getattr(w, fam)(n))
best = 1e30
for _ in range(3):
    t = time.perf_counter()
    r = liecl.closure_pauli_sums_arrays(off, x, z, c, n, liecl.Method.orthonorm_dimonly, liecl.ClosureConfig(tolerance=1e-10))
    best = min(best, r.stats.wall_seconds)
print(json.dumps({"dim": r.dimension, "engine_s": round(best, 4), "kernels": r.stats.engine["kernels"]}))
'''
for fb in sys.argv[1:] or ["16", "256", "100000"]:
    for fam, n in (("tfim_hva_open", 12), ("tfim_hva_open", 16), ("tfim_hva_open", 20), ("xxz_hva", 6), ("spin_glass_hva", 4)):
        env = dict(os.environ, LIECL_B200_SUMS_FUSED_BATCH=fb)
        out = subprocess.run([sys.executable, "-c", CHILD, fam, str(n)], capture_output=True, text=True, env=env, timeout=600)
        row = {"fused_batch": int(fb), "family": fam, "n": n}
        row.update(json.loads(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else {"error": out.stderr[-200:]})
        print(json.dumps(row), flush=True)
