"""Multi-term PauliSum closures: GPU engine wall time vs the reference build
(default rounding, all host threads; each reference run in a subprocess with a
time limit)."""
import json, os, subprocess, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2506_01120_b200 import liecl
from oracle.oracle import Ref, REF_EXACT_SO

REF_SNIPPET = r'''
import sys, time, json, numpy as np
sys.path.insert(0, ".")
from oracle.oracle import Ref, REF_EXACT_SO
fam, n, dim = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
r = Ref(REF_EXACT_SO)
off, x, z, c = r.build_generators(fam, n)
t = time.perf_counter()
o = r.closure_pauli(off, x, z, c, n, method="orthonorm-dimonly", tol=1e-10, threads=%d, basis_cap=dim + 1, term_cap=1 << 26)
s = time.perf_counter() - t
np.savez("/tmp/ref_%%s_%%d.npz" %% (fam, n), *o.basis)
print(json.dumps({"ref_s": s, "dim": o.dimension}))
''' % (os.cpu_count() or 1)

ref = Ref(REF_EXACT_SO)
limit = float(os.environ.get("REF_LIMIT", "240"))
cases = [(f, int(n)) for f, n in (a.split(":") for a in sys.argv[1:])] or [
    ("tfim_hva_open", 12), ("tfim_hva_open", 16), ("tfim_hva_open", 20), ("xxz_hva", 6), ("spin_glass_hva", 4),
    ("xxz_hva", 8), ("spin_glass_hva", 5)]
for fam, n in cases:
    off, x, z, c = ref.build_generators(fam, n)
    cfg = liecl.ClosureConfig(tolerance=1e-10)
    liecl.closure_pauli_sums_arrays(off, x, z, c, n, liecl.Method.orthonorm_dimonly, cfg) if n <= 12 else None
    reps = []
    for _ in range(int(os.environ.get("REPS", "1"))):
        t = time.perf_counter()
        res = liecl.closure_pauli_sums_arrays(off, x, z, c, n, liecl.Method.orthonorm_dimonly, cfg)
        reps.append((time.perf_counter() - t, res.stats.wall_seconds))
    gpu = min(r[0] for r in reps)
    out = {"family": fam, "n": n, "dim": res.dimension, "terms": int(res.basis_array[0][-1]), "gpu_s": round(gpu, 4),
           "engine_s": round(min(r[1] for r in reps), 4), "engine_reps": [round(r[1], 3) for r in reps], "brackets": res.stats.commutators_evaluated,
           "engine": res.stats.engine}
    if os.environ.get("NO_REF"):
        print(json.dumps(out), flush=True)
        continue
    try:
        p = subprocess.run([sys.executable, "-c", REF_SNIPPET, fam, str(n), str(res.dimension)], capture_output=True,
                           text=True, timeout=limit)
        r = json.loads(p.stdout.strip().splitlines()[-1])
        got = np.load("/tmp/ref_%s_%d.npz" % (fam, n))
        out["ref_s"] = round(r["ref_s"], 3)
        out["ref_threads"] = os.cpu_count()
        out["bit_exact"] = bool(all(np.array_equal(np.asarray(a).view(np.uint64), got["arr_%d" % i].view(np.uint64))
                                    for i, a in enumerate(res.basis_array)))
    except subprocess.TimeoutExpired:
        out["ref_s"] = f"> {limit:.0f}"
    print(json.dumps(out), flush=True)
