"""Debug: where do multi-term closure coefficients differ from the reference?"""
import numpy as np
from paper_2506_01120_b200 import liecl
from oracle.oracle import Ref

ref = Ref()
rng = np.random.default_rng(4)
for trial in range(8):
    n = int(rng.integers(2, 5))
    gens = []
    for _ in range(int(rng.integers(2, 4))):
        k = int(rng.integers(1, 5))
        terms = [(liecl.PauliString(int(rng.integers(0, 1 << n)), int(rng.integers(0, 1 << n)), n),
                  complex(*rng.standard_normal(2))) for _ in range(k)]
        gens.append(liecl.pauli_sum_from_terms(n, terms))
    if trial == 0:
        gens.append(liecl.PauliSum(n, []))
    if trial == 1:
        gens.append(gens[0])
    offs, xs, zs, cs = [0], [], [], []
    for g in gens:
        for s, cc in g.terms:
            xs.append(s.x); zs.append(s.z); cs.append((cc.real, cc.imag))
        offs.append(len(xs))
    if max(np.diff(offs)) < 2:
        continue
    off, x, z, c = np.array(offs, np.int64), np.array(xs, np.uint64), np.array(zs, np.uint64), np.array(cs).reshape(-1, 2)
    for method in (liecl.Method.orthonorm_dimonly, liecl.Method.orthonorm):
        res = liecl.closure_pauli_sums_arrays(off, x, z, c, n, method, liecl.ClosureConfig(tolerance=1e-10, record_log=True))
        o = ref.closure_pauli(off, x, z, c, n, method=liecl.to_string(method), tol=1e-10)
        bo, bx, bz, bc = res.basis_array
        ro, rx, rz, rc = o.basis
        bad = np.nonzero((bc.view(np.uint64) != rc.view(np.uint64)).any(axis=1))[0]
        print(trial, method.name, "n", n, "dim", res.dimension, o.dimension, "ngens", len(gens), "bad terms", len(bad), "of", len(bc))
        for t in bad[:6]:
            el = np.searchsorted(bo, t, side="right") - 1
            print("   term", t, "element", el, "mine", bc[t].tolist(), "ref", rc[t].tolist())
        lg = ref.decision_log_pauli(off, x, z, c, n, keep_original=(method == liecl.Method.orthonorm), tol=1e-10)
        d = np.nonzero(res.decision_log["residual_norm"].view(np.uint64) != lg.log["residual_norm"].view(np.uint64))[0]
        if len(d):
            print("   log rn differs at", d[:5].tolist(), res.decision_log[d[:3]].tolist(), lg.log[d[:3]].tolist())
