"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified liecl sources (oracle/_ref/libliecl_ref.so, built from
/root/reference by oracle/Makefile) on the seeded BASELINE workloads
(paper_2506_01120_b200/workloads.py) and stores what they produce. Needs
/root/reference (this container only); the fixtures travel, the reference
does not.

    python tests/golden/make_golden.py [--c2] [--only-sums]   (--c2: ~10+ min)

Multi-term PauliSum fixtures come from the default-rounding
build oracle/_ref/libliecl_ref_exact.so (see oracle/Makefile).
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import REF_EXACT_SO, Ref, build, pauli_single_arrays  # noqa: E402
from paper_2506_01120_b200 import workloads as w  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
C2_ROWS = 100          # growth phase of config 2 (all accepts happen before it ends)
CHECK_SEED = 1234      # fixed random weights for basis checksums


def checksum_weights(D):
    rng = np.random.default_rng(CHECK_SEED)
    return rng.standard_normal(D) + 1j * rng.standard_normal(D)


def dense_case(ref, cfg, method, rows=0, threads=8, keep_vectors=None):
    keep = method == "orthonorm"
    out = {"name": cfg.name, "method": method, "d": cfg.d, "tol": cfg.tol, "digest": cfg.digest()}
    if rows == 0:
        full = ref.closure_dense(cfg.generators, cfg.d, method=method, tol=cfg.tol, threads=threads)
        out["stats"] = {k: int(v) for k, v in full.stats.items() if k != "wall_seconds" and k != "extra"}
        out["warnings"] = full.warnings
    rep = ref.decision_log_dense(cfg.generators, cfg.d, keep_original=keep, tol=cfg.tol, threads=threads,
                                 row_limit=rows)
    if rows == 0:
        assert rep.dimension == full.dimension
        assert np.array_equal(rep.basis.view(np.float64), full.basis.view(np.float64)), "replay != run_closure"
    out["dimension"] = int(rep.dimension)
    arrays = {
        "log_l": rep.log["l"], "log_m": rep.log["m"], "log_null": rep.log["null_cand"],
        "log_indep": rep.log["independent"], "log_rn": rep.log["residual_norm"],
        "basis_checksum": rep.basis @ checksum_weights(cfg.d * cfg.d),
        "ortho_checksum": rep.ortho @ checksum_weights(cfg.d * cfg.d),
        "basis_norms": np.linalg.norm(rep.basis, axis=1),
    }
    if keep_vectors is None:
        arrays["basis"] = rep.basis
        arrays["ortho"] = rep.ortho
    else:
        idx = np.array([i for i in keep_vectors if i < rep.dimension], np.int64)
        arrays["basis_rows"] = idx
        arrays["basis"] = rep.basis[idx]
        arrays["ortho"] = rep.ortho[idx]
    return out, arrays


def save(tag, meta, arrays):
    np.savez_compressed(os.path.join(OUT, tag + ".npz"), **arrays)
    with open(os.path.join(OUT, tag + ".json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", tag, meta.get("dimension"), meta.get("stats"))


SUM_CASES = (("tfim_hva_open", 6), ("spin_glass_hva", 3))


def sums_cases():
    refx = Ref(REF_EXACT_SO)
    for family, n in SUM_CASES:
        off, x, z, co = refx.build_generators(family, n)
        for method in ("orthonorm-dimonly", "orthonorm"):
            full = refx.closure_pauli(off, x, z, co, n, method=method, tol=1e-10)
            rep = refx.decision_log_pauli(off, x, z, co, n, keep_original=(method == "orthonorm"), tol=1e-10)
            bo, bx, bz, bc = full.basis
            ro, rx, rz, rc = rep.basis
            assert np.array_equal(bo, ro) and np.array_equal(bc.view(np.uint64), rc.view(np.uint64))
            meta = {"name": f"{family}_n{n}", "method": method, "qubits": n, "tol": 1e-10,
                    "dimension": int(full.dimension), "build": "libliecl_ref_exact.so",
                    "stats": {k: int(v) for k, v in full.stats.items() if k not in ("wall_seconds", "extra")},
                    "warnings": full.warnings}
            arrays = {"gen_offsets": off, "gen_x": x, "gen_z": z, "gen_coef_bits": co.view(np.uint64),
                      "offsets": bo, "x": bx, "z": bz, "coef_bits": bc.view(np.uint64),
                      "log_l": rep.log["l"], "log_m": rep.log["m"], "log_null": rep.log["null_cand"],
                      "log_indep": rep.log["independent"], "log_rn_bits": rep.log["residual_norm"].view(np.uint64)}
            save(f"sums_{family}_n{n}_{method}", meta, arrays)


def c3_golden():
    """Config 3's ordered check-and-append (R:src/closure.cpp:142-162 per
    candidate, accepted residual units appended) on w.Config3Exact: inputs a
    GPU box regenerates bit for bit with numpy alone (no BLAS or libm rounding
    in them), so only the reference's outputs are stored."""
    import time
    c = w.Config3Exact()
    V, cands = c.generate_numpy()
    t0 = time.perf_counter()
    ind, rn, secs = Ref().check_sequence_dense(V, cands, c.d, tol=c.tol, append=True)
    meta = {"name": c.name, "d": c.d, "n": c.n, "ncand": c.ncand, "tol": c.tol, "noise": c.noise,
            "input_digest": c.digest(V, cands), "accepted": int(ind.sum()), "seconds": round(secs, 1),
            "build": "libliecl_ref.so (liecl_ref_check_sequence_dense, append)"}
    save(c.name, meta, {"independent": ind, "residual_norm": rn})
    print(f"c3 golden: {ind.sum()} accepted of {len(ind)} in {time.perf_counter() - t0:.1f} s")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c2", action="store_true")
    ap.add_argument("--only-sums", action="store_true")
    ap.add_argument("--c2-orthonorm", action="store_true",
                    help="only config 2's growth phase under Alg. 3 (orthonorm, keep_original): ~10 min")
    ap.add_argument("--c3-golden", action="store_true",
                    help="only the exact-input config-3 stand-in (ordered check-and-append): ~1 min")
    a = ap.parse_args()
    build()
    if a.c2_orthonorm:
        cfg = w.config2()
        meta, arr = dense_case(Ref(), cfg, "orthonorm", rows=C2_ROWS, threads=os.cpu_count(),
                               keep_vectors=[0, 1, 2, 64, 512, 2048, 4094])
        meta["rows"] = C2_ROWS
        save(f"{cfg.name}_orthonorm_rows{C2_ROWS}", meta, arr)
        return
    if a.c3_golden:
        c3_golden()
        return
    sums_cases()
    if a.only_sums:
        return
    ref = Ref()
    for cfg in (w.config0(), w.config1()):
        for method in ("orthonorm-dimonly", "orthonorm"):
            meta, arr = dense_case(ref, cfg, method)
            save(f"{cfg.name}_{method}", meta, arr)
    p = w.config4()
    for method in ("orthonorm-dimonly", "orthonorm"):
        off, x, z, co = pauli_single_arrays(p.x, p.z, p.coef)
        full = ref.closure_pauli(off, x, z, co, p.qubits, method=method, tol=p.tol)
        rep = ref.decision_log_pauli(off, x, z, co, p.qubits, keep_original=(method == "orthonorm"), tol=p.tol)
        bo, bx, bz, bc = full.basis
        ro, rx, rz, rc = rep.basis
        assert np.array_equal(bx, rx) and np.array_equal(bc.view(np.uint64), rc.view(np.uint64))
        meta = {"name": p.name, "method": method, "qubits": p.qubits, "tol": p.tol, "digest": p.digest(),
                "dimension": int(full.dimension),
                "stats": {k: int(v) for k, v in full.stats.items() if k not in ("wall_seconds", "extra")}}
        arrays = {"x": bx, "z": bz, "coef_bits": bc.view(np.uint64), "log_l": rep.log["l"], "log_m": rep.log["m"],
                  "log_null": rep.log["null_cand"], "log_indep": rep.log["independent"],
                  "log_rn_bits": rep.log["residual_norm"].view(np.uint64)}
        save(f"{p.name}_{method}", meta, arrays)
    # SPEC.md known answers through the reference primitives
    spec = {}
    X, Y, Z = (1, 0), (1, 1), (0, 1)
    (rx, rz), ph, e, com = ref.string_product(X, Y, 1)
    spec["XY"] = {"string": [rx, rz], "phase": [ph.real, ph.imag], "exponent": e, "commute": com}
    x2 = ref.from_pauli(np.array([1], np.uint64), np.array([0], np.uint64), np.array([[1.0, 0.0]]), 1)
    y2 = ref.from_pauli(np.array([1], np.uint64), np.array([1], np.uint64), np.array([[1.0, 0.0]]), 1)
    z2 = ref.from_pauli(np.array([0], np.uint64), np.array([1], np.uint64), np.array([[1.0, 0.0]]), 1)
    cxy = ref.commutator_dense(x2, y2, 2)
    spec["commutator_XY_over_2iZ"] = [float(np.abs(cxy - 2j * z2).max())]
    spec["norm_3X_4iZ"] = ref.norm_dense(3 * x2 + 4j * z2, 2)
    spec["Y_matrix"] = [[c.real, c.imag] for c in y2]
    with open(os.path.join(OUT, "spec_examples.json"), "w") as f:
        json.dump(spec, f, indent=1, sort_keys=True)
    print("spec", spec)
    if a.c2:
        cfg = w.config2()
        meta, arr = dense_case(ref, cfg, "orthonorm-dimonly", rows=C2_ROWS, threads=os.cpu_count(),
                               keep_vectors=[0, 1, 2, 64, 512, 2048, 4094])
        meta["rows"] = C2_ROWS
        save(f"{cfg.name}_orthonorm-dimonly_rows{C2_ROWS}", meta, arr)


if __name__ == "__main__":
    main()
