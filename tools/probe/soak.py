"""Soak: many closures of every kind in random order in ONE process (engine
caches, recycled device memory), each checked against the oracle."""
import os, sys, random, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2506_01120_b200 import liecl, workloads as w
from oracle.oracle import Port, Ref, REF_EXACT_SO
from oracle.conditioning import dense_sensitivity, gram_sensitivity

port, ref, refx = Port(), Ref(), Ref(REF_EXACT_SO)
SEED = int(sys.argv[1]) if len(sys.argv) > 1 else 7
ITERS = int(sys.argv[2]) if len(sys.argv) > 2 else 240
rng = np.random.default_rng(SEED)
random.seed(SEED)
D, K = liecl.Method.orthonorm_dimonly, liecl.Method.orthonorm


def dense_case():
    n = int(rng.integers(1, 5)); d = 1 << n
    gens = []
    for _ in range(int(rng.integers(2, 4))):
        terms = [(liecl.PauliString(int(rng.integers(0, d)), int(rng.integers(0, d)), n), complex(rng.standard_normal()))
                 for _ in range(int(rng.integers(1, 4)))]
        s = liecl.pauli_sum_from_terms(n, terms)
        gens.append((1j * liecl.from_pauli(s).matrix).ravel(order="F") if s.terms else np.zeros(d * d, complex))
    return np.stack(gens), d


fails, counts, sensitive = [], {}, []
REF_ERRORS = ("CapacityError", "DegeneracyError")


def rounding_decided(gens, d, gram=False, rank_tol=None):
    if rank_tol is not None:
        # rank: commutator basis = the accepted unit candidates (as Alg. 3);
        # threshold = rank_tolerance, else eps * max(d^2, n+1) (R:src/dense.cpp:133-137)
        o = ref.decision_log_dense(gens, d, keep_original=True, tol=1e-10)
        return dense_sensitivity(o.log, o.basis, d, rank_tol or np.finfo(float).eps * d * d)["sensitive"]
    if gram:
        try:
            return gram_sensitivity(ref.closure_dense(gens, d, method="matrix-inversion", tol=1e-10).basis, d, 1e-10)["sensitive"]
        except Exception:
            return True
    o = ref.decision_log_dense(gens, d, tol=1e-10)
    return dense_sensitivity(o.log, o.basis, d, 1e-10)["sensitive"]

t0 = time.time()
for it in range(ITERS):
    t_it = time.time()
    if os.environ.get("SOAK_PROGRESS"):
        print("it", it, flush=True)
    kind = random.choice(["dense", "dense", "gram", "rank", "single", "sums"])
    counts[kind] = counts.get(kind, 0) + 1
    try:
        if kind in ("dense", "gram", "rank"):
            gens, d = dense_case()
            rank_tol = random.choice([0.0, 1e-10]) if kind == "rank" else None
            if rounding_decided(gens, d, gram=(kind == "gram"), rank_tol=rank_tol):
                # verdicts are rounding-decided (oracle/conditioning.py): only the
                # reference's error contract applies - finish, or raise its errors
                try:
                    m = {"dense": D, "gram": liecl.Method.matrix_inversion, "rank": liecl.Method.standard_rank}[kind]
                    liecl.closure_dense_arrays(gens, d, m, liecl.ClosureConfig(tolerance=1e-10, rank_tolerance=rank_tol or 0.0))
                except Exception as e:
                    if type(e).__name__ not in REF_ERRORS:
                        raise
                sensitive.append((it, kind))
                continue
            if kind == "dense":
                m = random.choice([D, K]); field = random.choice(["auto", "complex"])
                r = liecl.closure_dense_arrays(gens, d, m, liecl.ClosureConfig(tolerance=1e-10, field=field))
                o = port.closure_dense(gens, d, keep_original=(m == K), tol=1e-10)
                ok = r.dimension == o.dimension and (o.dimension == 0 or np.abs(r.basis_array - o.basis).max() < 1e-9 * max(1, np.abs(o.basis).max()))
                if not ok:
                    np.save(f"gpurun_out/soak_fail_{SEED}_{it}.npy", gens)
                    print("DENSE FAIL", it, "d", d, "method", m, "field", field, "gpu dim", r.dimension, "port dim", o.dimension,
                          "engine", r.stats.engine, flush=True)
            else:
                m = liecl.Method.matrix_inversion if kind == "gram" else liecl.Method.standard_rank
                try:
                    o = ref.closure_dense(gens, d, method=liecl.to_string(m), tol=1e-10, rank_tol=rank_tol or 0.0)
                except Exception:
                    continue  # the reference itself raises (degenerate Gram): skip
                r = liecl.closure_dense_arrays(gens, d, m, liecl.ClosureConfig(tolerance=1e-10, rank_tolerance=rank_tol or 0.0))
                ok = r.dimension == o.dimension
                if not ok:
                    np.save(f"gpurun_out/soak_fail_{SEED}_{it}.npy", gens)
                    print("FAIL", it, kind, "d", d, "gpu dim", r.dimension, "ref dim", o.dimension, flush=True)
        elif kind == "single":
            n = int(rng.integers(2, 7)); k = int(rng.integers(2, 6))
            x = rng.integers(0, 1 << n, k).astype(np.uint64); z = rng.integers(0, 1 << n, k).astype(np.uint64)
            c = rng.standard_normal((k, 2)); m = random.choice([D, K])
            r = liecl.closure_pauli_arrays(x, z, c, n, m, liecl.ClosureConfig(tolerance=1e-10))
            o = port.closure_pauli_single(x, z, c, n, keep_original=(m == K), tol=1e-10)
            bx, bz, bc = r.basis_array
            ok = r.dimension == o.dimension and np.array_equal(bc.view(np.uint64), o.basis[2].view(np.uint64))
        else:
            # n <= 4: random complex sums at n = 5 close to most of gl(32) with
            # ~1000-term elements; the reference build itself needs > 5 min there
            n = int(rng.integers(2, 5))
            offs, xs, zs, cs = [0], [], [], []
            for _ in range(int(rng.integers(2, 4))):
                s = liecl.pauli_sum_from_terms(n, [(liecl.PauliString(int(rng.integers(0, 1 << n)), int(rng.integers(0, 1 << n)), n),
                                                    complex(*rng.standard_normal(2))) for _ in range(int(rng.integers(1, 5)))])
                for st, cc in s.terms:
                    xs.append(st.x); zs.append(st.z); cs.append((cc.real, cc.imag))
                offs.append(len(xs))
            arr = (np.array(offs, np.int64), np.array(xs, np.uint64), np.array(zs, np.uint64), np.array(cs, np.float64).reshape(-1, 2))
            m = random.choice([D, K])
            r = liecl.closure_pauli_sums_arrays(*arr, n, m, liecl.ClosureConfig(tolerance=1e-10))
            o = refx.closure_pauli(*arr, n, method=liecl.to_string(m), tol=1e-10)
            ok = r.dimension == o.dimension and all(np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))
                                                    for a, b in zip(r.basis_array, o.basis))
        if not ok:
            fails.append((it, kind))
    except Exception as e:
        fails.append((it, kind, repr(e)[:200]))
        if kind in ("dense", "gram", "rank"):
            np.save(f"gpurun_out/soak_fail_{SEED}_{it}.npy", gens)
            print("EXC", it, kind, "d", d, locals().get("m"), locals().get("field"), repr(e)[:120], flush=True)
print({"seed": SEED, "iterations": ITERS, "kinds": counts, "rounding_decided": len(sensitive), "failures": fails, "seconds": round(time.time() - t0, 1)})
