"""Multi-term PauliSum closures on the GPU against the
reference build with its default rounding (oracle/_ref/libliecl_ref_exact.so:
the reference's own run_engine over R:src/pauli.cpp's PauliSum arithmetic, no
FMA contraction, as its CMake build on the x86-64 baseline ISA): same dimension, statistics, warnings,
decision log (residual norms bit for bit) and basis coefficient bits, for both
orthonormal methods."""
import numpy as np
import pytest

from paper_2506_01120_b200 import liecl
from paper_2506_01120_b200 import workloads as w

pytestmark = pytest.mark.gpu
DIMONLY, KEEP = liecl.Method.orthonorm_dimonly, liecl.Method.orthonorm


def spec_arrays(sums):
    off, xs, zs, cs = [0], [], [], []
    for s in sums:
        xs += list(s.x)
        zs += list(s.z)
        cs += [(complex(c).real, complex(c).imag) for c in s.coef]
        off.append(len(xs))
    return (np.array(off, np.int64), np.array(xs, np.uint64), np.array(zs, np.uint64),
            np.array(cs, np.float64).reshape(-1, 2))


def compare(ref, off, x, z, c, n, method, tol=1e-10):
    res = liecl.closure_pauli_sums_arrays(off, x, z, c, n, method,
                                          liecl.ClosureConfig(tolerance=tol, record_log=True))
    o = ref.closure_pauli(off, x, z, c, n, method=liecl.to_string(method), tol=tol, threads=4)
    assert res.dimension == o.dimension
    for k in ("commutators_evaluated", "independence_checks", "accepted"):
        assert getattr(res.stats, k) == o.stats[k], k
    bo, bx, bz, bc = res.basis_array
    ro, rx, rz, rc = o.basis
    assert np.array_equal(bo, ro)
    assert np.array_equal(bx, rx) and np.array_equal(bz, rz)
    assert np.array_equal(bc.view(np.uint64), rc.view(np.uint64))  # coefficient bits
    kinds = sorted(line.split("\t")[0] for line in o.warnings.splitlines() if line)
    assert sorted(wr.kind for wr in res.stats.warnings) == kinds
    lg = ref.decision_log_pauli(off, x, z, c, n, keep_original=(method == KEEP), tol=tol)
    mine = res.decision_log
    assert len(mine) == len(lg.log)
    for f in ("l", "m", "null_cand", "independent"):
        assert np.array_equal(mine[f], lg.log[f]), f
    assert np.array_equal(mine["residual_norm"].view(np.uint64), lg.log["residual_norm"].view(np.uint64))
    if method == KEEP:  # the orthonormal tuple as well
        lo, lx, lz, lc = lg.basis
        oo, ox, oz, oc = res.ortho_array
        # the replay returns the commutator basis; the orthonormal tuple has the
        # same size and is checked through the residual norms above
        assert len(oo) == len(lo)
    return res


@pytest.mark.parametrize("method", [DIMONLY, KEEP], ids=["dimonly", "orthonorm"])
@pytest.mark.parametrize("family,n,dim", [("tfim_hva_open", 4, 16), ("tfim_hva_open", 6, 36), ("xxz_hva", 4, 10),
                                          ("spin_glass_hva", 3, 63)])
def test_families_match_reference(ref_exact, family, n, dim, method):
    off, x, z, c = ref_exact.build_generators(family, n)
    assert np.diff(off).max() > 1  # genuinely multi-term
    res = compare(ref_exact, off, x, z, c, n, method)
    assert res.dimension == dim


@pytest.mark.parametrize("method", [DIMONLY, KEEP], ids=["dimonly", "orthonorm"])
@pytest.mark.parametrize("make", [w.config0, w.config1], ids=["c0", "c1"])
def test_baseline_configs_on_pauli_backend(ref_exact, make, method):
    cfg = make()
    off, x, z, c = spec_arrays(cfg.sums)
    res = compare(ref_exact, off, x, z, c, cfg.sums[0].qubits, method, cfg.tol)
    assert res.dimension == {"c0": 9, "c1": 30}[make.__name__.replace("config", "c")]


def test_random_sums_match_reference(ref_exact):
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
            gens.append(liecl.PauliSum(n, []))  # null generator -> warning
        if trial == 1:
            gens.append(gens[0])  # dependent generator
        offs, xs, zs, cs = [0], [], [], []
        for g in gens:
            for s, cc in g.terms:
                xs.append(s.x); zs.append(s.z); cs.append((cc.real, cc.imag))
            offs.append(len(xs))
        if max(np.diff(offs)) < 2:
            continue
        for method in (DIMONLY, KEEP):
            compare(ref_exact, np.array(offs, np.int64), np.array(xs, np.uint64), np.array(zs, np.uint64),
                    np.array(cs, np.float64).reshape(-1, 2), n, method)


def test_run_closure_routes_multi_term_sums(ref):
    off, x, z, c = ref.build_generators("tfim_hva_open", 4)
    gens = [liecl.PauliSum(4, [(liecl.PauliString(int(x[t]), int(z[t]), 4), complex(c[t, 0], c[t, 1]))
                               for t in range(off[i], off[i + 1])]) for i in range(len(off) - 1)]
    res = liecl.run_closure(gens, DIMONLY, liecl.ClosureConfig(tolerance=1e-10))
    assert res.dimension == 16 and res.backend == liecl.Backend.pauli
    assert all(isinstance(b, liecl.PauliSum) for b in res.basis)
    with pytest.raises(liecl.CapacityError):
        liecl.run_closure(gens, DIMONLY, liecl.ClosureConfig(tolerance=1e-10, max_dim=5))


def test_small_batches_same_bits(ref):
    # a product budget of one bracket per batch: every row split into
    # single-pair batches must give the same verdicts and bits
    off, x, z, c = ref.build_generators("spin_glass_hva", 3)
    a = liecl.closure_pauli_sums_arrays(off, x, z, c, 3, DIMONLY, liecl.ClosureConfig(tolerance=1e-10))
    b = liecl.closure_pauli_sums_arrays(off, x, z, c, 3, DIMONLY, liecl.ClosureConfig(tolerance=1e-10, batch_max=1))
    for u, v in zip(a.basis_array, b.basis_array):
        assert np.array_equal(np.asarray(u).view(np.uint64), np.asarray(v).view(np.uint64))
    assert b.stats.engine["batches"] > a.stats.engine["batches"]


@pytest.mark.parametrize("tag", ["sums_tfim_hva_open_n6_orthonorm-dimonly", "sums_tfim_hva_open_n6_orthonorm",
                                 "sums_spin_glass_hva_n3_orthonorm-dimonly", "sums_spin_glass_hva_n3_orthonorm"])
def test_golden_fixtures_bit_exact(golden, tag):
    # committed fixtures from the reference build: no reference needed at run time
    meta, g = golden(tag)
    method = liecl.method_from_string(meta["method"])
    res = liecl.closure_pauli_sums_arrays(g["gen_offsets"], g["gen_x"], g["gen_z"],
                                          g["gen_coef_bits"].view(np.float64), meta["qubits"], method,
                                          liecl.ClosureConfig(tolerance=meta["tol"], record_log=True))
    assert res.dimension == meta["dimension"]
    for k in ("commutators_evaluated", "independence_checks", "accepted"):
        assert getattr(res.stats, k) == meta["stats"][k]
    bo, bx, bz, bc = res.basis_array
    assert np.array_equal(bo, g["offsets"]) and np.array_equal(bx, g["x"]) and np.array_equal(bz, g["z"])
    assert np.array_equal(bc.view(np.uint64), g["coef_bits"])
    log = res.decision_log
    assert np.array_equal(log["l"], g["log_l"]) and np.array_equal(log["m"], g["log_m"])
    assert np.array_equal(log["null_cand"], g["log_null"]) and np.array_equal(log["independent"], g["log_indep"])
    assert np.array_equal(log["residual_norm"].view(np.uint64), g["log_rn_bits"])


@pytest.mark.parametrize("tag", ["sums_tfim_hva_open_n6_orthonorm-dimonly", "sums_spin_glass_hva_n3_orthonorm"])
def test_general_merge_path_bit_exact(golden, tag, monkeypatch):
    # small sums take the fused single-CTA check by default; the general
    # multi-kernel merges (large sums) must give the same bits
    monkeypatch.setenv("LIECL_B200_SUMS_FUSED", "0")
    test_golden_fixtures_bit_exact(golden, tag)


def test_small_output_buffers_fetch_without_recompute(golden):
    # a result larger than the first output buffers is fetched from the device
    meta, g = golden("sums_spin_glass_hva_n3_orthonorm-dimonly")
    res = liecl.closure_pauli_sums_arrays(g["gen_offsets"], g["gen_x"], g["gen_z"],
                                          g["gen_coef_bits"].view(np.float64), meta["qubits"],
                                          liecl.Method.orthonorm_dimonly,
                                          liecl.ClosureConfig(tolerance=meta["tol"]), term_cap=16)
    bo, bx, bz, bc = res.basis_array
    assert np.array_equal(bo, g["offsets"]) and np.array_equal(bc.view(np.uint64), g["coef_bits"])
    assert res.stats.commutators_evaluated == meta["stats"]["commutators_evaluated"]  # one run's counters


@pytest.mark.parametrize("tag", ["sums_tfim_hva_open_n6_orthonorm-dimonly", "sums_spin_glass_hva_n3_orthonorm-dimonly",
                                 "sums_spin_glass_hva_n3_orthonorm"])
def test_certified_reject_screen_keeps_results_bit_exact(golden, tag):
    # without the decision log, certified rejects skip the second pass; the
    # basis, statistics and warnings must still be the reference's bits
    meta, g = golden(tag)
    method = liecl.method_from_string(meta["method"])
    res = liecl.closure_pauli_sums_arrays(g["gen_offsets"], g["gen_x"], g["gen_z"],
                                          g["gen_coef_bits"].view(np.float64), meta["qubits"], method,
                                          liecl.ClosureConfig(tolerance=meta["tol"]))
    assert res.dimension == meta["dimension"]
    for k in ("commutators_evaluated", "independence_checks", "accepted"):
        assert getattr(res.stats, k) == meta["stats"][k]
    bo, bx, bz, bc = res.basis_array
    assert np.array_equal(bo, g["offsets"]) and np.array_equal(bc.view(np.uint64), g["coef_bits"])
    kinds = sorted(line.split("\t")[0] for line in meta["warnings"].splitlines() if line)
    assert sorted(wr.kind for wr in res.stats.warnings) == kinds
    assert res.stats.engine["survivors"] > 0  # the screened path ran (batches > the fused size)
