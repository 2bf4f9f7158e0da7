import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2506_01120_b200 import liecl
for f in ("soak_fail_8_221", "soak_fail_7_139"):
    gens = np.load(f"tools/probe/soak_cases/{f}.npy")
    r = liecl.closure_dense_arrays(gens, 8, liecl.Method.standard_rank,
                                   liecl.ClosureConfig(tolerance=1e-10, record_log=True, max_dim=64))
    np.save(f"gpurun_out/rank_gpu_basis_{f}.npy", np.asarray(r.basis_array))
    np.save(f"gpurun_out/rank_gpu_log_{f}.npy", r.decision_log)
    # also the orthonormal-keep closure's basis (same commutator basis semantics)
    r2 = liecl.closure_dense_arrays(gens, 8, liecl.Method.orthonorm, liecl.ClosureConfig(tolerance=1e-10, field="complex"))
    np.save(f"gpurun_out/keep_gpu_basis_{f}.npy", np.asarray(r2.basis_array))
    print(f, r.dimension, r2.dimension)
