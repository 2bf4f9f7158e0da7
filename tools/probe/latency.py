"""Wall-time probe of the latency-bound configs (0, 1, 4) through the C-ABI."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2506_01120_b200 import liecl, native, workloads as w

def run(name, fn, reps=20):
    fn()
    ts = []
    for _ in range(reps):
        k0 = native.kernel_count(0)
        t0 = time.perf_counter()
        r = fn()
        ts.append(time.perf_counter() - t0)
    print(f"{name}: median {1e3*np.median(ts):.3f} ms min {1e3*min(ts):.3f} ms, kernels/run {native.kernel_count(0)-k0}, "
          f"dim {r.dimension}, batches {r.stats.engine.get('batches')}, rechecks {r.stats.engine.get('rechecks')}")

c0, c1, c4 = w.config0(), w.config1(), w.config4()
for field in ("auto", "complex"):
    run(f"c0 {field}", lambda: liecl.closure_dense_arrays(c0.generators, c0.d, liecl.Method.orthonorm_dimonly,
                                                           liecl.ClosureConfig(tolerance=1e-10, field=field)))
    run(f"c1 {field}", lambda: liecl.closure_dense_arrays(c1.generators, c1.d, liecl.Method.orthonorm_dimonly,
                                                           liecl.ClosureConfig(tolerance=1e-10, field=field)))
run("c4", lambda: liecl.closure_pauli_arrays(c4.x, c4.z, c4.coef, c4.qubits, liecl.Method.orthonorm_dimonly,
                                             liecl.ClosureConfig(tolerance=1e-10)))
