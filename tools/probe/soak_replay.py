import os, sys, glob
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2506_01120_b200 import liecl
from oracle.oracle import Port
port = Port()
for f in sorted(glob.glob("tools/probe/soak_cases/soak_fail_*.npy")):
    gens = np.load(f)
    d = int(round(np.sqrt(gens.shape[1])))
    o = port.closure_dense(gens, d, keep_original=False, tol=1e-10)
    out = [os.path.basename(f), "d", d, "port", o.dimension]
    for field in ("auto", "complex"):
        for bs in (128, 512):
            try:
                r = liecl.closure_dense_arrays(gens, d, liecl.Method.orthonorm_dimonly,
                                               liecl.ClosureConfig(tolerance=1e-10, field=field, batch_max=bs))
                out += [f"{field}/b{bs}", r.dimension]
            except Exception as e:
                out += [f"{field}/b{bs}", type(e).__name__]
    print(*out, os.environ.get("LIECL_B200_BLOCK_GS", "1"), flush=True)
