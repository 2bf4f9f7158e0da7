"""Quick config-2 timing probe: growth phase via a session, then saturated windows."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2506_01120_b200 import liecl, workloads as w

cfg = w.config2()
s = liecl.ClosureSession(64, config=liecl.ClosureConfig(tolerance=1e-10))
t = time.time()
ind, rn, st = s.check_candidates(cfg.generators)
print("gens", ind, st["kernels"])
st = s.run_rows(1, 101)
print("growth rows 1..100: dim", s.size(), "t", time.time() - t, st)
for rows in [(1000, 1004), (2000, 2004), (3000, 3003)]:
    t = time.time()
    st = s.run_rows(*rows)
    dt = time.time() - t
    print(rows, "pairs", st["commutators_evaluated"], "checks", st["independence_checks"], "acc", st["accepted"],
          "survivors", st["survivors"], "t %.3f s" % dt, "brackets/s %.0f" % (st["commutators_evaluated"] / dt),
          "TFLOP/s(alg) %.2f" % (st["commutators_evaluated"] * (16 * 64**3 + 16 * 4095 * 4096) / dt / 1e12))
