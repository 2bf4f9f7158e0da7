"""Saturated-window throughput at one GPU for different batch caps
(ClosureConfig.batch_max): 8,192 (default), 7,104 = 3 x 37 column tiles and
9,472 = 4 x 37 (whole waves of the 32 x N-tile GEMM grids on 296 slots)."""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
import torch
from paper_2506_01120_b200 import liecl
from bench import random_saturated_basis
V = random_saturated_basis(64, 0)
for bm in (0, 8192, 7104, 9472, 8192, 9472):
    s = liecl.ClosureSession(64, config=liecl.ClosureConfig(tolerance=1e-10, batch_max=bm))
    s.set_basis(V)
    s.run_rows(1000, 1016)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    br = s.run_rows(1024, 1088)["commutators_evaluated"]
    torch.cuda.synchronize()
    long_rate = br / (time.perf_counter() - t0)
    t0 = time.perf_counter()
    br = 0
    for k in range(20):
        br += s.run_rows(1100 + 8 * k, 1108 + 8 * k)["commutators_evaluated"]
    torch.cuda.synchronize()
    win_rate = br / (time.perf_counter() - t0)
    print(json.dumps({"batch_max": bm, "one_64_row_window": round(long_rate), "twenty_8_row_windows": round(win_rate)}),
          flush=True)
    s.close()
