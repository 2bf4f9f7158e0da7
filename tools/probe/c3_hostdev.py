"""Debug: config-3 verdicts from device vs pinned-host candidates."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2506_01120_b200 import liecl, workloads as w
dev = torch.device("cuda", 0)
c3 = w.Config3()
V, cands = c3.generate(torch, dev)
s = liecl.ClosureSession(c3.d, config=liecl.ClosureConfig(tolerance=c3.tol, max_dim=c3.n + c3.ncand))
res = []
host = torch.empty(cands.shape, dtype=cands.dtype, pin_memory=True)
host.copy_(cands)
torch.cuda.synchronize()
print("host copy equal:", bool((host.to(dev) == cands).all()), flush=True)
for mode in ("dev", "host", "dev", "host"):
    s.set_basis(V.data_ptr(), on_device=True, n=c3.n)
    ptr = cands.data_ptr() if mode == "dev" else host.data_ptr()
    ind, rn, st = s.check_candidates(ptr, on_device=(mode == "dev"), n=c3.ncand)
    res.append((mode, ind, rn))
    print(mode, int(ind.sum()), bool(ind[0::2].all()), int(ind[1::2].sum()), st["rechecks"], flush=True)
for i in range(1, 4):
    d = np.nonzero(res[i][1] != res[0][1])[0]
    print(res[i][0], "vs dev0: mismatches", len(d), d[:10].tolist(), "max |drn|", float(np.abs(res[i][2] - res[0][2]).max()))
