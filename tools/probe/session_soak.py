"""Session soak: random bases and candidate streams through ClosureSession
(check_candidates in random chunks, numpy or pinned host pointers; run_rows
windows), verdicts against the C restatement (oracle Port, test-only)."""
import os, sys, random, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2506_01120_b200 import liecl
from oracle.oracle import Port

port = Port()
SEED = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ITERS = int(sys.argv[2]) if len(sys.argv) > 2 else 60
rng = np.random.default_rng(SEED); random.seed(SEED)
fails = []


def ortho_basis(d, n, antiherm):
    D = d * d
    vs = []
    while len(vs) < n:
        a = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
        if antiherm:
            a = a - a.conj().T
        v = a.ravel(order="F")
        for _ in range(2):
            for u in vs:
                v = v - (np.vdot(u, v) / d) * u
        nv = np.sqrt(np.vdot(v, v).real / d)
        if nv > 1e-3:
            vs.append(v / nv)
    return np.array(vs) if vs else np.zeros((0, D), complex)


t0 = time.time()
for it in range(ITERS):
    d = random.choice([4, 8, 16, 32, 64])
    D = d * d
    antiherm = random.random() < 0.6
    n = int(rng.integers(0, min(D - 8, 600)))
    V = ortho_basis(d, n, antiherm)
    # candidates: independent, in-span + 1e-14 noise, repeats of earlier ones
    cands = []
    for k in range(int(rng.integers(1, 80))):
        kind = rng.integers(0, 3)
        if kind == 0 or n == 0:
            a = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
            if antiherm:
                a = a - a.conj().T
            c = a.ravel(order="F")
        elif kind == 1:
            w = rng.standard_normal(n) * (1.0 if not antiherm else 1.0)
            c = w @ V + 1e-14 * (rng.standard_normal(D) + (0 if antiherm else 1j * rng.standard_normal(D)))
            if antiherm:  # keep it exactly anti-Hermitian
                m = c.reshape(d, d, order="F"); m = (m - m.conj().T) / 2; c = m.ravel(order="F")
        else:
            c = cands[int(rng.integers(0, len(cands)))] if cands else V[0]
        nc = np.sqrt(np.vdot(c, c).real / d)
        cands.append(c / nc)
    cands = np.array(cands)
    want_ind, want_rn, _ = port.check_sequence_dense(V, cands, d, tol=1e-10, append=True)
    s = liecl.ClosureSession(d, config=liecl.ClosureConfig(tolerance=1e-10, batch_max=random.choice([0, 1, 7, 64])))
    mode = random.choice(["numpy", "pinned", "prefetch"])
    if n:
        s.set_basis(V)
    got_ind, got_rn = [], []
    pos = 0
    pinned = torch.from_numpy(cands.copy()).pin_memory() if mode != "numpy" else None
    chunks = []
    while pos < len(cands):
        k = int(rng.integers(1, len(cands) - pos + 1))
        chunks.append((pos, k))
        pos += k
    if mode == "prefetch":  # chunk i+1's H2D in flight while chunk i is checked
        s.prefetch_candidates(pinned.data_ptr() + chunks[0][0] * D * 16, chunks[0][1])
    for i, (p0, k) in enumerate(chunks):
        if mode == "numpy":
            ind, rn, _ = s.check_candidates(cands[p0:p0 + k])
        else:
            if mode == "prefetch" and i + 1 < len(chunks):
                q0, qk = chunks[i + 1]
                s.prefetch_candidates(pinned.data_ptr() + q0 * D * 16, qk)
            ind, rn, _ = s.check_candidates(pinned.data_ptr() + p0 * D * 16, n=k)
        got_ind += list(ind); got_rn += list(rn)
    got_ind, got_rn = np.array(got_ind), np.array(got_rn)
    ok = np.array_equal(got_ind, want_ind) and np.allclose(got_rn, want_rn, rtol=1e-9, atol=1e-12)
    ok = ok and s.size() == n + int(want_ind.sum())
    # a bracket window on the resulting basis (rows [r0, r1))
    if ok and s.size() >= 3 and s.size() < 120:
        B = s.basis()
        r0 = int(rng.integers(1, s.size())); r1 = min(s.size(), r0 + int(rng.integers(1, 4)))
        nul, ind2, rn2 = port.bracket_window_dense(B, d, r0, r1, tol=1e-10)
        st = s.run_rows(r0, r1)
        # the restatement checks the window against the fixed basis, run_rows
        # appends as it goes: comparable is whether the window accepts at all
        ok = (st["accepted"] == 0) == (int(ind2.sum()) == 0)
        if not ok:
            print("WINDOW", it, d, antiherm, st, int(ind2.sum()), flush=True)
    if not ok:
        fails.append((it, d, antiherm, n, len(cands), mode))
        print("FAIL", it, "d", d, "antiherm", antiherm, "n", n, "cands", len(cands), mode,
              "ind diff", np.nonzero(got_ind != want_ind)[0][:5], flush=True)
    s.close()
print({"seed": SEED, "iterations": ITERS, "failures": fails, "seconds": round(time.time() - t0, 1)})
