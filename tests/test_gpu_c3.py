"""Config 3 at full size (N = 16384 basis vectors of D = 65536, 4096
candidates): size-independent properties, checked with cuBLAS (torch.matmul)
as an independent arithmetic. The oracle comparison of the same semantics at
a size the CPU finishes in seconds is test_gpu_parity.py::
test_ordered_check_candidates_vs_oracle."""
import numpy as np
import pytest

from paper_2506_01120_b200 import liecl
from paper_2506_01120_b200 import workloads as w

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def c3_run():
    import torch
    dev = torch.device("cuda", 0)
    c3 = w.Config3()
    V, cands = c3.generate(torch, dev)
    torch.cuda.synchronize(dev)  # the context's stream does not order against torch's
    s = liecl.ClosureSession(c3.d, config=liecl.ClosureConfig(tolerance=c3.tol, max_dim=c3.n + c3.ncand))
    s.set_basis(V.data_ptr(), on_device=True, n=c3.n)
    ind, rn, st = s.check_candidates(cands.data_ptr(), on_device=True, n=c3.ncand)
    torch.cuda.synchronize(dev)
    return torch, dev, c3, V, cands, s, ind, rn, st


def test_exactly_the_gaussian_candidates_are_accepted(c3_run):
    torch, dev, c3, V, cands, s, ind, rn, st = c3_run
    assert ind[0::2].all() and not ind[1::2].any()
    assert s.size() == c3.n + c3.ncand // 2
    assert st["independence_checks"] == c3.ncand
    # combination + 1e-14 noise: residual ~ 1e-15 after normalisation
    assert rn[1::2].max() < 1e-13
    # a Gaussian candidate keeps ~sqrt(1 - N/D) of its norm
    n_before = c3.n + np.arange(c3.ncand // 2)
    expect = np.sqrt(1.0 - n_before / c3.D)
    assert np.abs(rn[0::2] - expect).max() < 0.01


def test_first_accept_residual_matches_cublas(c3_run):
    torch, dev, c3, V, cands, s, ind, rn, st = c3_run
    c = cands[0]
    cu = c / (torch.linalg.vector_norm(c) / np.sqrt(c3.d))
    beta = (V.conj() @ cu) / c3.d
    r = cu - beta @ V
    beta2 = (V.conj() @ r) / c3.d
    r = r - beta2 @ V
    ref = float(torch.linalg.vector_norm(r)) / np.sqrt(c3.d)
    assert abs(rn[0] - ref) < 1e-12


def test_extended_basis_is_orthonormal(c3_run):
    torch, dev, c3, V, cands, s, ind, rn, st = c3_run
    k = c3.ncand // 2
    W = torch.empty((k, c3.D), dtype=torch.complex128, device=dev)
    s.vectors_to(c3.n, k, W.data_ptr())
    G = (W.conj() @ W.mT) / c3.d
    err_new = float((G - torch.eye(k, dtype=G.dtype, device=dev)).abs().max())
    cross = float(((V.conj() @ W.mT) / c3.d).abs().max())
    assert err_new < 1e-12 and cross < 1e-12
    # every accepted candidate lies in the span of the final basis
    acc = cands[0::2]
    cu = acc / (torch.linalg.vector_norm(acc, dim=1, keepdim=True) / np.sqrt(c3.d))
    r = cu - ((cu @ V.conj().mT) / c3.d) @ V
    r = r - ((r @ W.conj().mT) / c3.d) @ W
    assert float(torch.linalg.vector_norm(r, dim=1).max()) / np.sqrt(c3.d) < 1e-12
