"""GPU parity of the ipophp siblings (Hadamard, Kronecker) vs the oracle: bitwise
(one rounding per element), odd shapes, unaligned pointers, empty extents."""
import numpy as np
import pytest

from inputs import inputs as I
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_hadamard_bitwise(cuda_device, dt):
    import torch
    import paper_2306_11148_b200 as moa
    for (m, n) in [(1, 1), (7, 13), (256, 256), (1000, 777), (4096, 1024)]:
        A = I.host_matrix(m, n, 1, I.ID_A, dtype=dt)
        B = I.host_matrix(m, n, 1, I.ID_B, dtype=dt)
        C = moa.hadamard(torch.from_numpy(A).to(cuda_device), torch.from_numpy(B).to(cuda_device))
        torch.cuda.synchronize()
        assert np.array_equal(C.cpu().numpy(), O.hadamard(A, B)), (m, n)
    # unaligned (scalar path)
    A = I.host_matrix(33, 31, 2, I.ID_A, dtype=dt)
    B = I.host_matrix(33, 31, 2, I.ID_B, dtype=dt)
    tdt = torch.float64 if dt == np.float64 else torch.float32
    ba = torch.empty(33 * 31 + 1, dtype=tdt, device=cuda_device)
    bc = torch.empty(33 * 31 + 1, dtype=tdt, device=cuda_device)
    ta = ba[1:].view(33, 31)
    ta.copy_(torch.from_numpy(A))
    tc = bc[1:].view(33, 31)
    moa.hadamard(ta, torch.from_numpy(B).to(cuda_device), out=tc)
    torch.cuda.synchronize()
    assert np.array_equal(tc.cpu().numpy(), O.hadamard(A, B))


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_kron_bitwise(cuda_device, dt):
    import torch
    import paper_2306_11148_b200 as moa
    for (m, n, p, q) in [(1, 1, 1, 1), (1, 2, 1, 2), (3, 5, 4, 7), (16, 16, 32, 32), (5, 3, 100, 9), (64, 64, 64, 64)]:
        A = I.host_matrix(m, n, 3, I.ID_A, dtype=dt)
        B = I.host_matrix(p, q, 3, I.ID_B, dtype=dt)
        C = moa.kron(torch.from_numpy(A).to(cuda_device), torch.from_numpy(B).to(cuda_device))
        torch.cuda.synchronize()
        assert np.array_equal(C.cpu().numpy(), O.kron(A, B)), (m, n, p, q)


def test_empty_and_errors(cuda_device):
    import torch
    import paper_2306_11148_b200 as moa
    z = torch.empty((0, 5), dtype=torch.float64, device=cuda_device)
    assert moa.hadamard(z, z).shape == (0, 5)
    A = torch.ones((4, 4), dtype=torch.float64, device=cuda_device)
    with pytest.raises(moa.MoAError):
        moa.hadamard(A, A, out=A)
