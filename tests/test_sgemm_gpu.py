"""GPU parity of the fp32 paths against the oracle (BASELINE configs[2]).

K3 (exact fp32, FFMA2): bitwise vs oracle ``ip(fused=True)`` in float32 on any
finite input (k ascending fma chain from +0), bitwise vs the literal oracle on
integer-valued inputs, and relative Frobenius <= 1e-5*sqrt(n) vs the literal
unfused ip.c. K4 (3xTF32 on tcgen05): <= 5e-3 vs the literal oracle (north_star,
reported separately), and its error vs the fp64-accumulated truth is reported.
"""
from __future__ import annotations

import numpy as np
import pytest

from inputs import inputs as I
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _moa():
    import paper_2306_11148_b200 as moa
    return moa


def _host(m, n, p, seed, kind=I.UNIFORM):
    return (I.host_matrix(m, n, seed, I.ID_A, kind, np.float32),
            I.host_matrix(n, p, seed, I.ID_B, kind, np.float32))


def _run(A, B, dev, precision=None):
    import torch
    C = _moa().gemm(torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev), precision=precision)
    torch.cuda.synchronize()
    return C.cpu().numpy()


def _relfro(x, ref):
    x = x.astype(np.float64)
    ref = ref.astype(np.float64)
    r = np.linalg.norm(ref)
    return np.linalg.norm(x - ref) / r if r > 0 else np.linalg.norm(x)


SHAPES = [(1, 1, 4), (7, 5, 3), (128, 32, 128), (129, 33, 130), (255, 64, 257), (256, 256, 256), (300, 100, 500),
          (17, 1000, 40), (1000, 4, 8)]


@pytest.mark.parametrize("seed", [1, 2])
def test_ffma_exact_bitwise(cuda_device, seed):
    for (m, n, p) in SHAPES:
        A, B = _host(m, n, p, seed)
        C = _run(A, B, cuda_device)
        assert np.array_equal(C, O.ip(A, B, fused=True)), (m, n, p)
        assert _relfro(C, O.ip(A, B, fused=False)) <= 1e-5 * np.sqrt(n), (m, n, p)


def test_ffma_integer_exact(cuda_device):
    for (m, n, p) in [(256, 256, 256), (129, 333, 131)]:
        A, B = _host(m, n, p, 3, kind=I.INT)
        assert np.array_equal(_run(A, B, cuda_device), O.ip(A, B, fused=False))


def test_ffma_identities(cuda_device):
    m, n, p = 200, 96, 132
    A, _ = _host(m, n, p, 4)
    assert np.array_equal(_run(A, np.eye(n, dtype=np.float32), cuda_device), A)
    assert np.array_equal(_run(np.eye(m, dtype=np.float32), A, cuda_device), A)


def test_ffma_row_block_invariance(cuda_device):
    import torch
    moa = _moa()
    m, n, p = 700, 300, 260
    A, B = _host(m, n, p, 5)
    tA, tB = torch.from_numpy(A).to(cuda_device), torch.from_numpy(B).to(cuda_device)
    full = moa.gemm(tA, tB)
    for (r0, r1) in [(0, 1), (5, 133), (128, 700)]:
        assert torch.equal(moa.gemm(tA[r0:r1].contiguous(), tB), full[r0:r1])


def test_ffma_config2_n16384_sampled_rows(cuda_device):
    """BASELINE configs[2] at full size (fp32 N=16384): sampled rows bitwise vs the oracle."""
    import torch
    moa = _moa()
    N = 16384
    tA = torch.empty((N, N), dtype=torch.float32, device=cuda_device)
    tB = torch.empty((N, N), dtype=torch.float32, device=cuda_device)
    I.device_fill(tA, 1, I.ID_A)
    I.device_fill(tB, 1, I.ID_B)
    C = moa.gemm(tA, tB)
    torch.cuda.synchronize()
    rows = [0, 127, 128, N - 1]
    B = I.host_matrix(N, N, 1, I.ID_B, dtype=np.float32)
    ref = O.ip_rowblock(I.host_rows(rows, N, 1, I.ID_A, dtype=np.float32), B, fused=True)
    assert np.array_equal(C[torch.tensor(rows, device=cuda_device)].cpu().numpy(), ref)


def test_plan_fp32(cuda_device):
    moa = _moa()
    assert moa.plan(16384, 16384, 16384, moa.F32).kernel == "sgemm_ffma"
    assert moa.plan(100, 101, 102, moa.F32).kernel == "sgemm_generic"


# ----------------------------------------------------------------- K4 3xTF32 --

def test_3xtf32_tolerance_and_truth_error(cuda_device):
    """<= 5e-3 relative Frobenius vs the literal oracle (north_star); the error vs the
    fp64-accumulated truth is reported (printed) separately."""
    moa = _moa()
    assert moa.plan(1024, 1024, 1024, moa.F32_3XTF32).kernel == "sgemm_3xtf32"
    for (m, n, p) in [(128, 32, 128), (129, 40, 132), (256, 256, 256), (300, 1000, 260), (1000, 4, 8)]:
        A, B = _host(m, n, p, 11)
        C = _run(A, B, cuda_device, precision="3xtf32")
        err_lit = _relfro(C, O.ip(A, B, fused=False))
        err_truth = _relfro(C, O.ip_f32_truth(A, B))
        print(f"3xtf32 {m}x{n}x{p}: rel err vs literal ip.c {err_lit:.3e}, vs fp64 truth {err_truth:.3e}")
        assert err_lit <= 5e-3, (m, n, p, err_lit)
        assert err_truth <= 1e-5 * np.sqrt(n), (m, n, p, err_truth)  # 3xTF32 ~ fp32-level accuracy


def test_3xtf32_config2_n16384_sampled_rows(cuda_device):
    """BASELINE configs[2] tensor-core variant at full size (fp32 N=16384, 3xTF32):
    sampled rows within the north_star 5e-3 of the literal ip.c and within fp32-level
    error of the fp64-accumulated truth; plus a Freivalds check of all of C."""
    import torch
    moa = _moa()
    N = 16384
    tA = torch.empty((N, N), dtype=torch.float32, device=cuda_device)
    tB = torch.empty((N, N), dtype=torch.float32, device=cuda_device)
    I.device_fill(tA, 1, I.ID_A)
    I.device_fill(tB, 1, I.ID_B)
    C = moa.gemm(tA, tB, precision="3xtf32")
    torch.cuda.synchronize()
    rows = [0, 127, 128, 8191, N - 1]
    B = I.host_matrix(N, N, 1, I.ID_B, dtype=np.float32)
    Ar = I.host_rows(rows, N, 1, I.ID_A, dtype=np.float32)
    got = C[torch.tensor(rows, device=cuda_device)].cpu().numpy()
    assert _relfro(got, O.ip_rowblock(Ar, B, fused=False)) <= 5e-3
    assert _relfro(got, O.ip_f32_truth(Ar, B)) <= 1e-5 * np.sqrt(N)
    x = torch.randint(0, 2, (N, 1), generator=torch.Generator().manual_seed(3)).to(tA) * 2 - 1
    y, z = C.double() @ x.double(), tA.double() @ (tB.double() @ x.double())
    assert float(torch.linalg.norm(y - z) / torch.linalg.norm(z)) <= 5e-3


def test_3xtf32_integer_inputs_exact(cuda_device):
    """Values in {-4..4} are exact in TF32 (small part 0) and every partial sum is an
    integer < 2^24: the tensor-core result must equal the oracle bit for bit (P6)."""
    for (m, n, p) in [(256, 256, 256), (130, 96, 260)]:
        A, B = _host(m, n, p, 12, kind=I.INT)
        assert np.array_equal(_run(A, B, cuda_device, precision="3xtf32"), O.ip(A, B, fused=False))


def test_3xtf32_each_tile_config(cuda_device):
    import torch
    moa = _moa()
    m, n, p = 300, 200, 520
    A, B = _host(m, n, p, 14)
    ref = O.ip(A, B, fused=False)
    tA, tB = torch.from_numpy(A).to(cuda_device), torch.from_numpy(B).to(cuda_device)
    base = moa.plan(m, n, p, moa.F32_3XTF32)
    for (bn, st) in [(256, 2), (192, 3), (128, 3)]:
        pl = moa.Plan(**{**base.__dict__, "bn": bn, "stages": st})
        out = torch.empty((m, p), dtype=torch.float32, device=cuda_device)
        moa.gemm_with_plan(tA, tB, out, pl, precision="3xtf32")
        torch.cuda.synchronize()
        assert _relfro(out.cpu().numpy(), ref) <= 5e-3
        assert _relfro(out.cpu().numpy(), O.ip_f32_truth(A, B)) <= 1e-5 * np.sqrt(n)


def test_3xtf32_identity(cuda_device):
    m, n, p = 256, 128, 384
    A, _ = _host(m, n, p, 13)
    # A•I = big*1 + small*1: big is exact in TF32, small keeps >= 11 of its <= 13 bits
    C = _run(A, np.eye(n, dtype=np.float32), cuda_device, precision="3xtf32")
    assert np.max(np.abs(C - A) / np.maximum(np.abs(A), 1e-30)) <= 2.0 ** -20
