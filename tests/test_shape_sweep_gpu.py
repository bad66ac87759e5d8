"""Randomised shape sweep through the C ABI: ~250 shapes (1..300 per extent, odd and
even, so both the TMA and the generic kernels and every tile config the chooser
picks are exercised), fp64 / fp32 bitwise vs the fused oracle, 3xTF32 within
tolerance, and the accumulate path (two k-panels) bitwise."""
import numpy as np
import pytest

from inputs import inputs as I
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _shapes(seed, count):
    rng = np.random.default_rng(seed)
    out = set()
    while len(out) < count:
        m, n, p = (int(x) for x in rng.integers(1, 301, size=3))
        if rng.random() < 0.5:  # bias towards TMA-eligible (even / multiple of 4) extents
            n, p = n + (-n) % 4, p + (-p) % 4
        out.add((m, n, p))
    return sorted(out)


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_random_shapes_bitwise(cuda_device, dt):
    import torch
    import paper_2306_11148_b200 as moa
    ndt = np.float64 if dt == "f64" else np.float32
    kinds = set()
    for i, (m, n, p) in enumerate(_shapes(100 if dt == "f64" else 200, 120)):
        A = I.host_matrix(m, n, 1000 + i, I.ID_A, dtype=ndt)
        B = I.host_matrix(n, p, 1000 + i, I.ID_B, dtype=ndt)
        tA, tB = torch.from_numpy(A).to(cuda_device), torch.from_numpy(B).to(cuda_device)
        C = moa.gemm(tA, tB)
        torch.cuda.synchronize()
        assert np.array_equal(C.cpu().numpy(), O.ip(A, B, fused=True)), (m, n, p)
        kinds.add(moa.plan(m, n, p, moa.F64 if dt == "f64" else moa.F32).kernel)
        if i % 10 == 0 and n >= 2:  # accumulate chain over two k-panels
            k1 = n // 2
            C2 = torch.empty_like(C)
            moa.gemm_acc(tA[:, :k1], tB[:k1], C2, accumulate=False)
            moa.gemm_acc(tA[:, k1:], tB[k1:], C2, accumulate=True)
            torch.cuda.synchronize()
            assert torch.equal(C2, C), (m, n, p, k1)
    assert len(kinds) >= 2, kinds  # both TMA and generic paths were exercised


def test_random_shapes_3xtf32(cuda_device):
    import torch
    import paper_2306_11148_b200 as moa
    for i, (m, n, p) in enumerate(_shapes(300, 60)):
        A = I.host_matrix(m, n, 3000 + i, I.ID_A, dtype=np.float32)
        B = I.host_matrix(n, p, 3000 + i, I.ID_B, dtype=np.float32)
        C = moa.gemm(torch.from_numpy(A).to(cuda_device), torch.from_numpy(B).to(cuda_device), precision="3xtf32")
        torch.cuda.synchronize()
        ref = O.ip_f32_truth(A, B)
        err = np.linalg.norm(C.cpu().numpy().astype(np.float64) - ref) / max(np.linalg.norm(ref), 1e-300)
        assert err <= 5e-3 and err <= 1e-5 * np.sqrt(n), (m, n, p, err)


def test_random_mid_shapes_bitwise(cuda_device):
    """Mid-size random shapes (m, p up to 1500, n up to 400): the chooser's wide tiles
    (128x128 / 128x64 / 64x64 / 64x32) with whole-tile waves, stream-K cut tiles and the
    wave-gate-free static schedule, fp64 bitwise vs the fused oracle."""
    import torch
    import paper_2306_11148_b200 as moa
    rng = np.random.default_rng(77)
    picks = set()
    i = 0
    while i < 16:
        m, p = (int(x) for x in rng.integers(200, 1501, size=2))
        n = int(rng.integers(8, 401))
        if rng.random() < 0.7:
            n, p = n + (-n) % 2, p + (-p) % 2
        if m * p < 148 * 64 * 32:  # latency regime: covered above
            continue
        i += 1
        A = I.host_matrix(m, n, 5000 + i, I.ID_A)
        B = I.host_matrix(n, p, 5000 + i, I.ID_B)
        C = moa.gemm(torch.from_numpy(A).to(cuda_device), torch.from_numpy(B).to(cuda_device))
        torch.cuda.synchronize()
        assert np.array_equal(C.cpu().numpy(), O.ip(A, B, fused=True)), (m, n, p)
        pl = moa.plan(m, n, p)
        picks.add((pl.kernel, pl.bm, pl.bn, pl.tiles > pl.grid and pl.tiles % max(pl.grid, 1) != 0))
    assert len({q[1:3] for q in picks if q[0] == "dgemm_tma"}) >= 2, picks
