"""Parity at the largest sizes the path is meant for (SURVEY §8(a) size table).

* N = 32768 fp64 square on one GPU: the north_star's lifted size (8 GiB per
  matrix, 24 GiB resident; 2048 k-slabs per tile; dynamic tiles + stream-K runs).
* 2^20 x 64 x 96: tall, > 65536 tile rows of work, row coordinates up to 2^20.

Checks: sampled rows x sampled columns of C bitwise vs the fused ip.c oracle
(`oracle.ip_rowblock` on the sampled rows of A and the sampled columns of B —
rows and columns of C are independent, Fig. 1), plus a Freivalds product
check of every element. The sampled B columns are read back from the device
input buffer, which the seeded input generator (inputs/, no GEMM arithmetic)
wrote; host and device generators are bit-identical (tests/test_inputs.py).
"""
from __future__ import annotations

import numpy as np
import pytest

from inputs import inputs as I
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _freivalds(Ct, tA, tB, trials=2):
    import torch
    worst = 0.0
    for t in range(trials):
        g = torch.Generator(device="cpu").manual_seed(4321 + t)
        x = (torch.randint(0, 2, (Ct.shape[1], 1), generator=g) * 2 - 1).to(Ct)
        y = Ct @ x
        z = tA @ (tB @ x)
        worst = max(worst, float(torch.linalg.norm(y - z) / torch.linalg.norm(z)))
    return worst


@pytest.mark.parametrize("shape", [(32768, 32768, 32768), (1 << 20, 64, 96)])
def test_max_size_sampled_bitwise(cuda_device, shape):
    import torch

    import paper_2306_11148_b200 as moa
    m, n, p = shape
    seed = 5
    tA = torch.empty((m, n), dtype=torch.float64, device=cuda_device)
    tB = torch.empty((n, p), dtype=torch.float64, device=cuda_device)
    I.device_fill(tA, seed, I.ID_A)
    I.device_fill(tB, seed, I.ID_B)
    C = moa.gemm(tA, tB)
    torch.cuda.synchronize()
    rng = np.random.default_rng(1)
    rows = sorted(r for r in {0, 1, 127, 128, m // 2, m - 129, m - 1, *rng.integers(0, m, size=5).tolist()} if r < m)
    cols = sorted(c for c in {0, 15, 16, 127, 128, p // 2, p - 1, *rng.integers(0, p, size=25).tolist()} if c < p)
    Arows = I.host_rows(rows, n, seed, I.ID_A)
    Bcols = tB[:, torch.tensor(cols, device=cuda_device)].contiguous().cpu().numpy()
    ref = O.ip_rowblock(Arows, Bcols, fused=True)
    got = C[torch.tensor(rows, device=cuda_device)][:, torch.tensor(cols, device=cuda_device)].cpu().numpy()
    assert got.shape == ref.shape and bool(np.all(got == ref))
    assert _freivalds(C, tA, tB) <= 1e-12 * np.sqrt(n)
    pl = moa.plan(m, n, p)
    assert pl.tiles == -(-m // pl.bm) * -(-p // pl.bn)
