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


def test_wave_gate_many_waves_sampled_bitwise(cuda_device):
    """K1's wave gate is on from 48 whole-tile waves (moa_dgemm.cu kK1GateWaves):
    16384 x 48 x 16384 is 110 waves of 128x128 tiles with ragged k (3 slabs, the last
    half empty) and a stream-K tail — gated; sampled entries bitwise vs the fused ip.c
    oracle, every entry by Freivalds."""
    import torch

    import paper_2306_11148_b200 as moa
    m, n, p = 16384, 40, 16384
    seed = 9
    pl = moa.plan(m, n, p)
    assert pl.bm * pl.bn == 128 * 128 and pl.tiles >= 48 * pl.grid, pl
    tA = torch.empty((m, n), dtype=torch.float64, device=cuda_device)
    tB = torch.empty((n, p), dtype=torch.float64, device=cuda_device)
    I.device_fill(tA, seed, I.ID_A)
    I.device_fill(tB, seed, I.ID_B)
    C = moa.gemm(tA, tB)
    torch.cuda.synchronize()
    rng = np.random.default_rng(3)
    rows = sorted({0, 127, 128, m // 2, m - 1, *rng.integers(0, m, size=12).tolist()})
    cols = sorted({0, 127, 128, p - 1, *rng.integers(0, p, size=30).tolist()})
    ref = O.ip_rowblock(I.host_rows(rows, n, seed, I.ID_A),
                        tB[:, torch.tensor(cols, device=cuda_device)].contiguous().cpu().numpy(), fused=True)
    got = C[torch.tensor(rows, device=cuda_device)][:, torch.tensor(cols, device=cuda_device)].cpu().numpy()
    assert bool(np.all(got == ref))
    assert _freivalds(C, tA, tB) <= 1e-12 * np.sqrt(n)


_GATE_CHILD = r'''
import hashlib, json, sys
sys.path.insert(0, %r)
import torch
import paper_2306_11148_b200 as moa
from inputs import inputs as I
out = {}
for (m, n, p) in [(2000, 200, 2000), (4000, 64, 4000), (7040, 16, 7040)]:
    A = torch.empty((m, n), dtype=torch.float64, device="cuda"); B = torch.empty((n, p), dtype=torch.float64, device="cuda")
    I.device_fill(A, 2, I.ID_A); I.device_fill(B, 2, I.ID_B)
    C = moa.gemm(A, B); torch.cuda.synchronize()
    out["%%dx%%dx%%d" %% (m, n, p)] = hashlib.sha1(C.view(torch.int64).cpu().numpy().tobytes()).hexdigest()
print(json.dumps(out))
'''


def test_wave_gate_forced_modes_same_bits(cuda_device):
    """MOA_K1_WAVE_GATE=1 forces the gate on every multi-wave launch (here 2.7 to 20
    waves, with stream-K tails), =0 forces it off: the schedule only changes when a
    producer may issue, never the k order, so all three modes give identical bits."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for mode in ("0", "1", None):
        env = dict(os.environ)
        env.pop("MOA_K1_WAVE_GATE", None)
        if mode is not None:
            env["MOA_K1_WAVE_GATE"] = mode
        r = subprocess.run([sys.executable, "-c", _GATE_CHILD % root], env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        res[mode] = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["0"] == res["1"] == res[None], res
