"""Regression test for a cold-first-launch race (dynamic tile scheduling):
each fresh process runs the first launch of several kernel instantiations under
dynamic scheduling on uninitialised outputs and checks the bits against the oracle."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys
sys.path.insert(0, %r)
import numpy as np, torch
import paper_2306_11148_b200 as moa
from inputs import inputs as I
from oracle import oracle as O
bad = 0
for (m, n, p) in [(1984, 256, 2048), (4000, 256, 2048), (2048, 512, 2048)]:
    A = I.host_matrix(m, n, 9, I.ID_A); B = I.host_matrix(n, p, 9, I.ID_B)
    C = moa.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    torch.cuda.synchronize()
    bad += int((C.cpu().numpy() != O.ip(A, B, fused=True)).sum())
print("BAD", bad)
"""


def test_cold_first_launches_in_fresh_processes(cuda_device):
    for _ in range(4):
        out = subprocess.run([sys.executable, "-c", CHILD % ROOT], capture_output=True, text=True, timeout=300)
        assert "BAD 0" in out.stdout, out.stdout + out.stderr[-2000:]
