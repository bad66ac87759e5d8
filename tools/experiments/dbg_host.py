import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2306_11148_b200 as moa
from inputs import inputs as I
from oracle import oracle as O
for (m, n, p) in [(4000, 256, 2048), (4000, 1024, 2048), (8192, 512, 512), (333, 128, 210)]:
    A = I.host_matrix(m, n, 9, I.ID_A); B = I.host_matrix(n, p, 9, I.ID_B)
    hA = torch.from_numpy(A).pin_memory(); hB = torch.from_numpy(B).pin_memory()
    hC = torch.full((m, p), float("nan"), dtype=torch.float64).pin_memory()
    dA = torch.empty((m, n), dtype=torch.float64, device="cuda"); dB = torch.empty((n, p), dtype=torch.float64, device="cuda")
    dC = torch.empty((m, p), dtype=torch.float64, device="cuda")
    moa.gemm_host(hA, hB, hC, dA, dB, dC)
    ref = O.ip(A, B, fused=True)
    got = hC.numpy()
    bad = np.argwhere(~(got == ref))
    print((m, n, p), "plan", moa.plan(m, n, p).tiles_n, "bad", len(bad), bad[:3].tolist(), "rows with nan", int(np.isnan(got).any(axis=1).sum()))
    if len(bad):
        rows = sorted(set(bad[:, 0].tolist()))
        print("   bad row range", rows[0], rows[-1], "count", len(rows))
