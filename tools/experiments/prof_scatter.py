"""One 8192^3 fp64 GEMM with the fused-gather epilogue to 7 local destinations (the
G = 8 store pattern) for an ncu capture: DMMA activity and DRAM writes (8x C)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2306_11148_b200 as moa  # noqa: E402
from inputs import inputs as I  # noqa: E402

N = 8192
A = torch.empty((N, N), dtype=torch.float64, device="cuda")
B = torch.empty_like(A)
I.device_fill(A, 1, I.ID_A)
I.device_fill(B, 1, I.ID_B)
C = torch.empty_like(A)
dst = [torch.empty_like(A) for _ in range(7)]
for _ in range(2):
    moa.gemm_scatter(A, B, C, dst)
torch.cuda.synchronize()
print("ok")
