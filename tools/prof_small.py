"""Small-N fp64 runs for ncu: each compiled tile config at N (default 2048)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2306_11148_b200 as moa
from inputs import inputs as I
N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
A = torch.empty((N, N), dtype=torch.float64, device="cuda"); B = torch.empty_like(A); C = torch.empty_like(A)
I.device_fill(A, 1, I.ID_A); I.device_fill(B, 1, I.ID_B)
base = moa.plan(N, N, N)
for (bm, bn, st) in [(128, 128, 6), (64, 64, 4)]:
    q = moa.Plan(**{**base.__dict__, "bm": bm, "bn": bn, "stages": st})
    for _ in range(3):
        moa.gemm_with_plan(A, B, C, q)
torch.cuda.synchronize()
print("ok")
