"""Short fp32 run for ncu: one exact FFMA and one 3xTF32 GEMM at N=8192 (after warm-up)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2306_11148_b200 as moa
from inputs import inputs as I
N = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
A = torch.empty((N, N), dtype=torch.float32, device="cuda"); B = torch.empty((N, N), dtype=torch.float32, device="cuda")
C = torch.empty((N, N), dtype=torch.float32, device="cuda")
I.device_fill(A, 1, I.ID_A); I.device_fill(B, 1, I.ID_B)
for prec in (None, "3xtf32"):
    for _ in range(2):
        moa.gemm(A, B, out=C, precision=prec)
torch.cuda.synchronize()
print("ok")
