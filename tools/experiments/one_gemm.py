"""Two fp64 moa_gemm calls through a given libmoa build (plain ctypes, no binding) —
for ncu captures of one build against another (-s 1 -c 1 takes the second).

    python tools/experiments/one_gemm.py LIB M N P
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from inputs import inputs as I  # noqa: E402

lib = ctypes.CDLL(os.path.abspath(sys.argv[1]))
lib.moa_gemm.argtypes = [ctypes.c_int64] * 3 + [ctypes.c_void_p] * 3 + [ctypes.c_int, ctypes.c_void_p]
m, n, p = (int(x) for x in sys.argv[2:5])
A = torch.empty((m, n), dtype=torch.float64, device="cuda")
B = torch.empty((n, p), dtype=torch.float64, device="cuda")
C = torch.empty((m, p), dtype=torch.float64, device="cuda")
I.device_fill(A, 1, I.ID_A)
I.device_fill(B, 1, I.ID_B)
s = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    assert lib.moa_gemm(m, n, p, A.data_ptr(), B.data_ptr(), C.data_ptr(), 0, s) == 0
torch.cuda.synchronize()
print("ok")
