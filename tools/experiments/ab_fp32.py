"""A/B timing of fp32 exact GEMM (K3) between libmoa builds, each in its own subprocess."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
code = r'''
import sys, json, ctypes
sys.path.insert(0, %r)
import torch
lib = ctypes.CDLL(%r)
lib.moa_gemm.argtypes = [ctypes.c_int64]*3 + [ctypes.c_void_p]*3 + [ctypes.c_int, ctypes.c_void_p]
from inputs import inputs as I
res = {}
for N in (8192, 16384):
    A = torch.empty((N, N), dtype=torch.float32, device="cuda"); B = torch.empty_like(A); C = torch.empty_like(A)
    I.device_fill(A, 1, I.ID_A); I.device_fill(B, 1, I.ID_B)
    f = lambda: lib.moa_gemm(N, N, N, A.data_ptr(), B.data_ptr(), C.data_ptr(), 1, None)
    for _ in range(2): f()
    torch.cuda.synchronize()
    reps = 10 if N == 8192 else 3
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    res[N] = round(2 * N**3 / (ms / 1e3) / 1e12, 3)
    res["bits" + str(N)] = int(C.view(torch.int32).to(torch.int64).sum().item())  # equal bits across builds
print(json.dumps(res))
'''
for rnd in range(2):
    for name in sys.argv[1:]:
        out = subprocess.run([sys.executable, "-c", code % (ROOT, name)], capture_output=True, text=True)
        print(name, out.stdout.strip(), out.stderr.strip()[-300:])
