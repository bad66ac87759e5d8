"""A/B timing of two libmoa.so builds in one process-free way: each run in a subprocess."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
code = r'''
import sys, os, json, ctypes
sys.path.insert(0, %r)
import torch
lib = ctypes.CDLL(%r)
lib.moa_gemm.argtypes = [ctypes.c_int64]*3 + [ctypes.c_void_p]*3 + [ctypes.c_int, ctypes.c_void_p]
from inputs import inputs as I
res = {}
for N in (4096, 16384):
    A = torch.empty((N, N), dtype=torch.float64, device="cuda"); B = torch.empty_like(A); C = torch.empty_like(A)
    I.device_fill(A, 1, I.ID_A); I.device_fill(B, 1, I.ID_B)
    f = lambda: lib.moa_gemm(N, N, N, A.data_ptr(), B.data_ptr(), C.data_ptr(), 0, None)
    for _ in range(3): f()
    torch.cuda.synchronize()
    reps = 40 if N == 4096 else 4
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    res[N] = round(2 * N**3 / (ms / 1e3) / 1e12, 3)
print(json.dumps(res))
'''
for rnd in range(2):
    for name in sys.argv[1:]:
        out = subprocess.run([sys.executable, "-c", code % (ROOT, name)], capture_output=True, text=True)
        print(name, out.stdout.strip(), out.stderr.strip()[-300:])
