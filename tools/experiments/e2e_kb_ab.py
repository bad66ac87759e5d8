"""A/B of the e2e host pipeline (moa_gemm_host) between two libmoa builds in one
process (ctypes, RTLD_LOCAL: separate symbol namespaces), alternating, at BASELINE
configs[4]'s 32768^3 fp64 with pinned host buffers. One JSON line per (lib, rep)."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from inputs import inputs as I  # noqa: E402

N = int(os.environ.get("E2E_N", "32768"))
libs = sys.argv[1:]
L = []
for p in libs:
    l = ctypes.CDLL(os.path.abspath(p))
    l.moa_gemm_host.argtypes = [ctypes.c_int64] * 3 + [ctypes.c_void_p] * 6 + [ctypes.c_int, ctypes.c_void_p]
    L.append(l)
A = torch.empty((N, N), dtype=torch.float64, device="cuda")
B = torch.empty((N, N), dtype=torch.float64, device="cuda")
C = torch.empty((N, N), dtype=torch.float64, device="cuda")
I.device_fill(A, 1, I.ID_A)
I.device_fill(B, 1, I.ID_B)
hA, hB, hC = (torch.empty((N, N), dtype=torch.float64).pin_memory() for _ in range(3))
hA.copy_(A)
hB.copy_(B)
torch.cuda.synchronize()
s = torch.cuda.current_stream().cuda_stream
for rep in range(4):
    for p, l in zip(libs, L):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        rc = l.moa_gemm_host(N, N, N, hA.data_ptr(), hB.data_ptr(), hC.data_ptr(), A.data_ptr(), B.data_ptr(),
                             C.data_ptr(), 0, s)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        print(json.dumps({"lib": os.path.basename(p), "rep": rep, "rc": rc, "ms": round(ms, 2),
                          "tflops": round(2.0 * N ** 3 / ms / 1e9, 3)}), flush=True)
