#!/usr/bin/env python3
"""Host-side cost per call of the binding / C ABI pieces (wall clock, GPU not the
bottleneck: tiny shapes, many calls, one sync at the end)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_11148_b200 as moa  # noqa: E402

N = 64
A = torch.ones((N, N), dtype=torch.float64, device="cuda")
B = torch.ones_like(A)
C = torch.empty_like(A)
pl = moa.plan(N, N, N)
lib = moa._lib
s = torch.cuda.current_stream().cuda_stream


def per_call(fn, reps=20000):
    for _ in range(100):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e6


out = {}
out["ctypes_abi_version"] = per_call(lambda: lib.moa_abi_version())
pt = moa._PlanT()
out["c_moa_plan"] = per_call(lambda: lib.moa_plan(ctypes.c_int64(N), ctypes.c_int64(N), ctypes.c_int64(N), 0, -1, ctypes.byref(pt)))
a, b, c = A.data_ptr(), B.data_ptr(), C.data_ptr()
out["c_moa_gemm_raw_ptrs"] = per_call(lambda: lib.moa_gemm(ctypes.c_int64(N), ctypes.c_int64(N), ctypes.c_int64(N),
                                                         ctypes.c_void_p(a), ctypes.c_void_p(b), ctypes.c_void_p(c), 0,
                                                         ctypes.c_void_p(s)))
out["py_moa_gemm_out"] = per_call(lambda: moa.gemm(A, B, out=C))
out["torch_add_inplace"] = per_call(lambda: C.add_(1.0))
print(out)
