"""A/B of the C-store cost in K1: the product library vs a timing-only build whose
consumers skip the epilogue stores (-DMOA_EXPERIMENT_NO_STORE, wrong results).
fp64 shapes with shallow to deep k per tile; CUDA events, median of 5 windows."""
import ctypes, json, os, statistics, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
code = r'''
import sys, json, ctypes, statistics
sys.path.insert(0, %r)
import torch
lib = ctypes.CDLL(%r)
lib.moa_gemm.argtypes = [ctypes.c_int64]*3 + [ctypes.c_void_p]*3 + [ctypes.c_int, ctypes.c_void_p]
from inputs import inputs as I
res = {}
for (m, n, p) in [(65536, 512, 512), (16384, 1024, 1024), (4096, 4096, 4096), (8192, 8192, 8192)]:
    A = torch.empty((m, n), dtype=torch.float64, device="cuda"); B = torch.empty((n, p), dtype=torch.float64, device="cuda")
    C = torch.empty((m, p), dtype=torch.float64, device="cuda")
    I.device_fill(A, 1, I.ID_A); I.device_fill(B, 1, I.ID_B)
    f = lambda: lib.moa_gemm(m, n, p, A.data_ptr(), B.data_ptr(), C.data_ptr(), 0, None)
    for _ in range(3): f()
    torch.cuda.synchronize()
    reps = max(3, int(0.3 / (2.0 * m * n * p / 36e12)))
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps): f()
        b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / reps)
    ms = statistics.median(ts)
    res["%%dx%%dx%%d" %% (m, n, p)] = {"ms": round(ms, 4), "tflops": round(2 * m * n * p / (ms / 1e3) / 1e12, 3)}
print(json.dumps(res))
'''
for rnd in range(2):
    for name in sys.argv[1:]:
        out = subprocess.run([sys.executable, "-c", code % (ROOT, name)], capture_output=True, text=True)
        print(name, out.stdout.strip(), out.stderr.strip()[-300:])
