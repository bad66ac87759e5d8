"""A/B timing of libmoa.so builds on a list of fp64 shapes, each build in its own
subprocess, alternating builds over R rounds (same box, same inputs).

    python tools/experiments/ab_shapes.py SHAPES LIB [LIB ...]
SHAPES: "m,n,p;m,n,p;..."  LIB: path to a libmoa build (e.g. ab/libmoa_pre_desc.so)
One JSON line per (round, lib): {lib, round, shape: TF/s}. Bitwise equality of C
across builds is checked through a checksum of the bits.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CODE = r'''
import sys, json, ctypes, hashlib
sys.path.insert(0, %r)
import torch
lib = ctypes.CDLL(%r)
lib.moa_gemm.argtypes = [ctypes.c_int64] * 3 + [ctypes.c_void_p] * 3 + [ctypes.c_int, ctypes.c_void_p]
from inputs import inputs as I
import os
DT = int(os.environ.get("AB_DTYPE", "0"))  # 0 fp64, 1 exact fp32, 2 3xTF32 (moa.h moa_dtype)
tt = torch.float64 if DT == 0 else torch.float32
res, sums = {}, {}
for (m, n, p) in %r:
    A = torch.empty((m, n), dtype=tt, device="cuda"); B = torch.empty((n, p), dtype=tt, device="cuda")
    C = torch.empty((m, p), dtype=tt, device="cuda")
    I.device_fill(A, 1, I.ID_A); I.device_fill(B, 1, I.ID_B)
    s = torch.cuda.current_stream().cuda_stream
    f = lambda: lib.moa_gemm(m, n, p, A.data_ptr(), B.data_ptr(), C.data_ptr(), DT, s)
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); f(); b.record(); torch.cuda.synchronize()
    est = max(a.elapsed_time(b), 1e-3)
    reps = max(5, int(600 / est))
    a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    key = "%%dx%%dx%%d" %% (m, n, p)
    res[key] = round(2 * m * n * p / (ms / 1e3) / 1e12, 3)
    sums[key] = hashlib.sha1(C.view(torch.int64 if DT == 0 else torch.int32).cpu().numpy().tobytes()).hexdigest()[:12]
print(json.dumps({"tflops": res, "bits": sums}))
'''


def main():
    shapes = [tuple(int(x) for x in s.split(",")) for s in sys.argv[1].split(";") if s]
    libs = sys.argv[2:]
    rounds = int(os.environ.get("AB_ROUNDS", "2"))
    for rnd in range(rounds):
        for spec in libs:
            # LIB[@VAR=VAL,...]: extra environment for this build's process (e.g. MOA_K1_WAVE_GATE=0)
            lib, _, envs = spec.partition("@")
            env = dict(os.environ, **dict(kv.split("=", 1) for kv in envs.split(",") if kv))
            out = subprocess.run([sys.executable, "-c", CODE % (ROOT, os.path.abspath(lib), shapes)],
                                 capture_output=True, text=True, env=env)
            try:
                d = json.loads(out.stdout.strip().splitlines()[-1])
            except Exception:
                d = {"error": out.stderr[-500:]}
            print(json.dumps({"lib": os.path.basename(lib) + ("@" + envs if envs else ""), "round": rnd, **d}),
                  flush=True)


if __name__ == "__main__":
    main()
