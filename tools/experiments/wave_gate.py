"""A/B of K1's schedules: static (default) or dynamic tile claiming (MOA_K1_SCHED),
each with or without the wave gate (MOA_K1_WAVE_GATE). Per N: CUDA-event time and
NVML J/GEMM over a >= 1.2 s window, plus a checksum of C's bits (the schedule must
not change them). Each setting runs in its own process (the library reads the
variables once); rounds alternate the settings so drift hits all alike.

    python tools/experiments/wave_gate.py N[,N...] [ROUNDS] [SETTINGS]
SETTINGS: comma list of static_gate,static_nogate,dyn_gate,dyn_nogate (default all).
With WG_NCU=1: one launch per N only (for ncu's dram__bytes metrics).
"""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CHILD = r'''
import sys, os, json, time, hashlib
sys.path.insert(0, %r)
import torch, pynvml
import paper_2306_11148_b200 as moa
from inputs import inputs as I
out = []
for N in %r:
    A = torch.empty((N, N), dtype=torch.float64, device="cuda"); B = torch.empty_like(A); C = torch.empty_like(A)
    I.device_fill(A, 1, I.ID_A); I.device_fill(B, 1, I.ID_B)
    moa.gemm(A, B, out=C); torch.cuda.synchronize()
    if os.environ.get("WG_NCU") == "1":
        continue
    h = hashlib.sha1(C.view(torch.int64).sum(dim=1).cpu().numpy().tobytes()).hexdigest()[:12]
    pynvml.nvmlInit(); hd = pynvml.nvmlDeviceGetHandleByIndex(0)
    reps = max(2, int(1.2 / (2.0 * N ** 3 / 36e12)) + 1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(hd)
    a.record()
    for _ in range(reps): moa.gemm(A, B, out=C)
    b.record(); torch.cuda.synchronize()
    e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(hd)
    ms = a.elapsed_time(b) / reps
    out.append({"N": N, "setting": os.environ["WG_SETTING"], "ms": round(ms, 4),
                "tflops": round(2.0 * N ** 3 / ms / 1e9, 3), "j_per_gemm": round((e1 - e0) / 1e3 / reps, 3),
                "reps": reps, "bits": h})
    del A, B, C; torch.cuda.empty_cache()
print(json.dumps(out))
'''
sizes = [int(x) for x in sys.argv[1].split(",")]
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
settings = (sys.argv[3] if len(sys.argv) > 3 else "static_gate,static_nogate,dyn_gate,dyn_nogate").split(",")
for r in range(rounds):
    for st in settings:
        env = dict(os.environ, WG_SETTING=st, MOA_K1_SCHED="dynamic" if st.startswith("dyn") else "static",
                   MOA_K1_WAVE_GATE="0" if st.endswith("nogate") else "1")
        res = subprocess.run([sys.executable, "-c", CHILD % (ROOT, sizes)], env=env, capture_output=True, text=True)
        if res.returncode != 0:
            print(json.dumps({"setting": st, "error": res.stderr[-2000:]}), flush=True)
            continue
        if os.environ.get("WG_NCU") == "1":
            continue
        for d in json.loads(res.stdout.strip().splitlines()[-1]):
            d["round"] = r
            print(json.dumps(d), flush=True)
