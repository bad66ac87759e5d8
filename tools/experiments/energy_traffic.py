"""What K1's DRAM re-reads cost in joules (round-2 review item 7).

At m = n = p = N (default 16384) the rasterisation group of K1's tile schedule
(tile-rows per group) changes how often A/B panels are re-read from DRAM without
changing the arithmetic (bitwise identical C). This script times each group with CUDA
events and NVML energy over interleaved windows of >= 1.2 s (round-robin over the
groups, so thermal drift hits all of them alike) and prints, per group, the median
J/GEMM and its spread. Run the same groups under
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_dgemm_tma
(RASTER_NCU=1 runs one launch per group for that) to get the DRAM bytes; the slope
J per DRAM GB bounds what cutting the re-reads could save.

    python tools/experiments/energy_traffic.py [N] [groups]
"""
import dataclasses
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import pynvml  # noqa: E402
import torch  # noqa: E402

import paper_2306_11148_b200 as moa  # noqa: E402
from inputs import inputs as I  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
groups = [int(g) for g in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8,16").split(",")]
A = torch.empty((N, N), dtype=torch.float64, device="cuda")
B = torch.empty_like(A)
C = torch.empty_like(A)
I.device_fill(A, 1, I.ID_A)
I.device_fill(B, 1, I.ID_B)
ref = moa.gemm(A, B)
base = moa.plan(N, N, N)
plans = {g: dataclasses.replace(base, raster_group=g) for g in groups}
if os.environ.get("RASTER_NCU") == "1":
    for g in groups:
        moa.gemm_with_plan(A, B, C, plans[g])
    torch.cuda.synchronize()
    sys.exit(0)
pynvml.nvmlInit()
pr = torch.cuda.get_device_properties(0)
h = pynvml.nvmlDeviceGetHandleByPciBusId(("%08X:%02X:%02X.0" % (pr.pci_domain_id, pr.pci_bus_id,
                                                                  pr.pci_device_id)).encode())
for g in groups:
    moa.gemm_with_plan(A, B, C, plans[g])
    torch.cuda.synchronize()
    assert torch.equal(C, ref), g
t1 = 2.0 * N ** 3 / 36e12
reps = max(2, int(1.2 / t1) + 1)
rounds = int(os.environ.get("ROUNDS", "4"))
res = {g: [] for g in groups}
time.sleep(1.0)
e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
time.sleep(2.0)
idle_w = (pynvml.nvmlDeviceGetTotalEnergyConsumption(h) - e0) / 1e3 / 2.0
for r in range(rounds):
    for g in groups:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        a.record()
        for _ in range(reps):
            moa.gemm_with_plan(A, B, C, plans[g])
        b.record()
        torch.cuda.synchronize()
        e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        ms = a.elapsed_time(b) / reps
        res[g].append(((e1 - e0) / 1e3 / reps, ms))
for g in groups:
    js = sorted(x[0] for x in res[g])
    ms = statistics.median(x[1] for x in res[g])
    print(json.dumps({"N": N, "raster_group": g, "reps_per_window": reps, "windows": len(js),
                      "j_per_gemm_median": round(statistics.median(js), 3), "j_spread": [round(js[0], 3), round(js[-1], 3)],
                      "ms_median": round(ms, 3), "idle_w": round(idle_w, 1),
                      "j_above_idle": round(statistics.median(js) - idle_w * ms / 1e3, 3)}), flush=True)
