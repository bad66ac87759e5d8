#!/usr/bin/env python3
"""One launch of the product kernel for a BASELINE config, for an ncu --set full capture
(tools/gpu_prof_configs.sh). The first call warms up (plan, attributes, L2); ncu skips
it with -s 1 and captures the second.

    python tools/prof_configs.py <config>
configs: c0 (fp64 256^3), c3 (fp64 65536x512x512), c16k (fp64 16384^3),
         f32 (exact fp32 16384^3), tf32 (3xTF32 16384^3), had (Hadamard fp64 16384^2),
         kron (Kronecker fp64 128^2 x 128^2), l1/l2/l4/l8 (rank 0's rows of configs[4] at G)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2306_11148_b200 as moa  # noqa: E402
from inputs import inputs as I  # noqa: E402

SHAPES = {"c0": (256, 256, 256, torch.float64), "c3": (65536, 512, 512, torch.float64),
          "c16k": (16384, 16384, 16384, torch.float64), "c8k": (8192, 8192, 8192, torch.float64), "f32": (16384, 16384, 16384, torch.float32),
          "tf32": (16384, 16384, 16384, torch.float32), "had": (16384, 16384, 0, torch.float64),
          "kron": (128, 128, 128, torch.float64),
          # BASELINE configs[4]: rank 0's rows of the row-lifted 32768^3 at G = 1, 2, 4, 8
          "l1": (32768, 32768, 32768, torch.float64), "l2": (16384, 32768, 32768, torch.float64),
          "l4": (8192, 32768, 32768, torch.float64), "l8": (4096, 32768, 32768, torch.float64)}


def main(cfg):
    m, n, p, dt = SHAPES[cfg]
    if cfg == "had":
        A = torch.empty((m, n), dtype=dt, device="cuda")
        B = torch.empty_like(A)
        I.device_fill(A, 1, I.ID_A)
        I.device_fill(B, 1, I.ID_B)
        C = torch.empty_like(A)
        fn = lambda: moa.hadamard(A, B, out=C)  # noqa: E731
    elif cfg == "kron":
        A = torch.empty((m, n), dtype=dt, device="cuda")
        B = torch.empty((p, p), dtype=dt, device="cuda")
        I.device_fill(A, 1, I.ID_A)
        I.device_fill(B, 1, I.ID_B)
        C = torch.empty((m * p, n * p), dtype=dt, device="cuda")
        fn = lambda: moa.kron(A, B, out=C)  # noqa: E731
    else:
        A = torch.empty((m, n), dtype=dt, device="cuda")
        B = torch.empty((n, p), dtype=dt, device="cuda")
        I.device_fill(A, 1, I.ID_A)
        I.device_fill(B, 1, I.ID_B)
        C = torch.empty((m, p), dtype=dt, device="cuda")
        prec = "3xtf32" if cfg == "tf32" else None
        fn = lambda: moa.gemm(A, B, out=C, precision=prec)  # noqa: E731
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    print(cfg, "ok", moa.plan(m, n, max(p, 1), 0 if dt == torch.float64 else (2 if cfg == "tf32" else 1)))


if __name__ == "__main__":
    main(sys.argv[1])
