#!/usr/bin/env python3
"""Measure every BASELINE.json config on one B200 (not the driver's bench line).

  configs[0] fp64 m=n=p=256                 configs[1] fp64 N sweep 1024..8192 (+16384 target)
  configs[2] fp32 N=16384 exact vs 3xTF32   configs[3] fp64 65536x512x512
plus the paper's block-size experiment (Figs. 3-8 analogue): every
compiled tile config at each N, time and J/GEMM, with the static chooser's pick.
Timing: CUDA events around R back-to-back launches after 3 warm-ups, R sized so a
window lasts >= ~1 s (NVML energy granularity); inputs resident in HBM.
Output: one JSON document on stdout.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2306_11148_b200 as moa  # noqa: E402
from bench import FP64_DMMA_PEAK_TFLOPS, ClockSampler  # noqa: E402
from inputs import inputs as I  # noqa: E402

FFMA_PEAK_TFLOPS = 74.0  # measured FFMA2, 16 chains/thread (profiles/r01_ffma_mix_probe.jsonl); 74.4 nominal
TF32_NOMINAL_TFLOPS = 1100.0  # B200_PROFILING.md nominal dense TF32


def timed(fn, window_s, sampler, est_s):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    reps = max(3, int(window_s / max(est_s, 1e-6)))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0 = sampler.energy_mj()
    with sampler:
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
    e1 = sampler.energy_mj()
    ms = a.elapsed_time(b) / reps
    out = {"ms": round(ms, 5), "reps": reps}
    if e0 is not None and e1 is not None:
        out["j_per_gemm"] = round((e1 - e0) / 1e3 / reps, 6)
        out["avg_w"] = round((e1 - e0) / 1e3 / (ms * reps / 1e3), 1)
        if IDLE_W[0] is not None:
            out["j_per_gemm_above_idle"] = round(((e1 - e0) / 1e3 - IDLE_W[0] * ms * reps / 1e3) / reps, 6)
    summ = sampler.summary()
    out["temp_c_max"] = summ.get("temp_c_max")
    out["sm_mhz"] = summ.get("sm_mhz")
    out["power_w_median"] = summ.get("power_w_median")
    out["throttle"] = summ.get("reasons")
    return out


IDLE_W = [None]


def mats(m, n, p, dtype):
    A = torch.empty((m, n), dtype=dtype, device="cuda")
    B = torch.empty((n, p), dtype=dtype, device="cuda")
    C = torch.empty((m, p), dtype=dtype, device="cuda")
    I.device_fill(A, 1, I.ID_A)
    I.device_fill(B, 1, I.ID_B)
    return A, B, C


def rec(m, n, p, r, peak):
    fl = 2.0 * m * n * p
    r["gflops"] = round(fl / (r["ms"] / 1e3) / 1e9, 1)
    r["frac_of_peak"] = round(fl / (r["ms"] / 1e3) / 1e12 / peak, 4)
    if peak == FP64_DMMA_PEAK_TFLOPS and r.get("sm_mhz"):
        # DMMA nominal at the SM clock the window actually ran at: 148 SMs x 128 flop/clk
        r["frac_of_nominal_at_clock"] = round(fl / (r["ms"] / 1e3) / (148 * 128 * r["sm_mhz"] * 1e6), 4)
    r["hbm_gbs_algorithmic"] = None
    return r


HBM_GBS = 6535.7  # MEASURED_PEAKS.json hbm_gbs (copy, read+write)


def ipophp(a, sampler):
    """Hadamard and Kronecker (NEXT-4) against the HBM roofline: algorithmic bytes
    (each input read once, output written once) / time."""
    res = {}
    N = 16384
    A = torch.empty((N, N), dtype=torch.float64, device="cuda")
    B = torch.empty_like(A)
    C = torch.empty_like(A)
    I.device_fill(A, 1, I.ID_A)
    I.device_fill(B, 1, I.ID_B)
    r = timed(lambda: moa.hadamard(A, B, out=C), a.window, sampler, 3 * 8 * N * N / 6e12)
    byts = 3 * 8 * N * N
    r.update({"shape": [N, N], "bytes": byts, "gbs": round(byts / (r["ms"] / 1e3) / 1e9, 1)})
    r["frac_of_hbm"] = round(r["gbs"] / HBM_GBS, 4)
    res["hadamard_f64_16384"] = r
    del A, B
    Ak = torch.empty((128, 128), dtype=torch.float64, device="cuda")
    Bk = torch.empty((128, 128), dtype=torch.float64, device="cuda")
    I.device_fill(Ak, 1, I.ID_A)
    I.device_fill(Bk, 1, I.ID_B)
    r = timed(lambda: moa.kron(Ak, Bk, out=C), a.window, sampler, 8 * N * N / 6e12)
    byts = 8 * (N * N + 2 * 128 * 128)
    r.update({"shape": "128x128 (x) 128x128 -> 16384x16384", "bytes": byts,
              "gbs": round(byts / (r["ms"] / 1e3) / 1e9, 1)})
    r["frac_of_hbm"] = round(r["gbs"] / HBM_GBS, 4)
    res["kron_f64_128x128_128x128"] = r
    # write-only ceiling reference on the same buffer (driver memset, not our kernel)
    w = timed(lambda: C.zero_(), a.window, sampler, 8 * N * N / 6e12)
    w_gbs = round(8 * N * N / (w["ms"] / 1e3) / 1e9, 1)
    res["write_ceiling_memset_16384"] = {"ms": w["ms"], "gbs": w_gbs}
    r["frac_of_write_ceiling"] = round(r["gbs"] / w_gbs, 4)
    del C
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--window", type=float, default=1.0)
    ap.add_argument("--sizes", default="1024,1536,2048,3072,4096,6144,8192,16384")
    ap.add_argument("--skip-blocks", action="store_true")
    ap.add_argument("--sections", default="c0,c1,c2,c3,ipophp")
    a = ap.parse_args()
    secs = set(a.sections.split(","))
    sampler = ClockSampler(0, period=0.1)
    torch.cuda.synchronize()
    IDLE_W[0] = sampler.idle_watts(2.0)  # 2 s idle window
    out = {"idle_w": IDLE_W[0]}
    out.update({"device": torch.cuda.get_device_name(0), "fp64_peak_tflops": FP64_DMMA_PEAK_TFLOPS,
           "ffma_peak_tflops": FFMA_PEAK_TFLOPS, "time": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())})

    if "ipophp" in secs:
        out["ipophp"] = ipophp(a, sampler)
    # configs[0]
    if "c0" in secs:
        A, B, C = mats(256, 256, 256, torch.float64)
        r = timed(lambda: moa.gemm(A, B, out=C), a.window, sampler, 5e-6)
        out["config0_fp64_256"] = rec(256, 256, 256, r, FP64_DMMA_PEAK_TFLOPS)
        out["config0_fp64_256"]["plan"] = moa.plan(256, 256, 256).__dict__

    # configs[1] sweep + block-size experiment
    sweep = []
    for N in ([int(x) for x in a.sizes.split(",")] if "c1" in secs else []):
        A, B, C = mats(N, N, N, torch.float64)
        est = 2.0 * N ** 3 / (FP64_DMMA_PEAK_TFLOPS * 0.9e12)
        pl = moa.plan(N, N, N)
        r = rec(N, N, N, timed(lambda: moa.gemm(A, B, out=C), a.window, sampler, est), FP64_DMMA_PEAK_TFLOPS)
        r.update({"N": N, "plan": {"bm": pl.bm, "bn": pl.bn, "stages": pl.stages, "grid": pl.grid,
                                   "tiles": pl.tiles}, "clocks": sampler.summary()})
        sampler.samples = []
        if not a.skip_blocks:
            blocks = []
            for (bm, bn, st) in [(128, 128, 6), (128, 64, 4), (64, 64, 4), (64, 32, 4), (16, 32, 4), (16, 16, 4)]:
                q = moa.Plan(**{**pl.__dict__, "bm": bm, "bn": bn, "stages": st, "grid": 0})
                rb = rec(N, N, N, timed(lambda: moa.gemm_with_plan(A, B, C, q), min(a.window, 0.5), sampler, est),
                         FP64_DMMA_PEAK_TFLOPS)
                rb.update({"bm": bm, "bn": bn, "stages": st, "chosen": (bm, bn) == (pl.bm, pl.bn)})
                blocks.append(rb)
            best = min(blocks, key=lambda x: x["ms"])
            r["block_sweep"] = blocks
            r["chooser_vs_best"] = round(best["ms"] / next(x["ms"] for x in blocks if x["chosen"]), 4)
        sweep.append(r)
        del A, B, C
        torch.cuda.empty_cache()
    out["config1_fp64_sweep"] = sweep
    import math
    pts = [(x["N"], x["j_per_gemm"]) for x in sweep if x.get("j_per_gemm") and x["N"] <= 8192]
    if len(pts) >= 3:
        xs, ys = [math.log(x) for x, _ in pts], [math.log(y) for _, y in pts]
        mx, my = sum(xs) / len(xs), sum(ys) / len(ys)
        out["energy_exponent_fit_1024_8192"] = round(
            sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs), 3)

    if "c2" in secs:
        fp32_section(a, sampler, out)
    if "c3" in secs:
        skinny_section(a, sampler, out)
    json.dump(out, sys.stdout, indent=1)
    print()


def fp32_section(a, sampler, out):
    # configs[2] fp32 N=16384
    N = 16384
    A, B, C = mats(N, N, N, torch.float32)
    r = rec(N, N, N, timed(lambda: moa.gemm(A, B, out=C), a.window, sampler, 2.0 * N ** 3 / 60e12), FFMA_PEAK_TFLOPS)
    r["kernel"] = moa.plan(N, N, N, moa.F32).kernel
    out["config2_fp32_16384_exact"] = r
    try:
        r = rec(N, N, N, timed(lambda: moa.gemm(A, B, out=C, precision="3xtf32"), a.window, sampler,
                               2.0 * N ** 3 / 200e12), TF32_NOMINAL_TFLOPS / 3)
        r["kernel"] = moa.plan(N, N, N, moa.F32_3XTF32).kernel
        r["peak_note"] = "frac against TF32 nominal / 3 (three TF32 products per output term)"
        out["config2_fp32_16384_3xtf32"] = r
        base = moa.plan(N, N, N, moa.F32_3XTF32)
        blocks = []
        for (bn, st) in [(256, 2), (192, 3), (128, 3)]:
            q = moa.Plan(**{**base.__dict__, "bn": bn, "stages": st})
            rb = rec(N, N, N, timed(lambda: moa.gemm_with_plan(A, B, C, q, precision="3xtf32"), a.window, sampler,
                                    2.0 * N ** 3 / 200e12), TF32_NOMINAL_TFLOPS / 3)
            rb.update({"bn": bn, "stages": st, "variant": "TS (A in TMEM)" if bn != 128 else "SS",
                       "clocks": sampler.summary()})
            sampler.samples = []
            blocks.append(rb)
        r["block_sweep"] = blocks
    except moa.MoAError as e:
        out["config2_fp32_16384_3xtf32"] = {"error": str(e)}
    del A, B, C
    torch.cuda.empty_cache()


def skinny_section(a, sampler, out):
    # configs[3] skinny
    m, n, p = 65536, 512, 512
    A, B, C = mats(m, n, p, torch.float64)
    r = rec(m, n, p, timed(lambda: moa.gemm(A, B, out=C), a.window, sampler, 2.0 * m * n * p / 33e12),
            FP64_DMMA_PEAK_TFLOPS)
    byts = 8 * (m * n + n * p + m * p)
    r["hbm_gbs_algorithmic"] = round(byts / (r["ms"] / 1e3) / 1e9, 1)
    r["plan"] = moa.plan(m, n, p).__dict__
    out["config3_fp64_65536x512x512"] = r


if __name__ == "__main__":
    main()
