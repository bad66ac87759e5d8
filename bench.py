#!/usr/bin/env python3
"""Benchmark of the B200 MoA-ONF fp64 GEMM (arXiv 2306.11148) — driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl moa|reference] [--N 8192]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1: row-lifted path)

One "step" = one C := A • B (Eq. 3) over inputs resident in HBM.
N = 1: square fp64 GEMM m = n = p = 8192 (BASELINE configs[1], the top of the
paper's energy-vs-N sweep shape), through moa_gemm.
N > 1: the row-lifted path (moa_gemm_lifted): rank g owns 8192 rows of A and C
(weak scaling: m = 8192·N), n = p = 8192, B is broadcast from rank 0 over NVLink
with NCCL every step (the path's one real exchange, reading R13).
--gather nccl|fused adds the optional all-gather of C (reading R14): ncclAllGather
after the GEMM, or fused into the GEMM epilogue (moa_gemm_lifted_gather: NVLink
peer stores into NCCL symmetric windows). --lifted runs the lifted path at N = 1
too (a 1-rank NCCL communicator), which exercises the N > 1 code on one GPU.

Rank 0 prints ONE JSON line: value = GFLOP/s of the whole job (all ranks' flops
÷ the max-over-ranks device time of exactly K steps), plus roofline (DMMA fp64
tensor peak), e2e (the same metric through moa_gemm_host / host buffers with the
H2D and D2H copies inside the timed region), cpu_baseline (the oracle on this
host's cores on a bounded row sample), energy (NVML joules per GEMM), an N sweep
(GFLOP/s and J/GEMM vs N, the paper's time/energy-vs-N study), clocks.
"""
from __future__ import annotations

import argparse
import faulthandler
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# fp64 tensor-core (DMMA.8x8x4) peak measured on this pool's B200 by tools/probe
# (profiles/r01_fp64_probe.jsonl: 37.0 TF/s at 1965 MHz, flat from 4 to 32 warps/SM,
# held for a 125 ms sustained run). MEASURED_PEAKS.json carries no fp64 figure.
FP64_DMMA_PEAK_TFLOPS = 37.0
FP64_PEAK_SOURCE = "measured DMMA.8x8x4 microbenchmark, profiles/r01_fp64_probe.jsonl (MEASURED_PEAKS.json has no fp64 entry)"
METRIC = "fp64 GEMM GFLOP/s (joules/GEMM vs N in energy/sweep)"
DATA = "synthetic (seeded splitmix64 uniform[-1,1), inputs/)"


def workload_config(N, ws, lifted=False, gather="none"):
    """The config object both arms report (same workload, same keys)."""
    rows = N
    m_total = rows * ws
    lifted = lifted or ws > 1
    gtxt = {"none": "", "nccl": ", C all-gathered with NCCL after the GEMM",
            "fused": ", C all-gathered inside the GEMM epilogue (NVLink peer stores)"}[gather]
    return {"workload": f"square fp64 GEMM m=n=p={N} per GPU (BASELINE configs[1], top of the 1024-8192 sweep)"
                        + ("" if not lifted else f"; row-lifted over {ws} GPUs, m={m_total}, NCCL broadcast of B each step"
                           + gtxt),
            "m": m_total, "n": N, "p": N, "rows_per_rank": rows,
            "parallelism": "single GPU" if not lifted else
            f"row-lifted x{ws} ({'moa_gemm_lifted_gather' if gather == 'fused' else 'moa_gemm_lifted'})",
            "gather": gather,
            "l2": f"inputs larger than L2 ({(rows * N + N * N + rows * N) * 8 / 2**20:.0f} MiB resident vs 126 MB L2), no flush"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["moa", "reference"], default="moa")
    ap.add_argument("--N", type=int, default=8192, help="square size per rank (rows per rank = N)")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sweep-sizes", default="1024,1536,2048,3072,4096,6144,8192")
    ap.add_argument("--lifted", action="store_true",
                    help="use the row-lifted (communicator) path even at N=1 (a 1-rank NCCL communicator)")
    ap.add_argument("--gather", choices=["none", "nccl", "fused"], default="none",
                    help="lifted path: also all-gather C (after the GEMM with NCCL, or fused into its epilogue)")
    return ap.parse_args()


# ----------------------------------------------------------------- helpers --

class ClockSampler:
    """NVML sampling of SM clock / power / throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int, period: float = 0.05):
        self.ok = False
        self.samples = []
        self.reasons = 0
        self.period = period
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = self._handle(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - NVML absent
            self.err = str(e)

    def _handle(self, device_index):
        import torch
        nv = self.nv
        try:  # map CUDA device -> NVML by PCI bus id (CUDA_VISIBLE_DEVICES order != NVML order)
            pr = torch.cuda.get_device_properties(device_index)
            bus = "%08X:%02X:%02X.0" % (int(pr.pci_domain_id), int(pr.pci_bus_id), int(pr.pci_device_id))
            return nv.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            pass
        return nv.nvmlDeviceGetHandleByIndex(device_index)

    def energy_mj(self):
        if not self.ok:
            return None
        try:
            return self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h)
        except Exception:
            return None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                tc = nv.nvmlDeviceGetTemperature(self.h, nv.NVML_TEMPERATURE_GPU)
                self.samples.append((sm, pw, rs, tc))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._stop = threading.Event()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"]}
        loaded = [s for s in self.samples if not (s[2] & 0x1)] or self.samples
        mask = 0
        for s in loaded:
            mask |= s[2]
        reasons = [name for bit, name in self.REASONS.items() if mask & bit and bit != 0x1]
        return {"sm_mhz": statistics.median(s[0] for s in loaded), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "power_w_median": round(statistics.median(s[1] for s in loaded), 1),
                "temp_c_median": statistics.median(s[3] for s in loaded), "temp_c_max": max(s[3] for s in loaded),
                "samples": len(loaded)}

    def idle_watts(self, seconds: float = 1.0):
        """Idle-power baseline: NVML energy over a quiet window (J/s)."""
        e0 = self.energy_mj()
        if e0 is None:
            return None
        t0 = time.perf_counter()
        time.sleep(seconds)
        e1 = self.energy_mj()
        return round((e1 - e0) / 1e3 / (time.perf_counter() - t0), 1)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------ cpu baseline --

def _oracle_sample_rows(want: int, m: int, cores: int) -> tuple[int, int]:
    """(rows, threads) for a bounded oracle sample: ip_rows.c needs np | rows."""
    threads = max(1, min(cores, m))
    rows = max(threads, min(want, m)) // threads * threads
    return rows, threads


def cpu_oracle_sample(m, n, p, seed=1, target_s=12.0, max_rows=None):
    """Time the CPU oracle as it stands on this host's cores: Fig. 4 ip_rows.c (row
    lifting, one thread per host core, literal unfused ip.c update in each) on a
    bounded row sample of the workload. Rows of C are independent (Fig. 1) and
    each costs 2·n·p flops, so GFLOP/s over the sample is the oracle's rate on the
    whole job. The single-thread ip.c rate is reported beside it."""
    from inputs import inputs as I
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    B = I.host_matrix(n, p, seed, I.ID_B)
    A1 = I.host_matrix(1, n, seed, I.ID_A)
    t0 = time.perf_counter()
    O.ip_rowblock(A1, B)
    t1 = time.perf_counter() - t0
    want = int(target_s * cores / max(t1, 1e-6))
    if max_rows:
        want = min(want, max_rows)
    rows, threads = _oracle_sample_rows(want, m, cores)
    A = I.host_matrix(rows, n, seed, I.ID_A)
    t0 = time.perf_counter()
    O.ip_rows(A, B, threads)
    dt = time.perf_counter() - t0
    return {"value": round(2.0 * rows * n * p / dt / 1e9, 4), "unit": "GFLOP/s", "cores": threads, "kind": "oracle",
            "sample": f"{rows} of {m} rows of the m=n=p={n} fp64 workload, Fig. 4 ip_rows.c over {threads} threads "
                      f"(literal unfused ip.c update), {dt:.1f} s; host nproc={cores}",
            "seconds": round(dt, 2), "single_thread_gflops": round(2.0 * n * p / t1 / 1e9, 4)}


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, bounded sample per step."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from inputs import inputs as I
    from oracle import oracle as O
    N = args.N
    m = N * max(1, args.gpus)
    n = p = N
    cores = os.cpu_count() or 1
    B = I.host_matrix(n, p, 1, I.ID_B)
    A1 = I.host_matrix(1, n, 1, I.ID_A)
    t0 = time.perf_counter()
    O.ip_rowblock(A1, B)
    t_row = time.perf_counter() - t0
    total_budget = 150.0  # seconds for warmup + steps
    want = int(total_budget * cores / max(t_row, 1e-6) / (args.steps + args.warmup))
    rows_per_step, threads = _oracle_sample_rows(want, m, cores)
    A = I.host_matrix(rows_per_step, n, 1, I.ID_A)
    for _ in range(args.warmup):
        O.ip_rows(A, B, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.ip_rows(A, B, threads)
    dt = time.perf_counter() - t0
    value = 2.0 * rows_per_step * n * p * args.steps / dt / 1e9
    cfg = workload_config(N, max(1, args.gpus))
    cfg["reference_sample"] = (f"each step runs the CPU oracle (Fig. 4 ip_rows.c over {threads} threads, literal "
                               f"unfused ip.c update) on a bounded sample of {rows_per_step} of the {m} rows; "
                               f"GFLOP/s = 2*rows*n*p / time")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4),
        "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": cfg,
        "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": threads, "kind": "oracle",
                         "sample": f"{rows_per_step} rows x {args.steps} steps of the m=n=p={N} workload, "
                                   f"ip_rows.c over {threads} threads"},
        "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


# ----------------------------------------------------------------- GPU arm --

_JSON_FD = None


def _quiet_stdout():
    """Route fd 1 to stderr for the whole run: native libraries (NCCL prints its
    version banner on communicator init on some boxes) must not add lines to the ONE
    JSON line the driver parses; emit() writes that line to the original stdout."""
    global _JSON_FD
    if _JSON_FD is None:
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


def emit(line: dict):
    sys.stdout.flush()
    os.write(_JSON_FD if _JSON_FD is not None else 1, (json.dumps(line) + "\n").encode())


def main():
    faulthandler.enable()
    _quiet_stdout()
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_2306_11148_b200 as moa
    from inputs import inputs as I

    ws, rank, local = dist_env()
    lifted = ws > 1 or args.lifted or args.gather != "none"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if lifted:
        if ws == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()

    N = args.N
    n = p = N
    rows = N                      # rows of A/C per rank (weak scaling)
    m_total = rows * ws
    row0 = rank * rows
    A = torch.empty((rows, n), dtype=torch.float64, device=dev)
    B = torch.empty((n, p), dtype=torch.float64, device=dev)
    C = torch.empty((rows, p), dtype=torch.float64, device=dev)
    I.device_fill(A, 1, I.ID_A, row0=row0)
    if rank == 0:
        I.device_fill(B, 1, I.ID_B)
    else:
        B.zero_()
    comm = moa.Comm() if lifted else None
    C_full = None
    if args.gather == "fused":
        C_full = comm.alloc_window((m_total, p))       # NCCL symmetric window
    elif args.gather == "nccl":
        C_full = torch.empty((m_total, p), dtype=torch.float64, device=dev)

    def step():
        if comm is None:
            moa.gemm(A, B, out=C)
        elif args.gather == "fused":
            moa.gemm_lifted_gather(m_total, A, B, C_full, comm)
        else:
            moa.gemm_lifted(m_total, A, B, C, comm, C_full=C_full)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    torch.cuda.synchronize()
    idle_w = sampler.idle_watts(1.0)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if lifted:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = sampler.energy_mj()
    with sampler:
        t_start.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
        e1 = sampler.energy_mj()
    if lifted:
        dist.barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    per_step = [a.elapsed_time(b) for a, b in ev]
    if ws > 1:
        t = torch.tensor([elapsed_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    flops_step = 2.0 * m_total * n * p
    value = flops_step * args.steps / (elapsed_ms / 1e3) / 1e9  # GFLOP/s whole job

    # dominant kernel (the GEMM itself) on the launching stream; on the lifted path the
    # step also holds the B broadcast (and any gather), so time moa_gemm alone on this
    # rank's rows afterwards.
    if lifted:
        kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
        for a, b in kev:
            a.record(stream)
            moa.gemm(A, B, out=C)
            b.record(stream)
        torch.cuda.synchronize()
        kern_ms = statistics.mean(a.elapsed_time(b) for a, b in kev)
    else:
        kern_ms = statistics.mean(per_step)
    kflops = 2.0 * rows * n * p
    achieved_tf = kflops / (kern_ms / 1e3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_k1_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(str(N))
        except Exception:
            traffic = None
    plan = moa.plan(rows, n, p)

    # energy (NVML; J per GEMM step summed over every participating GPU)
    energy = None
    if ws > 1:
        t = torch.tensor([float((e1 - e0) if (e0 is not None and e1 is not None) else -1e30)], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        e0, e1 = (0.0, float(t.item())) if t.item() >= 0 else (None, None)
    if e0 is not None and e1 is not None:
        j = (e1 - e0) / 1e3
        idle_j = (idle_w or 0.0) * ws * (elapsed_ms / 1e3)
        energy = {"j_per_gemm": round(j / args.steps, 4), "idle_w": idle_w,
                  "j_per_gemm_above_idle": round((j - idle_j) / args.steps, 4) if idle_w is not None else None,
                  "window_s": round(elapsed_ms / 1e3, 3),
                  "avg_w": round(j / (elapsed_ms / 1e3), 1), "gflops_per_w": round(value / (j / (elapsed_ms / 1e3)), 2)}

    # e2e through moa_gemm_host (host buffers, copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        hA = torch.empty((rows, n), dtype=torch.float64).pin_memory()
        hB = torch.empty((n, p), dtype=torch.float64).pin_memory()
        hC = torch.empty((rows, p), dtype=torch.float64).pin_memory()
        hA.copy_(A.cpu())
        hB.copy_(B.cpu())
        k_e2e = max(1, min(args.steps, 5))
        if ws > 1:
            dist.barrier()

        def e2e_step():
            if comm is None:
                moa.gemm_host(hA, hB, hC, A, B, C)
            else:
                moa.gemm_lifted_host(m_total, hA, hB if rank == 0 else None, hC, A, B, C, comm)
        e2e_step()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(k_e2e):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        e2e_ms = a.elapsed_time(b)
        if ws > 1:
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        h2d = (rows * n + (n * p if rank == 0 or ws == 1 else 0)) * 8
        e2e = {"value": round(flops_step * k_e2e / (e2e_ms / 1e3) / 1e9, 2), "unit": "GFLOP/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": rows * p * 8, "steps": k_e2e,
               "ms_per_step": round(e2e_ms / k_e2e, 3),
               "api": "moa_gemm_host" if comm is None else "moa_gemm_lifted_host"}

    # N sweep (GFLOP/s and J/GEMM vs N), rank 0 at N = 1 only
    sweep = None
    if ws == 1 and not args.no_sweep:
        sweep = []
        for Ns in [int(x) for x in args.sweep_sizes.split(",") if x]:
            As = torch.empty((Ns, Ns), dtype=torch.float64, device=dev)
            Bs = torch.empty((Ns, Ns), dtype=torch.float64, device=dev)
            Cs = torch.empty((Ns, Ns), dtype=torch.float64, device=dev)
            I.device_fill(As, 1, I.ID_A)
            I.device_fill(Bs, 1, I.ID_B)
            for _ in range(3):
                moa.gemm(As, Bs, out=Cs)
            torch.cuda.synchronize()
            est = 2.0 * Ns ** 3 / (FP64_DMMA_PEAK_TFLOPS * 0.8e12)
            reps = max(5, int(1.0 / est))  # >= ~1 s window for NVML energy granularity
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0 = sampler.energy_mj()
            a.record(stream)
            for _ in range(reps):
                moa.gemm(As, Bs, out=Cs)
            b.record(stream)
            torch.cuda.synchronize()
            s1 = sampler.energy_mj()
            ms = a.elapsed_time(b) / reps
            rec = {"N": Ns, "ms": round(ms, 4), "gflops": round(2.0 * Ns ** 3 / (ms / 1e3) / 1e9, 1),
                   "frac_of_peak": round(2.0 * Ns ** 3 / (ms / 1e3) / 1e12 / FP64_DMMA_PEAK_TFLOPS, 4), "reps": reps,
                   "l2": "warm (back-to-back launches)" if 3 * 8 * Ns * Ns < 126e6 else "inputs larger than L2"}
            if s0 is not None and s1 is not None:
                rec["j_per_gemm"] = round((s1 - s0) / 1e3 / reps, 5)
            if 3 * 8 * Ns * Ns < 126e6:
                # cold variant: a 256 MiB write flushes L2 before each launch;
                # events bracket the GEMM alone
                flush = torch.empty(32 * 2 ** 20, dtype=torch.float64, device=dev)
                cold = []
                for _ in range(10):
                    flush.fill_(1.0)
                    a.record(stream)
                    moa.gemm(As, Bs, out=Cs)
                    b.record(stream)
                    torch.cuda.synchronize()
                    cold.append(a.elapsed_time(b))
                del flush
                rec["cold_l2_ms"] = round(statistics.median(cold), 4)
            sweep.append(rec)
            del As, Bs, Cs
        pts = [(r["N"], r.get("j_per_gemm")) for r in sweep if r.get("j_per_gemm")]
        if len(pts) >= 3:
            import math
            xs = [math.log(x) for x, _ in pts]
            ys = [math.log(y) for _, y in pts]
            mx, my = sum(xs) / len(xs), sum(ys) / len(ys)
            slope = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs)
            sweep = {"points": sweep, "energy_exponent_fit": round(slope, 3),
                     "paper_claim": "energy quadratic in N (P:14-15)"}
        else:
            sweep = {"points": sweep}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu = cpu_oracle_sample(m_total, n, p)

    if comm is not None:
        comm.close()
    if lifted:
        dist.destroy_process_group()
    if rank != 0:
        return 0
    cfg = workload_config(N, ws, lifted, args.gather)
    cfg["plan"] = {"kernel": plan.kernel, "bm": plan.bm, "bn": plan.bn, "bk": plan.bk, "stages": plan.stages,
                   "grid": plan.grid, "tiles": plan.tiles}
    line = {
        "metric": METRIC, "value": round(value, 2),
        "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(elapsed_ms / args.steps, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": cfg,
        "roofline": {"bound": "tensor", "achieved": round(achieved_tf, 3), "peak": FP64_DMMA_PEAK_TFLOPS,
                     "unit": "TFLOP/s", "frac": round(achieved_tf / FP64_DMMA_PEAK_TFLOPS, 4),
                     "traffic": traffic, "kernel": "k_dgemm_tma (fp64 DMMA)", "kernel_ms": round(kern_ms, 4),
                     "algorithmic_flops_per_launch": kflops, "peak_source": FP64_PEAK_SOURCE},
        "components": {"step_ms": round(elapsed_ms / args.steps, 4), "gemm_ms": round(kern_ms, 4),
                       "exchange_ms": round(max(0.0, elapsed_ms / args.steps - kern_ms), 4)},
        "e2e": e2e,
        "gpu_launches": args.steps,
        "energy": energy,
        "sweep": sweep,
        "clocks": sampler.summary(),
        "cpu_baseline": cpu,
    }
    emit(line)
    return 0


if __name__ == "__main__":
    sys.exit(main())
