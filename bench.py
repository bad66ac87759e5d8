#!/usr/bin/env python3
"""Benchmark of the B200 MoA-ONF fp64 GEMM (arXiv 2306.11148) — driver contract.

    python bench.py [--gpus G] [--steps K] [--warmup W] [--impl moa|reference] [--N 32768]
    torchrun --nproc-per-node G bench.py --gpus G ...   (the same; bench.py self-launches
                                                          its G ranks when WORLD_SIZE is unset)

Workload: BASELINE configs[4] — the row-lifted fp64 GEMM m = n = p = 32768 on G B200
("Dimension lifting over the rows of A and C ... assigns an index to
processors"; Fig. 4 ip_rows.c P:150-171), STRONG scaling: the total problem is fixed
and rank g owns rows moa_lift_rows(32768, G, g) of A and C. One "step" is one
C := A • B (Eq. 3) through moa_gemm_lifted with inputs resident in HBM:
B travels from rank 0 to every rank each step (P:165 — B carries no processor index),
then each rank computes its rows. At G = 1 the same call runs on a 1-rank
communicator (nothing travels).

The exchange of B (G > 1): copy-engine pulls of B's k-panels from rank 0's symmetric
window over NVLink (moa_pull_panels; no SMs taken from the GEMM), overlapped with the
k-panel chain of the rank's GEMM. The NCCL-broadcast exchange (pipelined k-panels on a
CTA-limited communicator) is measured beside it in "exchange_variants"; if the pulled
exchange fails on a box, the NCCL one is the headline and the line says so.

Rank 0 prints ONE JSON line: value = GFLOP/s of the whole job (2·m·n·p per step ÷ the
max-over-ranks device time of exactly K steps), with the per-step component breakdown
(compute alone, exchange alone, exposed exchange), roofline (the K1 DMMA kernel on the
rank's rows), e2e (the same metric through moa_gemm_host / moa_gemm_lifted_host with
host buffers, copies inside the timed region), energy (NVML J per GEMM summed over
ranks, raw and idle-subtracted), at G = 1 the paper's time/energy-vs-N sweep (1024 …
8192, 16000 = the paper's largest N, 16384 = the north_star's target; ≥ 3 windows of
≥ 1 s each) with the fitted energy exponent, cpu_baseline (the oracle on this host's
cores on a bounded row sample) and clocks.
"""
from __future__ import annotations

import argparse
import faulthandler
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# fp64 tensor-core (DMMA.8x8x4) peak measured on this pool's B200 by tools/probe
# (profiles/r01_fp64_probe.jsonl: 37.0 TF/s at 1965 MHz, flat from 4 to 32 warps/SM,
# held for a 125 ms sustained run; = 148 SM x 64 FMA/clk x 2 x 1.965 GHz within 0.5%).
# MEASURED_PEAKS.json carries no fp64 figure.
FP64_DMMA_PEAK_TFLOPS = 37.0
FP64_PEAK_SOURCE = ("measured DMMA.8x8x4 microbenchmark, profiles/r01_fp64_probe.jsonl (MEASURED_PEAKS.json has no "
                    "fp64 entry); nominal at the sampled SM clock in nominal_at_clock")
METRIC = "fp64 GEMM GFLOP/s (joules/GEMM vs N in energy/sweep)"
DATA = "synthetic (seeded splitmix64 uniform[-1,1), inputs/)"
WORKLOAD_N = 32768


def workload_config(N, G, exchange="pull"):
    """The config object both arms report (same workload, same keys)."""
    rows = []
    for g in range(G):
        q, r = divmod(N, G)
        rows.append(q + (1 if g < r else 0))
    ex = {"pull": "copy-engine pulls of B's k-panels from rank 0's symmetric window over NVLink (moa_pull_panels), "
                  "overlapped with the k-panel chain of each rank's GEMM",
          "nccl": "NCCL broadcast of B in pipelined k-panels (moa_lift_panels) on a CTA-limited communicator",
          "direct": "no copy of B: every rank's GEMM reads rank 0's window in place over NVLink (moa_gemm_lifted_direct)",
          "none": "none (one rank)"}[exchange if G > 1 else "none"]
    return {"workload": f"row-lifted fp64 GEMM m=n=p={N} on {G} B200 (BASELINE configs[4]), strong scaling: rank g "
                        f"owns rows moa_lift_rows({N}, {G}, g) of A and C; B ({N * N * 8 / 2 ** 30:.3g} GiB) travels "
                        "from rank 0 to every rank each step",
            "m": N, "n": N, "p": N, "rows_per_rank": rows, "parallelism": f"row-lifted x{G} (moa_gemm_lifted)",
            "exchange": ex, "gather": "none (reading R14: the gather of C is optional)",
            "l2": f"inputs larger than L2 ({(rows[0] * N * 2 + N * N) * 8 / 2 ** 30:.1f} GiB resident per GPU vs "
                  "126 MB L2), no flush"}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["moa", "reference"], default="moa")
    ap.add_argument("--N", type=int, default=WORKLOAD_N, help="m = n = p (default: BASELINE configs[4], 32768)")
    ap.add_argument("--exchange", choices=["pull", "nccl", "direct"], default="pull")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--sweep-sizes", default="1024,1536,2048,3072,4096,6144,8192,16000,16384")
    ap.add_argument("--sweep-windows", type=int, default=3)
    ap.add_argument("--watchdog-s", type=float, default=1800.0, help="exit with stack dumps after this long (0: off)")
    return ap.parse_args(argv)


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
            self.samples = []
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

    def idle_watts(self, seconds: float = 2.0):
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


def self_launch(args, argv) -> int:
    """bench.py --gpus G without torchrun: start G ranks (one process per GPU) under
    torch.distributed.run on 127.0.0.1 and pass rank 0's one JSON line through.
    Fails loudly when fewer than G GPUs are visible (MOA_BENCH_SHARE_GPU=1 lets the
    ranks share cuda:0 — for the one-GPU test of this code path with the test-only
    NCCL stand-in, never for a measurement)."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus and os.environ.get("MOA_BENCH_SHARE_GPU") != "1":
        sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}\n")
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "bench.py"), *argv]
    sys.stdout.flush()
    r = subprocess.run(cmd, cwd=ROOT, stdout=_JSON_FD if _JSON_FD is not None else None)
    return r.returncode


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
    m = n = p = N
    cores = os.cpu_count() or 1
    B = I.host_matrix(n, p, 1, I.ID_B)
    A1 = I.host_matrix(1, n, 1, I.ID_A)
    t0 = time.perf_counter()
    O.ip_rowblock(A1, B)
    t_row = time.perf_counter() - t0
    total_budget = 150.0  # seconds for warmup + steps
    want = int(total_budget * cores / max(t_row, 1e-6) / max(1, args.steps + args.warmup))
    rows_per_step, threads = _oracle_sample_rows(want, m, cores)
    A = I.host_matrix(rows_per_step, n, 1, I.ID_A)
    for _ in range(args.warmup):
        O.ip_rows(A, B, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.ip_rows(A, B, threads)
    dt = time.perf_counter() - t0
    value = 2.0 * rows_per_step * n * p * args.steps / dt / 1e9
    G = max(1, args.gpus)
    cfg = workload_config(N, G, args.exchange)
    cfg["reference_sample"] = (f"each step runs the CPU oracle (Fig. 4 ip_rows.c over {threads} threads, literal "
                               f"unfused ip.c update) on a bounded sample of {rows_per_step} of the {m} rows; "
                               f"GFLOP/s = 2*rows*n*p / time")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4),
        "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / max(1, args.steps) * 1e3, 3), "higher_is_better": True, "scaling": "strong",
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


def _fit_exponent(pts):
    xs = [math.log(x) for x, _ in pts]
    ys = [math.log(y) for _, y in pts]
    mx, my = sum(xs) / len(xs), sum(ys) / len(ys)
    return sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs)


def main(argv=None):
    faulthandler.enable()
    _quiet_stdout()
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    # Watchdog: a rank that stops making progress (a collective that never completes
    # on a box this build could not test on) dumps its stacks and exits instead of
    # holding the run; torchrun then stops the other ranks.
    if args.watchdog_s > 0:
        faulthandler.dump_traceback_later(args.watchdog_s, exit=True)
    if args.impl == "reference":
        return run_reference(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args, argv)

    import torch
    import torch.distributed as dist
    import paper_2306_11148_b200 as moa
    from inputs import inputs as I

    ws, rank, local = dist_env()
    if ws != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}\n")
        return 2
    shared = os.environ.get("MOA_BENCH_SHARE_GPU") == "1"
    device = 0 if shared else local
    if not shared and torch.cuda.device_count() <= device:
        sys.stderr.write(f"bench.py: rank {rank} needs cuda:{device}, {torch.cuda.device_count()} visible\n")
        return 2
    torch.cuda.set_device(device)
    dev = torch.device("cuda", device)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if ws == 1:
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
    # control plane (barriers, max over ranks, the 128-byte NCCL id) over gloo; the
    # data plane is libmoa's own communicator
    dist.init_process_group("gloo")
    stream = torch.cuda.current_stream()
    comm = moa.Comm(device=device)
    G = comm.world

    N = args.N
    m = n = p = N
    row0, rows = moa.lift_rows(m, G, rank)
    A = torch.empty((rows, n), dtype=torch.float64, device=dev)
    C = torch.empty((rows, p), dtype=torch.float64, device=dev)
    if rows:
        I.device_fill(A, 1, I.ID_A, row0=row0)

    def make_B(kind):
        Bt = comm.alloc_window((n, p)) if (kind in ("pull", "direct") and G > 1) else torch.empty((n, p), dtype=torch.float64,
                                                                                    device=dev)
        if rank == 0:
            I.device_fill(Bt, 1, I.ID_B)
        else:
            Bt.zero_()  # every other rank receives B through the exchange each step
        return Bt

    def free_B(Bt):
        if G > 1 and Bt is not None and args.exchange in ("pull", "direct") and Bt.data_ptr() in comm._windows:
            torch.cuda.synchronize()
            dist.barrier()
            comm.free_window(Bt)

    exchange = args.exchange if G > 1 else "none"
    fallback = None
    B = make_B(exchange)
    B_hold = {}

    def step(Bt, kind=None):
        if (kind or exchange) == "direct":
            moa.gemm_lifted_direct(m, A, Bt, C, comm)
        else:
            moa.gemm_lifted(m, A, Bt, C, comm)

    def timed(fn, k):
        """k calls of fn between a barrier + synchronize on both sides; device time (ms)
        on the launching stream, max over ranks."""
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        t0.record(stream)
        for i in range(k):
            evs[i][0].record(stream)
            fn()
            evs[i][1].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        el = t0.elapsed_time(t1)
        per = [a.elapsed_time(b) for a, b in evs]
        return max_over_ranks(el), per

    def max_over_ranks(x):
        t = torch.tensor([float(x)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        t = torch.tensor([float(x)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # warm-up (and the fallback if the pulled exchange is refused on this box)
    try:
        for _ in range(args.warmup):
            step(B)
        torch.cuda.synchronize()
    except moa.MoAError as e:
        if exchange != "pull":
            raise
        fallback = f"pulled exchange failed ({e}); NCCL exchange is the headline"
        sys.stderr.write("bench.py: " + fallback + "\n")
        exchange = "nccl"
        B = torch.empty((n, p), dtype=torch.float64, device=dev)
        if rank == 0:
            I.device_fill(B, 1, I.ID_B)
        for _ in range(args.warmup):
            step(B)
        torch.cuda.synchronize()

    sampler = ClockSampler(device)
    idle_w = sampler.idle_watts(2.0)
    idle_w_sum = sum_over_ranks(idle_w or 0.0) if idle_w is not None else None
    e0 = sampler.energy_mj()
    with sampler:
        elapsed_ms, per_step = timed(lambda: step(B), args.steps)
    e1 = sampler.energy_mj()
    clocks = sampler.summary()
    flops_step = 2.0 * m * n * p
    value = flops_step * args.steps / (elapsed_ms / 1e3) / 1e9  # GFLOP/s whole job

    # components on each rank (max over ranks): compute alone (moa_gemm on the rank's
    # rows, the dominant kernel), exchange alone (the same lifted call with no rows:
    # B's exchange plan and nothing else), exposed exchange = step - compute
    kreps = 3 if N >= 16384 else 5
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(kreps)]
    torch.cuda.synchronize()
    for a, b in kev:
        a.record(stream)
        if rows:
            moa.gemm(A, B, out=C)
        b.record(stream)
    torch.cuda.synchronize()
    gemm_ms_rank = statistics.mean(a.elapsed_time(b) for a, b in kev)
    gemm_ms = max_over_ranks(gemm_ms_rank)
    exch_ms = 0.0
    if G > 1:
        A0 = torch.empty((0, n), dtype=torch.float64, device=dev)
        C0 = torch.empty((0, p), dtype=torch.float64, device=dev)
        lifted0 = moa.gemm_lifted_direct if exchange == "direct" else moa.gemm_lifted
        exch_ms, _ = timed(lambda: lifted0(0, A0, B, C0, comm), 3)
        exch_ms /= 3
    step_ms = elapsed_ms / args.steps
    kflops = 2.0 * rows * n * p
    achieved_tf = kflops / (gemm_ms_rank / 1e3) / 1e12 if rows else 0.0
    achieved_tf = max_over_ranks(-achieved_tf) * -1 if G > 1 else achieved_tf  # the slowest rank's kernel
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_k1_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(f"{rows}x{n}x{p}")
        except Exception:
            traffic = None
    plan = moa.plan(rows, n, p)
    if exchange == "pull" and G > 1 and rank != 0:
        launches = len(moa.pull_panels(n)) - 1
    elif exchange == "nccl" and G > 1:
        launches = moa.lift_panels(n, p, moa.F64, G)
    else:
        launches = 1
    launches = int(max_over_ranks(launches))

    # energy (NVML; J per GEMM step summed over every participating GPU)
    energy = None
    ej = sum_over_ranks((e1 - e0) / 1e3 if (e0 is not None and e1 is not None) else -1e30)
    if ej > 0:  # (a window shorter than NVML's energy-counter update reads 0 J: no energy figure)
        idle_j = (idle_w_sum or 0.0) * (elapsed_ms / 1e3)
        energy = {"j_per_gemm": round(ej / args.steps, 3), "idle_w_all_gpus": idle_w_sum,
                  "j_per_gemm_above_idle": round((ej - idle_j) / args.steps, 3) if idle_w_sum is not None else None,
                  "window_s": round(elapsed_ms / 1e3, 3), "avg_w_all_gpus": round(ej / (elapsed_ms / 1e3), 1),
                  "gflops_per_w": round(value / (ej / (elapsed_ms / 1e3)), 2)}

    # the other exchange, measured beside the headline (G > 1)
    variants = None
    if G > 1 and not args.no_variants:
        variants = {exchange: {"ms_per_step": round(step_ms, 3), "gflops": round(value, 1)}}
        other = "nccl" if exchange == "pull" else "pull"
        try:
            B_hold["other"] = make_B(other)
            Bo = B_hold["other"]
            step(Bo, other)
            torch.cuda.synchronize()
            k2 = max(2, min(args.steps, 5))
            el2, _ = timed(lambda: step(Bo, other), k2)
            variants[other] = {"ms_per_step": round(el2 / k2, 3), "gflops": round(flops_step * k2 / (el2 / 1e3) / 1e9, 1)}
            if other == "pull":
                torch.cuda.synchronize()
                dist.barrier()
                comm.free_window(Bo)
            B_hold.clear()
        except Exception as e:  # report, keep the headline
            variants[other] = {"error": f"{type(e).__name__}: {e}"[:300]}

    # e2e through the public host-buffer API (copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        hA = torch.empty((rows, n), dtype=torch.float64).pin_memory()
        hC = torch.empty((rows, p), dtype=torch.float64).pin_memory()
        hA.copy_(A.cpu())
        hB = None
        if rank == 0:
            hB = torch.empty((n, p), dtype=torch.float64).pin_memory()
            hB.copy_(B.cpu())
        Bd = B  # (a window when the exchange is pulled: a valid NCCL buffer for the host path's broadcasts)

        def e2e_step():
            if G == 1:
                moa.gemm_host(hA, hB, hC, A, Bd, C)
            else:
                moa.gemm_lifted_host(m, hA, hB, hC, A, Bd, C, comm)
        e2e_step()
        torch.cuda.synchronize()
        k_e2e = max(1, min(args.steps, 3))
        e2e_ms, _ = timed(e2e_step, k_e2e)
        h2d = int(sum_over_ranks((rows * n + (n * p if rank == 0 else 0)) * 8))
        d2h = int(sum_over_ranks(rows * p * 8))
        e2e = {"value": round(flops_step * k_e2e / (e2e_ms / 1e3) / 1e9, 2), "unit": "GFLOP/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": k_e2e,
               "ms_per_step": round(e2e_ms / k_e2e, 3),
               "api": "moa_gemm_host" if G == 1 else "moa_gemm_lifted_host (B via NCCL panels)"}
        del hA, hB, hC

    free_B(B)
    del A, B, C

    # N sweep (GFLOP/s and J/GEMM vs N, the paper's study), G = 1 only
    sweep = None
    if G == 1 and not args.no_sweep:
        torch.cuda.empty_cache()
        idle_s = sampler.idle_watts(2.0)
        pts, points = [], []
        for Ns in [int(x) for x in args.sweep_sizes.split(",") if x]:
            As = torch.empty((Ns, Ns), dtype=torch.float64, device=dev)
            Bs = torch.empty((Ns, Ns), dtype=torch.float64, device=dev)
            Cs = torch.empty((Ns, Ns), dtype=torch.float64, device=dev)
            I.device_fill(As, 1, I.ID_A)
            I.device_fill(Bs, 1, I.ID_B)
            for _ in range(3):
                moa.gemm(As, Bs, out=Cs)
            torch.cuda.synchronize()
            est = 2.0 * Ns ** 3 / (FP64_DMMA_PEAK_TFLOPS * 1e12)  # a lower bound on the GEMM's time
            reps = max(3, math.ceil(1.1 / est))  # so each window is >= 1.1 s (NVML energy granularity)
            wins = []
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(args.sweep_windows):
                s0 = sampler.energy_mj()
                a.record(stream)
                for _ in range(reps):
                    moa.gemm(As, Bs, out=Cs)
                b.record(stream)
                torch.cuda.synchronize()
                s1 = sampler.energy_mj()
                ms = a.elapsed_time(b)
                wins.append((ms / reps, (s1 - s0) / 1e3 / reps if s0 is not None else None, ms / 1e3))
            ms = statistics.median(w[0] for w in wins)
            rec = {"N": Ns, "ms": round(ms, 4), "gflops": round(2.0 * Ns ** 3 / (ms / 1e3) / 1e9, 1),
                   "frac_of_peak": round(2.0 * Ns ** 3 / (ms / 1e3) / 1e12 / FP64_DMMA_PEAK_TFLOPS, 4),
                   "reps_per_window": reps, "windows": len(wins), "window_s": round(min(w[2] for w in wins), 3),
                   "l2": "warm (back-to-back launches)" if 3 * 8 * Ns * Ns < 126e6 else "inputs larger than L2"}
            if wins[0][1] is not None:
                js = sorted(w[1] for w in wins)
                rec["j_per_gemm"] = round(statistics.median(js), 5)
                rec["j_per_gemm_spread"] = [round(js[0], 5), round(js[-1], 5)]
                if idle_s is not None:
                    rec["j_per_gemm_above_idle"] = round(statistics.median(js) - idle_s * ms / 1e3, 5)
                pts.append((Ns, rec["j_per_gemm"], rec.get("j_per_gemm_above_idle")))
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
            points.append(rec)
            del As, Bs, Cs
            torch.cuda.empty_cache()
        sweep = {"points": points, "idle_w": idle_s, "windows_per_size": args.sweep_windows,
                 "paper_claim": "energy quadratic in N, i.e. linear in the size of matrix (P:14-15)"}
        if len(pts) >= 3:
            sweep["energy_exponent_fit"] = round(_fit_exponent([(x, y) for x, y, _ in pts]), 3)
            if all(z and z > 0 for _, _, z in pts):
                sweep["energy_exponent_fit_above_idle"] = round(_fit_exponent([(x, z) for x, _, z in pts]), 3)
            sweep["fit_range"] = [pts[0][0], pts[-1][0]]

    cpu = None
    if rank == 0 and G == 1 and not args.no_cpu:
        cpu = cpu_oracle_sample(m, n, p)

    comm.close()
    dist.destroy_process_group()
    if rank != 0:
        return 0
    cfg = workload_config(N, G, exchange)
    cfg["plan_rank0"] = {"kernel": plan.kernel, "bm": plan.bm, "bn": plan.bn, "bk": plan.bk, "stages": plan.stages,
                         "grid": plan.grid, "tiles": plan.tiles}
    if fallback:
        cfg["exchange_fallback"] = fallback
    sm = clocks.get("sm_mhz")
    line = {
        "metric": METRIC, "value": round(value, 2),
        "unit": "GFLOP/s", "n_gpus": G, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(step_ms, 4), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": cfg,
        "roofline": {"bound": "tensor", "achieved": round(achieved_tf, 3), "peak": FP64_DMMA_PEAK_TFLOPS,
                     "unit": "TFLOP/s", "frac": round(achieved_tf / FP64_DMMA_PEAK_TFLOPS, 4),
                     "traffic": traffic, "kernel": "k_dgemm_tma (fp64 DMMA) on one rank's rows",
                     "kernel_ms": round(gemm_ms, 3), "algorithmic_flops_per_launch": kflops,
                     "peak_source": FP64_PEAK_SOURCE,
                     "nominal_at_clock": round(148 * 64 * 2 * sm / 1e6, 2) if sm else None,
                     "frac_of_nominal_at_clock": round(achieved_tf / (148 * 64 * 2 * sm / 1e6), 4) if sm else None},
        "components": {"step_ms": round(step_ms, 3), "compute_ms": round(gemm_ms, 3),
                       "exchange_alone_ms": round(exch_ms, 3),
                       "exposed_exchange_ms": round(max(0.0, step_ms - gemm_ms), 3), "gather_ms": 0.0,
                       "step_ms_min_median_max": [round(min(per_step), 3), round(statistics.median(per_step), 3),
                                                  round(max(per_step), 3)]},
        "exchange_variants": variants,
        "e2e": e2e,
        "gpu_launches": launches * args.steps,
        "energy": energy,
        "sweep": sweep,
        "clocks": clocks,
        "cpu_baseline": cpu,
    }
    emit(line)
    return 0


if __name__ == "__main__":
    sys.exit(main())
