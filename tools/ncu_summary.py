#!/usr/bin/env python3
"""Summarise ncu artefacts into profiles/ (tracked evidence).

  ncu_summary.py launches <launches.csv>              -> per-kernel share of the step
  ncu_summary.py full <report.ncu-rep> [--flops F] [--bytes B]
                                                      -> key metrics of one --set full capture
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tc.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "lts__t_bytes.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "gpc__cycles_elapsed.avg.per_second",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            d[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    out = []
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        out.append({"kernel": k, "launches": len(v), "total_ms": round(sum(v) / 1e6, 4),
                    "mean_ms": round(sum(v) / len(v) / 1e6, 4), "share": round(sum(v) / tot, 4)})
    return {"source": path, "note": "ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised)",
            "kernels": out}


def full(path, flops=None, nbytes=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        rec = {"kernel": r[h.index("Kernel Name")].split("(")[0] if "Kernel Name" in h else "?"}
        for i, name in enumerate(h):
            if name in KEYS:
                try:
                    rec[name] = {"value": float(r[i].replace(",", "")), "unit": units[i]}
                except ValueError:
                    rec[name] = {"value": r[i], "unit": units[i]}
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        try:
            rd = rec["dram__bytes_read.sum"]
            wr = rec["dram__bytes_write.sum"]
            rec["traffic_bytes"] = rd["value"] * scale.get(rd["unit"], 1) + wr["value"] * scale.get(wr["unit"], 1)
        except KeyError:
            pass
        t = rec.get("gpu__time_duration.sum")
        if t and flops:
            sec = t["value"] * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
                                "second": 1.0}.get(t["unit"], 1e-9)
            rec["achieved_tflops_under_ncu"] = round(flops / sec / 1e12, 3)
        if nbytes and "traffic_bytes" in rec:
            rec["traffic_over_algorithmic"] = round(rec["traffic_bytes"] / nbytes, 3)
        res.append(rec)
    return {"source": path, "captures": res}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["launches", "full"])
    ap.add_argument("path")
    ap.add_argument("--flops", type=float)
    ap.add_argument("--bytes", type=float)
    a = ap.parse_args()
    out = launches(a.path) if a.mode == "launches" else full(a.path, a.flops, a.bytes)
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
