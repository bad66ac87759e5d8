"""Every `nranks > 1` branch of the lifted paths, executed with G = 2, 3, 4 processes.

The row lift (Fig. 4 ip_rows.c P:150-171), the column lift (Fig. 5
ip_cols.c) and the 2-D lift all have an exchange step (B, A
or both travel; C is optionally gathered). Round 1 could only run them on 1-rank
communicators, where the exchange is skipped. Here each rank is its own process
(tests/mp_lifted_worker.py) and drives the product's entry points through the
binding with real multi-rank semantics; every output a rank holds (its rows / block
of C, the gathered C_full, the broadcast B / A) must equal the CPU oracle bit for
bit, with NaN in every buffer a rank does not own beforehand.

With fewer GPUs than ranks (the one-GPU box), the ranks share cuda:0 through the
test-only NCCL stand-in tests/nccl_shim (LD_PRELOAD; real NCCL refuses two ranks on
one device). The stand-in logs every collective, and the executed sequence on every
rank must equal the library's own exchange plan (moa_exchange_plan) op for op — the
check that caught round 1's duplicate broadcast of A in moa_gemm_lifted_cols. With
>= G GPUs the same cases run over real NCCL (one GPU per rank) without the log check.
"""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "tests", "nccl_shim", "libmoa_nccl_shim.so")
WORKER = os.path.join(ROOT, "tests", "mp_lifted_worker.py")

CASES = {
    2: [
        dict(name="rows_k1_allgather", kind="rows", m=300, n=96, p=200, npanels=1, gather=True),
        dict(name="rows_k3_uneven_gather", kind="rows", m=301, n=160, p=136, npanels=3, gather=True),
        dict(name="rows_static_f32", kind="rows", m=256, n=128, p=192, npanels=2, dtype="f32"),
        dict(name="rows_pull", kind="rows_pull", m=300, n=256, p=200, gather=True),
        dict(name="rows_pull_f32", kind="rows_pull", m=130, n=512, p=96, dtype="f32"),
        dict(name="rows_direct", kind="rows_direct", m=300, n=256, p=200, gather=True),
        dict(name="rows_direct_f32", kind="rows_direct", m=130, n=96, p=96, dtype="f32"),
        dict(name="rows_fused", kind="rows_fused", m=301, n=96, p=200, npanels=2),
        dict(name="rows_pull_fused", kind="rows_pull_fused", m=300, n=128, p=200),
        dict(name="rows_host", kind="rows_host", m=600, n=512, p=256),
        dict(name="cols_gather", kind="cols", m=200, n=96, p=301, gather=True),
        dict(name="cols_nogather", kind="cols", m=200, n=96, p=300),
        dict(name="cols_fused", kind="cols_fused", m=200, n=96, p=300),
        dict(name="cols_fused_f32", kind="cols_fused", m=100, n=64, p=256, dtype="f32"),
        dict(name="grid_1x2", kind="2d", m=130, n=64, p=200, grid=[1, 2]),
        dict(name="grid_2x1", kind="2d", m=130, n=64, p=200, grid=[2, 1]),
        dict(name="grid_1x2_fused", kind="2d_fused", m=130, n=64, p=200, grid=[1, 2]),
        # the 3xTF32 tcgen05 kernel's fused-gather epilogue (tolerance, not bits: reading R20's variant)
        dict(name="rows_fused_3xtf32", kind="rows_fused", m=300, n=96, p=200, npanels=2, dtype="3xtf32"),
    ],
    3: [
        dict(name="rows_zero_row_rank", kind="rows", m=2, n=64, p=96, gather=True),
        dict(name="rows_uneven_k2", kind="rows", m=301, n=128, p=72, npanels=2, gather=True),
        dict(name="rows_pull_uneven", kind="rows_pull", m=100, n=512, p=64, gather=True),
        dict(name="rows_direct_uneven", kind="rows_direct", m=100, n=512, p=64),
        dict(name="rows_fused_uneven", kind="rows_fused", m=200, n=64, p=128),
        dict(name="rows_fused_3xtf32_uneven", kind="rows_fused", m=301, n=128, p=128, dtype="3xtf32"),
        dict(name="cols_uneven", kind="cols", m=64, n=48, p=100, gather=True),
        dict(name="rows_host_uneven", kind="rows_host", m=301, n=512, p=96),
    ],
    4: [
        dict(name="grid_2x2", kind="2d", m=257, n=96, p=131, grid=[2, 2]),
        dict(name="grid_2x2_fused", kind="2d_fused", m=257, n=96, p=132, grid=[2, 2]),
        dict(name="grid_1x4_f32", kind="2d", m=64, n=32, p=200, grid=[1, 4], dtype="f32"),
        dict(name="rows_allgather_g4", kind="rows", m=500, n=128, p=256, gather=True),
        dict(name="rows_pull_fused_g4", kind="rows_pull_fused", m=501, n=256, p=136),
    ],
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _plan_for(moa, case, G, rank):
    dt = {"f32": moa.F32, "3xtf32": moa.F32_3XTF32}.get(case.get("dtype"), moa.F64)
    m, n, p, kind = case["m"], case["n"], case["p"], case["kind"]
    gr, gc = case.get("grid", [0, 0])
    v, flags = {
        "rows": (moa.XPLAN_ROWS, moa.XF_GATHER if case.get("gather") else 0),
        "rows_pull": (moa.XPLAN_ROWS, moa.XF_PULL_B | (moa.XF_GATHER if case.get("gather") else 0)),
        "rows_fused": (moa.XPLAN_ROWS, moa.XF_FUSED_GATHER),
        "rows_pull_fused": (moa.XPLAN_ROWS, moa.XF_FUSED_GATHER | moa.XF_PULL_B),
        "rows_direct": (moa.XPLAN_ROWS, moa.XF_DIRECT_B | (moa.XF_GATHER if case.get("gather") else 0)),
        "rows_host": (moa.XPLAN_ROWS_HOST, 0),
        "cols": (moa.XPLAN_COLS, moa.XF_GATHER if case.get("gather") else 0),
        "cols_fused": (moa.XPLAN_COLS, moa.XF_FUSED_GATHER),
        "2d": (moa.XPLAN_2D, 0),
        "2d_fused": (moa.XPLAN_2D, moa.XF_FUSED_GATHER),
    }[kind]
    return moa.exchange_plan(v, m, n, p, dt, G, rank, gr, gc, case.get("npanels", 0), flags), (gr, gc)


def _comm_matches(kind, entry, G, grid):
    if kind == "world":
        return entry["comm"] == "world"
    if kind == "pipe":
        return entry["comm"] != "world" and entry["max_ctas"] == 4 and entry["nranks"] == G
    if kind == "row":
        return entry["comm"] != "world" and entry["nranks"] == grid[1]
    return entry["comm"] != "world" and entry["nranks"] == grid[0]   # col


def _run(G, tmp_path, shared_gpu, cases):
    import torch
    out = tmp_path / f"g{G}"
    out.mkdir()
    cases_file = out / "cases.json"
    cases_file.write_text(json.dumps(cases))
    env = dict(os.environ)
    env["MOA_NCCL_SHIM_TIMEOUT"] = "90"
    if shared_gpu:
        if not os.path.exists(SHIM):
            subprocess.check_call([sys.executable, os.path.join(ROOT, "tools", "build.py"), "shim"])
        env["LD_PRELOAD"] = SHIM + ((":" + env["LD_PRELOAD"]) if env.get("LD_PRELOAD") else "")
    port = _free_port()
    procs = [subprocess.Popen([sys.executable, WORKER, str(r), str(G), str(port), str(out), str(cases_file),
                               "0" if shared_gpu else str(r)], env=env, cwd=ROOT)
             for r in range(G)]
    try:
        for pr in procs:
            pr.wait(timeout=900)
    finally:
        for pr in procs:
            if pr.poll() is None:
                pr.kill()
    assert [pr.returncode for pr in procs] == [0] * G
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 3, 4])
def test_lifted_paths_multiprocess(G, tmp_path, cuda_device):
    import torch
    import paper_2306_11148_b200 as moa
    shared = torch.cuda.device_count() < G
    out = _run(G, tmp_path, shared, CASES[G])
    res = [json.loads((out / f"rank{r}.json").read_text()) for r in range(G)]
    bad = {(c["name"], r): res[r][c["name"]] for c in CASES[G] for r in range(G) if not res[r][c["name"]]["ok"]}
    assert not bad, json.dumps(bad, indent=1)[:4000]
    # tolerance-checked cases: every rank's gathered copy holds the same bits
    for c in CASES[G]:
        if c.get("dtype") == "3xtf32":
            digests = {res[r][c["name"]]["digest"] for r in range(G)}
            assert len(digests) == 1 and None not in digests, (c["name"], digests)
    if not shared:
        return
    # the collective sequence each rank executed == the library's exchange plan
    for case in CASES[G]:
        logs = []
        for r in range(G):
            f = out / f"{case['name']}.rank{r}.jsonl"
            entries = [json.loads(line) for line in f.read_text().splitlines()] if f.exists() else []
            plan, grid = _plan_for(moa, case, G, r)
            want = [o for o in plan if o.op != "pull"]
            got = [(e["op"], e["root"], e["count"], e["esize"]) for e in entries]
            exp = [(o.op if o.op != "barrier" else "allreduce", o.root, o.count if o.op != "barrier" else 1,
                    (4 if case.get("dtype") in ("f32", "3xtf32") else 8) if o.op != "barrier" else 4) for o in want]
            assert got == exp, (case["name"], r, got, exp)
            assert all(_comm_matches(o.comm, e, G, grid) for o, e in zip(want, entries)), (case["name"], r, entries)
            logs.append(entries)
        # identical across ranks on the world communicator (per sub-communicator for 2-D)
        worlds = [[(e["op"], e["root"], e["count"]) for e in L if e["comm"] == "world"] for L in logs]
        assert all(w == worlds[0] for w in worlds), (case["name"], worlds)


@pytest.mark.gpu
def test_cols_broadcasts_A_once_per_call(tmp_path, cuda_device):
    """Regression (round-1 review): moa_gemm_lifted_cols with C_full in a window
    broadcast A twice (8 GiB extra at m = n = 32768). One broadcast of A per call."""
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("the collective log needs the one-GPU stand-in")
    out = _run(2, tmp_path, True, [c for c in CASES[2] if c["name"] in ("cols_fused", "cols_gather")])
    for name in ("cols_fused", "cols_gather"):
        for r in range(2):
            entries = [json.loads(x) for x in (out / f"{name}.rank{r}.jsonl").read_text().splitlines()]
            a_bcasts = [e for e in entries if e["op"] == "broadcast" and e["root"] == 0 and e["count"] == 200 * 96]
            assert len(a_bcasts) == 1, (name, r, entries)
