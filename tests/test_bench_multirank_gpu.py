"""bench.py's multi-rank path (the driver's SCALE run: G = 2/4/8 ranks of BASELINE
configs[4]) executed on the one-GPU box: `bench.py --gpus G` self-launches its G ranks
under torch.distributed.run, the ranks share cuda:0 (MOA_BENCH_SHARE_GPU=1, test only)
and libmoa's collectives go through the test-only NCCL stand-in (tests/nccl_shim).
The numbers are meaningless here (G processes time-slice one GPU); what is checked is
the control flow the 8-GPU run depends on: one JSON line from rank 0, n_gpus = the
communicator's size, the row partition, both exchanges (pulled headline, NCCL
variant), the component breakdown, the e2e leg through moa_gemm_lifted_host, and a
clean exit of every rank."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "tests", "nccl_shim", "libmoa_nccl_shim.so")


@pytest.mark.gpu
@pytest.mark.parametrize("G,N", [(2, 2048), (3, 1536)])
def test_bench_self_launches_G_ranks(G, N, cuda_device):
    if not os.path.exists(SHIM):
        subprocess.check_call([sys.executable, os.path.join(ROOT, "tools", "build.py"), "shim"])
    env = dict(os.environ)
    env.update({"LD_PRELOAD": SHIM, "MOA_BENCH_SHARE_GPU": "1", "MOA_NCCL_SHIM_TIMEOUT": "120"})
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(G), "--N", str(N), "--steps",
                        "3", "--warmup", "1", "--no-cpu"], capture_output=True, text=True, timeout=900, cwd=ROOT,
                       env=env)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == G and d["scaling"] == "strong" and d["steps"] == 3
    cfg = d["config"]
    assert cfg["m"] == N and sum(cfg["rows_per_rank"]) == N and len(cfg["rows_per_rank"]) == G
    assert "BASELINE configs[4]" in cfg["workload"] and "copy-engine" in cfg["exchange"]
    assert "exchange_fallback" not in cfg, cfg
    assert d["value"] > 0 and d["components"]["compute_ms"] > 0 and d["components"]["exchange_alone_ms"] > 0
    assert set(d["exchange_variants"]) == {"pull", "nccl"}, d["exchange_variants"]
    assert all("gflops" in v for v in d["exchange_variants"].values()), d["exchange_variants"]
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == (N * N + N * N) * 8
    assert d["e2e"]["d2h_bytes_per_step"] == N * N * 8
    assert d["gpu_launches"] == 3 * (len(__import__("paper_2306_11148_b200").pull_panels(N)) - 1)
    assert d["sweep"] is None and d["cpu_baseline"] is None


@pytest.mark.gpu
def test_bench_direct_exchange(cuda_device):
    """bench.py --exchange direct (NEXT-1 step 2: every rank's GEMM reads rank 0's B in
    place): the line names the exchange and carries the pulled one beside it."""
    if not os.path.exists(SHIM):
        subprocess.check_call([sys.executable, os.path.join(ROOT, "tools", "build.py"), "shim"])
    env = dict(os.environ)
    env.update({"LD_PRELOAD": SHIM, "MOA_BENCH_SHARE_GPU": "1", "MOA_NCCL_SHIM_TIMEOUT": "120"})
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--N", "1024", "--steps", "3",
                        "--warmup", "1", "--no-cpu", "--no-e2e", "--exchange", "direct"], capture_output=True, text=True,
                       timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-4000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.strip()][-1])
    assert "no copy of B" in d["config"]["exchange"] and d["gpu_launches"] == 3
    assert set(d["exchange_variants"]) == {"direct", "pull"}, d["exchange_variants"]
    assert d["value"] > 0
