"""bench.py's driver contract, checked without a GPU on the reference arm (the CPU
oracle): stdout carries exactly ONE JSON line with the contract's keys, even when a
native library writes to fd 1 (bench.py routes fd 1 to stderr and writes the line
to the saved stdout), and the line's config names the same workload as the GPU arm."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=300, cwd=ROOT, env=e)


def test_reference_arm_prints_one_json_line():
    r = _run(["--impl", "reference", "--N", "64", "--steps", "2", "--warmup", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["unit"] == "GFLOP/s" and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["warmup"] == 1 and d["value"] > 0
    assert d["config"]["n"] == 64 and "BASELINE configs[4]" in d["config"]["workload"]
    assert d["scaling"] == "strong" and d["config"]["rows_per_rank"] == [64]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"


def test_stray_fd1_writes_do_not_reach_stdout():
    """A native write to fd 1 during the run (as NCCL's version banner is on the GPU
    boxes) lands on stderr; stdout still parses as the one JSON line."""
    code = ("import os, runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--N', '32', '--steps', '1', "
            "'--warmup', '0']; import bench; bench._quiet_stdout(); os.write(1, b'NCCL version banner\\n'); "
            "sys.exit(bench.main())")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1 and json.loads(lines[0])["impl"] == "reference", r.stdout
    assert "NCCL version banner" in r.stderr


def test_reference_arm_other_ranks_exit_quietly():
    r = _run(["--impl", "reference", "--N", "32", "--steps", "1", "--warmup", "0"],
             env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0 and r.stdout.strip() == "", r.stdout


def test_gpus_without_enough_devices_fails_loudly():
    """bench.py --gpus 2 (no torchrun) launches its 2 ranks itself — or, with fewer
    visible GPUs (here: none), exits non-zero with a clear message instead of silently
    measuring one GPU (round-1 review)."""
    r = _run(["--gpus", "2", "--steps", "1", "--warmup", "0"])
    assert r.returncode != 0
    assert "needs 2 visible GPUs" in r.stderr, r.stderr[-2000:]
    assert r.stdout.strip() == ""


def test_world_size_must_match_gpus():
    r = _run(["--gpus", "4", "--steps", "1", "--warmup", "0"], env={"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert r.returncode != 0 and "WORLD_SIZE=2" in r.stderr, r.stderr[-2000:]


def test_reference_arm_config_matches_gpu_arm_for_each_G():
    import bench
    for G in (1, 2, 4, 8):
        cfg = bench.workload_config(32768, G)
        assert cfg["m"] == cfg["n"] == cfg["p"] == 32768
        assert sum(cfg["rows_per_rank"]) == 32768 and len(cfg["rows_per_rank"]) == G
