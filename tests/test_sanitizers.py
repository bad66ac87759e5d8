"""Host-code sanitizers: the CPU oracle and the C-ABI host layer of
libmoa.so (validation, psi / row lifting, the static plans, the exchange plan, the
error paths that return before any CUDA call) built with
-fsanitize=address,undefined -fno-sanitize-recover=all (tools/build.py asan) and
driven by the CPU tests that exercise them, in a subprocess with the ASan/UBSan
runtimes preloaded. Any heap/stack overflow, use-after-free, signed overflow,
misaligned access or other undefined behaviour aborts that run and fails this test.
(Device code is covered by compute-sanitizer on the GPU box: tools/gpu_sanitize.sh.)
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _runtime(name):
    p = subprocess.run(["gcc", f"-print-file-name={name}"], capture_output=True, text=True).stdout.strip()
    return p if os.path.isabs(p) and os.path.exists(p) else None


def test_host_code_under_asan_ubsan():
    if shutil.which("gcc") is None or shutil.which("g++") is None:
        pytest.skip("no gcc/g++")
    asan, ubsan = _runtime("libasan.so"), _runtime("libubsan.so")
    if not asan or not ubsan:
        pytest.skip("sanitizer runtimes not installed")
    subprocess.check_call([sys.executable, os.path.join(ROOT, "tools", "build.py"), "asan"], cwd=ROOT,
                          stdout=subprocess.DEVNULL)
    env = dict(os.environ)
    env.update({"LD_PRELOAD": f"{asan}:{ubsan}", "ASAN_OPTIONS": "detect_leaks=0:verify_asan_link_order=0",
                "UBSAN_OPTIONS": "print_stacktrace=1:halt_on_error=1",
                "MOA_LIBRARY": os.path.join(ROOT, "build", "asan", "libmoa_asan.so"),
                "MOA_ORACLE_LIBRARY": os.path.join(ROOT, "oracle", "liboracle_asan.so")})
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "not gpu", "-p", "no:cacheprovider",
                        "tests/test_oracle.py", "tests/test_oracle_ipophp.py", "tests/test_abi.py",
                        "tests/test_exchange_plan.py", "tests/test_fused_gather.py", "tests/test_lifted.py",
                        "tests/test_inputs.py"],
                       capture_output=True, text=True, cwd=ROOT, env=env, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "runtime error" not in out and "AddressSanitizer" not in out, out[-4000:]
    assert "passed" in r.stdout
    # the instrumented libraries were the ones loaded
    code = ("import paper_2306_11148_b200, oracle.oracle as O; O._load(); "
            "print(open('/proc/self/maps').read())")
    m = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, env=env, timeout=300)
    assert "libmoa_asan.so" in m.stdout and "liboracle_asan.so" in m.stdout, m.stderr[-2000:]
