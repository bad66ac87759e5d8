"""Mutation test of the parity harness (idea from SPEC S:495: an off-by-one
offset must make verification fail).

Each mutant is a copy of oracle/moa_oracle.c with ONE plausible slip in Fig. 3 ip.c
 — the definition every GPU parity test compares against — compiled to its
own library and loaded in a subprocess through MOA_ORACLE_LIBRARY:
  * the last sigma term dropped (off by one in the sigma bound);
  * a column index off by one in B's read (B[(sigma*sizer) + j] -> row-reversed j);
  * the sigma order reversed (same terms, other rounding sequence);
  * the literal update contracted to an fma (reading R3 mixed up);
  * C not zeroed before the accumulation (reading R1 dropped).
CPU: the oracle's pins (tests/test_oracle.py) must FAIL for every mutant — a pin set
that let one through would not be pinning the oracle. GPU: the GPU parity test must
fail against the off-by-one mutant (the harness does compare).
"""
from __future__ import annotations

import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "moa_oracle.c")

# (name, pattern inside DEF_IP's body, replacement); applied to the first match only
MUTANTS = [
    ("drop_last_sigma", r"for \(sigma = 0; sigma < shr0; sigma\+\+\)", "for (sigma = 0; sigma < shr0 - 1; sigma++)"),
    ("b_column_off", r"B\[\(sigma \* sizer\) \+ j\]\);", "B[(sigma * sizer) + (sizer - 1 - j)]);"),
    ("sigma_reversed", r"A\[\(i \* shr0\) \+ sigma\], B\[\(sigma \* sizer\) \+ j\]\);",
     "A[(i * shr0) + (shr0 - 1 - sigma)], B[((shr0 - 1 - sigma) * sizer) + j]);"),
    ("unfused_is_fma", r"#define UPD_UNFUSED\(c, a, b\) \(c\) = \(c\) \+ \(a\) \* \(b\)",
     "#define UPD_UNFUSED(c, a, b) (c) = fma((a), (b), (c))"),
    ("c_not_zeroed", r"for \(i = 0; i < sizel \* sizer; i\+\+\) C\[i\] = \(T\)0;", "C[0] = C[0];"),
]


def _build(tmp_path, name, pat, rep):
    src = open(SRC).read()
    # mutate inside the DEF_IP macro (Fig. 3 ip.c) only
    start = src.index("#define DEF_IP(NAME")
    end = src.index("DEF_IP(oracle_ip_unfused_f64")
    body, n = re.subn(pat, rep.replace("\\", "\\\\"), src[start:end], count=1)
    assert n == 1, f"mutation {name} did not apply"
    mut = tmp_path / f"oracle_{name}.c"
    mut.write_text(src[:start] + body + src[end:])
    so = tmp_path / f"liboracle_{name}.so"
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC", "-shared",
                           "-pthread", str(mut), "-o", str(so), "-lm"])
    return str(so)


def _pytest(so, target, extra=()):
    env = dict(os.environ, MOA_ORACLE_LIBRARY=so)
    return subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", *extra, target],
                          capture_output=True, text=True, cwd=ROOT, env=env, timeout=600)


@pytest.mark.parametrize("name,pat,rep", MUTANTS, ids=[m[0] for m in MUTANTS])
def test_oracle_pins_kill_every_mutant(tmp_path, name, pat, rep):
    so = _build(tmp_path, name, pat, rep)
    r = _pytest(so, "tests/test_oracle.py", ("-m", "not gpu"))
    assert r.returncode != 0, f"mutant {name} survived the oracle pins:\n{r.stdout[-2000:]}"
    assert "failed" in r.stdout


def test_unmutated_copy_passes(tmp_path):
    """Control: the same build path with no mutation passes the pins."""
    src = open(SRC).read()
    c = tmp_path / "oracle_same.c"
    c.write_text(src)
    so = tmp_path / "liboracle_same.so"
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC", "-shared",
                           "-pthread", str(c), "-o", str(so), "-lm"])
    r = _pytest(str(so), "tests/test_oracle.py", ("-m", "not gpu"))
    assert r.returncode == 0, r.stdout[-2000:]


@pytest.mark.gpu
def test_gpu_parity_harness_catches_off_by_one(tmp_path, cuda_device):
    so = _build(tmp_path, "drop_last_sigma", *MUTANTS[0][1:])
    r = _pytest(so, "tests/test_gemm_gpu.py::test_each_compiled_tile_config_bitwise", ("-m", "gpu"))
    assert r.returncode != 0 and "failed" in r.stdout, r.stdout[-2000:]
