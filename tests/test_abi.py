"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/moa.h declares, and its host-only entry points (psi, row lifting,
paper block arithmetic, argument validation) behave as documented."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2306_11148_b200 as moa
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "moa.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|void)\s+(moa_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(moa.lib_path)
    syms = _declared_symbols()
    assert len(syms) >= 14, syms
    for s in syms:
        assert hasattr(lib, s), s
    assert moa.abi_version() == 1


def test_psi_matches_oracle():
    rng = np.random.default_rng(0)
    for _ in range(300):
        rank = int(rng.integers(0, 5))
        shape = [int(x) for x in rng.integers(1, 6, size=rank)]
        q = int(rng.integers(0, rank + 1))
        idx = [int(rng.integers(0, s)) for s in shape[:q]]
        assert moa.psi(idx, shape) == O.psi(idx, shape)
    assert moa.psi([1], [2, 2]) == (2, 2)
    assert moa.psi([1, 0], [2, 2]) == (2, 1)
    assert moa.psi([1, 2], [3, 4]) == (6, 1)
    assert moa.psi([], []) == (0, 1)            # scalar
    for bad_idx, shape in [([2], [2, 2]), ([0, 0, 0], [2, 2]), ([-1], [3])]:
        with pytest.raises(moa.MoAError) as e:
            moa.psi(bad_idx, shape)
        assert e.value.name == "MOA_ERR_INVALID_INDEX"


def test_psi_onf_rows_are_contiguous():
    """In the ONF, psi(<i>, A) = [i*n, i*n+n) and psi(<sigma>, B) = [sigma*p, sigma*p+p) (Fig. 1)."""
    m, n, p = 7, 5, 3
    for i in range(m):
        assert moa.psi([i], [m, n]) == (i * n, n)
    for s in range(n):
        assert moa.psi([s], [n, p]) == (s * p, p)


def test_lift_rows_matches_oracle():
    for m in range(0, 50):
        for G in range(1, 9):
            for g in range(G):
                assert moa.lift_rows(m, G, g) == O.lift_rows(m, G, g)
    for args in [(10, 0, 0), (10, 2, 2), (-1, 2, 0), (10, 2, -1)]:
        with pytest.raises(moa.MoAError):
            moa.lift_rows(*args)


def test_select_block_paper_matches_oracle_and_paper():
    assert moa.select_block_paper(32 * 1024, 8) == 32
    assert moa.select_block_paper(128 * 1024, 8) == 64
    for budget in [24, 100, 4096, 50000, 1 << 20]:
        for e in (4, 8):
            if budget >= 3 * e:
                assert moa.select_block_paper(budget, e) == O.select_block_paper(budget, e)
    with pytest.raises(moa.MoAError):
        moa.select_block_paper(10, 8)


def _raw_gemm(m, n, p, A, B, C, dtype=0):
    return moa._moa_gemm(m, n, p, A, B, C, dtype, None)


def test_validation_before_any_cuda_call():
    """These return before touching CUDA, so they work without a GPU."""
    st = {v: k for k, v in {0: "OK", 1: "SHAPE", 2: "DTYPE", 3: "NULL", 4: "ALIAS", 5: "MISALIGNED"}.items()}
    A, B, C = 0x10000, 0x20000, 0x30000
    assert _raw_gemm(-1, 2, 2, A, B, C) == st["SHAPE"]
    assert _raw_gemm(2, 2, 2, A, B, C, dtype=7) == st["DTYPE"]
    assert _raw_gemm(2, 2, 2, None, B, C) == st["NULL"]
    assert _raw_gemm(2, 2, 2, A, B, None) == st["NULL"]
    assert _raw_gemm(2, 2, 2, A + 4, B, C) == st["MISALIGNED"]
    assert _raw_gemm(2, 2, 2, A, B, A + 8) == st["ALIAS"]
    assert _raw_gemm(2, 2, 2, A, B, B) == st["ALIAS"]
    assert _raw_gemm(1 << 40, 1 << 40, 2, A, B, C) == st["SHAPE"]
    # empty operands may be NULL
    assert _raw_gemm(0, 5, 5, None, B, None) in (0, 7, 9)  # OK, or CUDA/device error when no GPU
    assert moa._moa_status_string(4) == b"MOA_ERR_ALIASING"


def test_gemm_host_and_lifted_validate_first():
    assert moa._moa_gemm_host(-1, 1, 1, None, None, None, None, None, None, 0, None) == 1
    assert moa._moa_gemm_lifted(4, 4, 4, None, None, None, None, 0, None, None) == 3  # NULL comm


def test_lift_panels_static_choice():
    assert moa.lift_panels(1000, 1000, 0, 1) == 1                 # B does not travel
    assert moa.lift_panels(32768, 32768, 0, 8) == 8               # 8 GiB of B -> 8 panels
    assert moa.lift_panels(8192, 8192, 0, 8) == 1                 # 512 MiB -> 1
    assert moa.lift_panels(16384, 16384, 0, 2) == 4               # 2 GiB -> 4
    assert moa.lift_panels(100, 1 << 22, 0, 4) == 1               # n/64 clamp


def test_gemm_acc_validation_without_gpu():
    A, B, C = 0x10000, 0x200000, 0x4000000
    assert moa._moa_gemm_acc(4, 8, 8, A, 7, B, 8, C, 8, 0, 0, None) == 1      # lda < n
    assert moa._moa_gemm_acc(4, 8, 8, A, 8, B, 8, C, 7, 0, 0, None) == 1      # ldc < p
    assert moa._moa_gemm_acc(4, 8, 8, A, 8, B, 8, A + 8 * 20, 8, 0, 0, None) == 4  # C inside A's span


def test_header_is_plain_c_and_links_from_c(tmp_path):
    """include/moa.h compiles as C99 (no C++ or torch types), and a plain C program
    links libmoa.so and calls host-only entry points through it."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    src = tmp_path / "abi_user.c"
    src.write_text(r"""
#include <stdio.h>
#include <string.h>
#include "moa.h"
int main(void) {
  int64_t row0 = -1, rows = -1, off = -1, cnt = -1, b = -1;
  const int64_t shape[2] = {3, 4}, idx[2] = {1, 2};
  if (moa_abi_version() != MOA_ABI_VERSION) return 1;
  if (moa_lift_rows(37, 2, 1, &row0, &rows) != MOA_OK || row0 != 19 || rows != 18) return 2;
  if (moa_psi(2, shape, 2, idx, &off, &cnt) != MOA_OK || off != 6 || cnt != 1) return 3;
  if (moa_select_block_paper(32 * 1024, 8, &b) != MOA_OK || b != 32) return 4;
  if (strcmp(moa_status_string(MOA_ERR_ALIASING), "MOA_ERR_ALIASING") != 0) return 5;
  if (moa_gemm(-1, 2, 2, 0, 0, 0, MOA_F64, 0) != MOA_ERR_INVALID_SHAPE) return 6;
  printf("C ABI OK\n");
  return 0;
}
""")
    libdir = os.path.dirname(moa.lib_path)
    exe = tmp_path / "abi_user"
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), str(src),
                        "-o", str(exe), "-L", libdir, "-l:" + os.path.basename(moa.lib_path), "-Wl,-rpath," + libdir],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "C ABI OK" in r.stdout, (r.returncode, r.stdout, r.stderr)
