"""CPU oracle for the MoA-ONF GEMM — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
and ``--impl reference`` legs may import this module. The product package
``paper_2306_11148_b200`` never imports it and shares no code with it.

ctypes binding to ``oracle/liboracle.so`` (built from ``oracle/moa_oracle.c``
with ``gcc -O2 -ffp-contract=off -fno-fast-math``, see ``tools/build.py``),
plus plain-Python shape helpers (ψ / γ_row, row lifting, the paper's block
arithmetic). Every function cites the PAPER.md passage it follows
(``P:n`` = line n of /root/reference/PAPER.md). Readings R1..R16 are listed in
DESIGN.md §Readings.

Parity status (DESIGN.md §Oracle pins): every function here is pinned by
``tests/test_oracle.py``; none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import math
import os
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MOA_ORACLE_LIBRARY: an instrumented build of the same source (tests/test_sanitizers.py
# loads oracle/liboracle_asan.so, -fsanitize=address,undefined); default: liboracle.so
_LIB_PATH = os.environ.get("MOA_ORACLE_LIBRARY") or os.path.join(_HERE, "liboracle.so")
_lib = None

_i64 = ctypes.c_int64
_vp = ctypes.c_void_p


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            import subprocess
            import sys
            subprocess.check_call([sys.executable, os.path.join(_HERE, "..", "tools", "build.py"), "oracle"])
        lib = ctypes.CDLL(_LIB_PATH)
        for t in ("f64", "f32"):
            for v in ("unfused", "fma"):
                getattr(lib, f"oracle_ip_{v}_{t}").argtypes = [_vp, _vp, _vp, _i64, _i64, _i64]
                getattr(lib, f"oracle_ip_{v}_{t}").restype = None
                getattr(lib, f"oracle_ip_rowset_{v}_{t}").argtypes = [_vp, _vp, _vp, _i64, _i64, _i64, _vp, _i64]
                getattr(lib, f"oracle_ip_rowset_{v}_{t}").restype = ctypes.c_int
                getattr(lib, f"oracle_ip_rowblock_{v}_{t}").argtypes = [_vp, _vp, _vp, _i64, _i64, _i64]
                getattr(lib, f"oracle_ip_rowblock_{v}_{t}").restype = None
            getattr(lib, f"oracle_ip_ijk_unfused_{t}").argtypes = [_vp, _vp, _vp, _i64, _i64, _i64]
            getattr(lib, f"oracle_ip_ijk_unfused_{t}").restype = None
        lib.oracle_ip_rows.argtypes = [_vp, _vp, _vp, _i64, _i64, _i64, _i64, ctypes.c_int, ctypes.c_int]
        lib.oracle_ip_rows.restype = ctypes.c_int
        lib.oracle_ip_cols_unfused_f64.argtypes = [_vp, _vp, _vp, _i64, _i64, _i64, _i64]
        lib.oracle_ip_cols_unfused_f64.restype = ctypes.c_int
        lib.oracle_ip_f32_in_f64_acc.argtypes = [_vp, _vp, _vp, _i64, _i64, _i64]
        lib.oracle_ip_f32_in_f64_acc.restype = None
        for t in ("f64", "f32"):
            getattr(lib, f"oracle_hadamard_{t}").argtypes = [_vp, _vp, _vp, _i64, _i64]
            getattr(lib, f"oracle_hadamard_{t}").restype = None
            getattr(lib, f"oracle_kron_{t}").argtypes = [_vp, _vp, _vp, _i64, _i64, _i64, _i64]
            getattr(lib, f"oracle_kron_{t}").restype = None
        _lib = lib
    return _lib


def _tag(dtype) -> str:
    dt = np.dtype(dtype)
    if dt == np.float64:
        return "f64"
    if dt == np.float32:
        return "f32"
    raise TypeError(f"oracle supports float64/float32, got {dt}")


def _check(A: np.ndarray, B: np.ndarray):
    if A.ndim != 2 or B.ndim != 2 or A.shape[1] != B.shape[0]:
        raise ValueError(f"shape mismatch: rho A={A.shape}, rho B={B.shape} (Eq. 1, P:59-64)")
    if A.dtype != B.dtype:
        raise TypeError("A and B must share a dtype")
    return np.ascontiguousarray(A), np.ascontiguousarray(B)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def ip(A: np.ndarray, B: np.ndarray, fused: bool = False) -> np.ndarray:
    """Fig. 3 ``ip.c`` = Eq. 3: C := A • B, loop order i-σ-j.

    ``fused=False``: each step ``C = C + A*B`` with two roundings (R3 unfused).
    ``fused=True``: each step ``C = fma(A, B, C)`` (R3 contracted).
    """
    A, B = _check(A, B)
    m, n = A.shape
    p = B.shape[1]
    C = np.empty((m, p), dtype=A.dtype)
    fn = getattr(_load(), f"oracle_ip_{'fma' if fused else 'unfused'}_{_tag(A.dtype)}")
    fn(_ptr(C), _ptr(A), _ptr(B), m, p, n)
    return C


def ip_rows_subset(A: np.ndarray, B: np.ndarray, rows: Sequence[int], fused: bool = False) -> np.ndarray:
    """ip.c restricted to the rows ``rows`` of C (Fig. 1: rows are independent).

    Returns a len(rows) x p array; row r equals row rows[r] of ``ip(A, B)`` bit for bit.
    """
    A, B = _check(A, B)
    m, n = A.shape
    p = B.shape[1]
    R = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    C = np.empty((len(R), p), dtype=A.dtype)
    fn = getattr(_load(), f"oracle_ip_rowset_{'fma' if fused else 'unfused'}_{_tag(A.dtype)}")
    if fn(_ptr(C), _ptr(A), _ptr(B), m, p, n, _ptr(R), len(R)) != 0:
        raise IndexError("row index out of range (Eq. 2, P:66-72)")
    return C


def ip_rowblock(A_rows: np.ndarray, B: np.ndarray, fused: bool = False) -> np.ndarray:
    """ip.c over a caller-held block of rows of A (the rows of C they produce)."""
    A_rows, B = _check(A_rows, B)
    r, n = A_rows.shape
    p = B.shape[1]
    C = np.empty((r, p), dtype=A_rows.dtype)
    fn = getattr(_load(), f"oracle_ip_rowblock_{'fma' if fused else 'unfused'}_{_tag(A_rows.dtype)}")
    fn(_ptr(C), _ptr(A_rows), _ptr(B), r, p, n)
    return C


def ip_rows(A: np.ndarray, B: np.ndarray, np_: int, fused: bool = False) -> np.ndarray:
    """Fig. 4 ``ip_rows.c``: row lifting i = ip + (sizel/np)·k, one thread per k.

    R5: the listing assumes np | sizel; a non-dividing np raises ValueError.
    """
    A, B = _check(A, B)
    m, n = A.shape
    p = B.shape[1]
    C = np.empty((m, p), dtype=A.dtype)
    rc = _load().oracle_ip_rows(_ptr(C), _ptr(A), _ptr(B), m, p, np_, n, A.dtype.itemsize, int(fused))
    if rc != 0:
        raise ValueError(f"ip_rows.c needs np | sizel (P:157): m={m}, np={np_}")
    return C


def ip_cols(A: np.ndarray, B: np.ndarray, rsize: int) -> np.ndarray:
    """Fig. 5 ``ip_cols.c``, double, unfused: j = jp·rsize + kp."""
    A, B = _check(A, B)
    if A.dtype != np.float64:
        raise TypeError("ip_cols oracle is double-only (the listing's type, P:175)")
    m, n = A.shape
    p = B.shape[1]
    C = np.empty((m, p), dtype=np.float64)
    if _load().oracle_ip_cols_unfused_f64(_ptr(C), _ptr(A), _ptr(B), m, p, n, rsize) != 0:
        raise ValueError(f"ip_cols.c needs rsize | sizer (P:181): p={p}, rsize={rsize}")
    return C


def ip_ijk(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Classical row-of-A times column-of-B definition, unfused, k ascending."""
    A, B = _check(A, B)
    m, n = A.shape
    p = B.shape[1]
    C = np.empty((m, p), dtype=A.dtype)
    getattr(_load(), f"oracle_ip_ijk_unfused_{_tag(A.dtype)}")(_ptr(C), _ptr(A), _ptr(B), m, p, n)
    return C


def ip_f32_truth(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """fp32 operands, fp64 accumulation (reporting the TF32 variant's error only)."""
    A, B = _check(A, B)
    if A.dtype != np.float32:
        raise TypeError("float32 operands expected")
    m, n = A.shape
    p = B.shape[1]
    C = np.empty((m, p), dtype=np.float64)
    _load().oracle_ip_f32_in_f64_acc(_ptr(C), _ptr(A), _ptr(B), m, p, n)
    return C


def hadamard(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Hadamard product (pointwise ×)."""
    if A.shape != B.shape or A.ndim != 2 or A.dtype != B.dtype:
        raise ValueError("hadamard needs equal 2-D shapes and dtypes")
    A, B = np.ascontiguousarray(A), np.ascontiguousarray(B)
    C = np.empty_like(A)
    getattr(_load(), f"oracle_hadamard_{_tag(A.dtype)}")(_ptr(C), _ptr(A), _ptr(B), A.shape[0], A.shape[1])
    return C


def kron(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Kronecker product via the outer-product definition."""
    if A.ndim != 2 or B.ndim != 2 or A.dtype != B.dtype:
        raise ValueError("kron needs 2-D operands of one dtype")
    A, B = np.ascontiguousarray(A), np.ascontiguousarray(B)
    (m, n), (p, q) = A.shape, B.shape
    C = np.empty((m * p, n * q), dtype=A.dtype)
    getattr(_load(), f"oracle_kron_{_tag(A.dtype)}")(_ptr(C), _ptr(A), _ptr(B), m, n, p, q)
    return C


# ---------------------------------------------------------------------------
# Shapes, ψ and γ_row (appendix; SPEC S:65-119 for interface ideas)
# ---------------------------------------------------------------------------

def gamma_row(idx: Sequence[int], shape: Sequence[int]) -> int:
    """γ_row: full index → offset, by enumerating the row-major order.

    Written as the definition "position of idx in the row-major enumeration":
    offset = Σ_d idx[d] · π(shape[d+1:]).
    """
    if len(idx) != len(shape):
        raise IndexError("gamma needs a full index")
    for i, s in zip(idx, shape):
        if not (0 <= i < s):
            raise IndexError("invalid index (0 <=* i <* rho xi, P:462)")
    off = 0
    for d in range(len(shape)):
        off += idx[d] * math.prod(shape[d + 1:])
    return off


def psi(idx: Sequence[int], shape: Sequence[int]) -> tuple[int, int]:
    """ψ with a (full or prefix) index on a row-major array of shape ``shape``.

    Returns (offset, count): ψ(idx, ξ) is the contiguous slice rav(ξ)[offset:offset+count]
    (bracket bridge rav(i⃗ ψ ξ) ≡ (rav ξ)[γ(i⃗; ρξ)]; prefix-ψ contiguity).
    """
    q = len(idx)
    if q > len(shape):
        raise IndexError("index longer than the shape")
    full = list(idx) + [0] * (len(shape) - q)
    count = math.prod(shape[q:])
    if count == 0:
        # no valid completion of the prefix; still validate the prefix itself
        for i, s in zip(idx, shape):
            if not (0 <= i < s):
                raise IndexError("invalid index")
        return (0, 0)
    return (gamma_row(full, shape), count)


def lift_rows(m: int, nparts: int, part: int) -> tuple[int, int]:
    """Row lifting of the i axis onto ``nparts`` processors (Fig. 4).

    R5: ip_rows.c's ``sizel/np`` drops m mod np rows; the reading is a
    balanced contiguous split. Computed here by DEALING rows one at a time to the
    parts in turn (counts), then laying the parts out contiguously in part order.
    Returns (row0, rows) for ``part``.
    """
    if nparts <= 0 or not (0 <= part < nparts) or m < 0:
        raise ValueError("bad lift arguments")
    counts = [0] * nparts
    for r in range(m):
        counts[r % nparts] += 1
    row0 = sum(counts[:part])
    return (row0, counts[part])


def select_block_paper(l1_budget_bytes: int, elem_bytes: int) -> int:
    """Paper-mode block side: largest power-of-two b with 3 blocks
    (A, B, C) of b×b elements fitting the per-SM L1 budget ("three blocks per SM:
    for A, B, and C"; "must be less than or equal to 1 L1")."""
    if elem_bytes <= 0 or 3 * elem_bytes > l1_budget_bytes:
        raise ValueError("budget too small for a 1x1 block")
    b = 1
    while 3 * (2 * b) * (2 * b) * elem_bytes <= l1_budget_bytes:
        b *= 2
    return b
