"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

Holds none of the method's arithmetic (see moa_inputs.h). Matrix ids:
``ID_A = 1``, ``ID_B = 2``. Element (i, k) of a row-major matrix with row
length ``ncols`` has linear index ``i*ncols + k`` (γ_row), so any row block
can be regenerated independently on either side.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

UNIFORM = 0
INT = 1
ID_A = 1
ID_B = 2

_HERE = os.path.dirname(os.path.abspath(__file__))
_host = None
_dev = None
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64


def _build(target: str):
    import subprocess
    import sys
    subprocess.check_call([sys.executable, os.path.join(_HERE, "..", "tools", "build.py"), target])


def _load_host():
    global _host
    if _host is None:
        path = os.path.join(_HERE, "libmoa_inputs.so")
        if not os.path.exists(path):
            _build("inputs")
        lib = ctypes.CDLL(path)
        for t in ("f64", "f32"):
            fn = getattr(lib, f"moa_gen_fill_{t}_host")
            fn.argtypes = [ctypes.c_void_p, _i64, _u64, _u64, ctypes.c_int, _i64]
            fn.restype = None
        lib.moa_gen_hash_host.argtypes = [_u64, _u64, _i64]
        lib.moa_gen_hash_host.restype = _u64
        _host = lib
    return _host


def _load_dev():
    global _dev
    if _dev is None:
        path = os.path.join(_HERE, "libmoa_inputs_cuda.so")
        if not os.path.exists(path):
            _build("inputs_cuda")
        lib = ctypes.CDLL(path)
        for t in ("f64", "f32"):
            fn = getattr(lib, f"moa_gen_fill_{t}_device")
            fn.argtypes = [ctypes.c_void_p, _i64, _u64, _u64, ctypes.c_int, _i64, ctypes.c_void_p]
            fn.restype = ctypes.c_int
        _dev = lib
    return _dev


def hash64(seed: int, mid: int, idx: int) -> int:
    return int(_load_host().moa_gen_hash_host(seed, mid, idx))


def host_matrix(rows: int, cols: int, seed: int, mid: int, kind: int = UNIFORM,
                dtype=np.float64, row0: int = 0) -> np.ndarray:
    """Rows [row0, row0+rows) of the seeded matrix with row length ``cols``."""
    dt = np.dtype(dtype)
    out = np.empty((rows, cols), dtype=dt)
    fn = _load_host().moa_gen_fill_f64_host if dt == np.float64 else _load_host().moa_gen_fill_f32_host
    if rows * cols:
        fn(out.ctypes.data_as(ctypes.c_void_p), rows * cols, seed, mid, kind, row0 * cols)
    return out


def host_rows(row_ids, cols: int, seed: int, mid: int, kind: int = UNIFORM, dtype=np.float64) -> np.ndarray:
    """Arbitrary rows (by global row id) of the seeded matrix."""
    out = np.empty((len(row_ids), cols), dtype=np.dtype(dtype))
    for r, i in enumerate(row_ids):
        out[r] = host_matrix(1, cols, seed, mid, kind, dtype, row0=int(i))[0]
    return out


def device_fill(tensor, seed: int, mid: int, kind: int = UNIFORM, row0: int = 0, stream=None) -> None:
    """Fill a contiguous CUDA tensor (2-D, rows of A/B) with the seeded values in place."""
    import torch
    assert tensor.is_cuda and tensor.is_contiguous()
    cols = tensor.shape[-1] if tensor.dim() >= 1 else 1
    s = stream if stream is not None else torch.cuda.current_stream()
    lib = _load_dev()
    fn = lib.moa_gen_fill_f64_device if tensor.dtype == torch.float64 else lib.moa_gen_fill_f32_device
    rc = fn(ctypes.c_void_p(tensor.data_ptr()), tensor.numel(), seed, mid, kind, row0 * cols,
            ctypes.c_void_p(s.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"device generator failed: cudaError {rc}")
