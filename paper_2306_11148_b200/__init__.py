"""B200-native MoA Operational-Normal-Form GEMM (arXiv 2306.11148) — Python binding.

A thin ctypes layer over ``libmoa.so`` (C ABI in ``include/moa.h``). It only
marshals arguments: every step of the GEMM runs in the library's sm_100a
kernels. There is no CPU or PyTorch fallback — if the shared library is
missing or fails to load, importing this package raises.

PyTorch is used only for device memory, streams and process groups.

    import paper_2306_11148_b200 as moa
    C = moa.gemm(A, B)                      # C := A • B   (Eq. 3)
    off, cnt = moa.psi([1], [2, 2])         # ψ: contiguous slice of rav ξ
    r0, rows = moa.lift_rows(m, G, g)       # dimension lifting of the i axis
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional, Sequence

__all__ = [
    "F64", "F32", "F32_3XTF32", "MoAError", "Plan", "gemm", "gemm_with_plan", "gemm_host", "gemm_lifted",
    "psi", "lift_rows", "plan", "select_block_paper", "Comm", "lib_path", "abi_version", "KERNEL_NAMES",
    "gemm_lifted_direct",
    "gemm_acc", "lift_panels", "hadamard", "kron", "gemm_lifted_cols", "gemm_lifted_2d", "gemm_scatter",
    "gemm_lifted_gather", "gemm_lifted_host", "exchange_plan", "pull_panels", "Coll", "XPLAN_ROWS",
    "XPLAN_ROWS_HOST", "XPLAN_COLS", "XPLAN_2D", "XF_GATHER", "XF_FUSED_GATHER", "XF_PULL_B",
]

F64, F32, F32_3XTF32 = 0, 1, 2
KERNEL_NAMES = {0: "none", 1: "zero_fill", 2: "dgemm_tma", 3: "dgemm_generic", 4: "sgemm_ffma", 5: "sgemm_3xtf32",
                6: "sgemm_generic"}

_HERE = os.path.dirname(os.path.abspath(__file__))
# MOA_LIBRARY: an instrumented build of the same sources (tests/test_sanitizers.py loads
# build/asan/libmoa_asan.so, host code under -fsanitize=address,undefined); default: the
# in-tree libmoa.so. Never a different implementation.
lib_path = os.environ.get("MOA_LIBRARY") or os.path.join(_HERE, "libmoa.so")

if not os.path.exists(lib_path):
    raise ImportError(
        f"{lib_path} not found: build it with `python tools/build.py moa` (or __graft_entry__.build()). "
        "There is deliberately no fallback implementation.")
_lib = ctypes.CDLL(lib_path)

_i64, _i32, _vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p


class _PlanT(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int32), ("bm", ctypes.c_int32), ("bn", ctypes.c_int32), ("bk", ctypes.c_int32),
                ("stages", ctypes.c_int32), ("threads", ctypes.c_int32), ("ctas_per_sm", ctypes.c_int32),
                ("grid", ctypes.c_int32), ("tiles_m", ctypes.c_int64), ("tiles_n", ctypes.c_int64),
                ("tiles", ctypes.c_int64), ("raster_group", ctypes.c_int32), ("smem_bytes", ctypes.c_int32),
                ("sms", ctypes.c_int32), ("reserved", ctypes.c_int32)]


def _sig(name, argtypes, restype=ctypes.c_int):
    fn = getattr(_lib, name)
    fn.argtypes = argtypes
    fn.restype = restype
    return fn


_moa_gemm = _sig("moa_gemm", [_i64, _i64, _i64, _vp, _vp, _vp, _i32, _vp])
_moa_gemm_with_plan = _sig("moa_gemm_with_plan", [_i64, _i64, _i64, _vp, _vp, _vp, _i32, ctypes.POINTER(_PlanT), _vp])
_moa_gemm_host = _sig("moa_gemm_host", [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp])
_moa_gemm_lifted_host = _sig("moa_gemm_lifted_host", [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _vp])
_moa_gemm_lifted = _sig("moa_gemm_lifted", [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _i32, _vp, _vp])
_moa_gemm_lifted_ex = _sig("moa_gemm_lifted_ex", [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _i32])
_moa_gemm_lifted_direct = _sig("moa_gemm_lifted_direct", [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _i32, _vp, _vp])
_moa_gemm_acc = _sig("moa_gemm_acc", [_i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _i32, _i32, _vp])
_moa_lift_panels = _sig("moa_lift_panels", [_i64, _i64, _i32, _i32])
_moa_gemm_lifted_cols = _sig("moa_gemm_lifted_cols", [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _i32, _vp, _vp])
_moa_gemm_lifted_2d = _sig("moa_gemm_lifted_2d", [_i64, _i64, _i64, _i32, _i32, _vp, _vp, _vp, _i32, _vp, _vp])
_moa_gemm_lifted_2d_gather = _sig("moa_gemm_lifted_2d_gather", [_i64, _i64, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _i32,
                                                                _vp, _vp])
_moa_gemm_scatter = _sig("moa_gemm_scatter", [_i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _i32, _i32,
                                              ctypes.POINTER(_vp), _i32, _vp])
_moa_gemm_lifted_gather = _sig("moa_gemm_lifted_gather", [_i64, _i64, _i64, _vp, _vp, _vp, _i32, _vp, _vp, _i32])
_moa_comm_alloc_window = _sig("moa_comm_alloc_window", [_vp, ctypes.c_size_t, ctypes.POINTER(_vp)])
_moa_comm_free_window = _sig("moa_comm_free_window", [_vp, _vp])
_moa_comm_window_peer = _sig("moa_comm_window_peer", [_vp, _vp, _i32, ctypes.POINTER(_vp)])
_moa_hadamard = _sig("moa_hadamard", [_i64, _i64, _vp, _vp, _vp, _i32, _vp])
_moa_kron = _sig("moa_kron", [_i64, _i64, _i64, _i64, _vp, _vp, _vp, _i32, _vp])
_moa_psi = _sig("moa_psi", [_i32, ctypes.POINTER(_i64), _i32, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                            ctypes.POINTER(_i64)])
_moa_lift_rows = _sig("moa_lift_rows", [_i64, _i32, _i32, ctypes.POINTER(_i64), ctypes.POINTER(_i64)])
_moa_plan = _sig("moa_plan", [_i64, _i64, _i64, _i32, _i32, ctypes.POINTER(_PlanT)])
_moa_select_block_paper = _sig("moa_select_block_paper", [_i64, _i32, ctypes.POINTER(_i64)])
_moa_comm_get_unique_id = _sig("moa_comm_get_unique_id", [ctypes.c_char_p])
_moa_comm_init = _sig("moa_comm_init", [_i32, _i32, ctypes.c_char_p, _i32, ctypes.POINTER(_vp)])
_moa_comm_destroy = _sig("moa_comm_destroy", [_vp])
_moa_comm_agree = _sig("moa_comm_agree", [_vp, _i32, ctypes.POINTER(_i32)])


class _CollT(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("comm", ctypes.c_int32), ("root", ctypes.c_int32), ("group", ctypes.c_int32),
                ("operand", ctypes.c_int32), ("phase", ctypes.c_int32), ("panel", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("offset", ctypes.c_int64), ("count", ctypes.c_int64)]


_moa_exchange_plan = _sig("moa_exchange_plan", [_i32, _i64, _i64, _i64, _i32, _i32, _i32, _i32, _i32, _i32, _i32,
                                                ctypes.POINTER(_CollT), _i32, ctypes.POINTER(_i32)])
_moa_pull_panels = _sig("moa_pull_panels", [_i64, ctypes.POINTER(_i64)])
_moa_status_string = _sig("moa_status_string", [_i32], ctypes.c_char_p)
_moa_last_error = _sig("moa_last_error", [], ctypes.c_char_p)
_moa_abi_version = _sig("moa_abi_version", [])


class MoAError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        name = _moa_status_string(status).decode()
        detail = (_moa_last_error() or b"").decode()
        super().__init__(f"{where}: {name} ({detail})")
        self.name = name


def _check(rc: int, where: str):
    if rc != 0:
        raise MoAError(rc, where)


def abi_version() -> int:
    return int(_moa_abi_version())


# ----------------------------------------------------------------- helpers ---

def psi(idx: Sequence[int], shape: Sequence[int]) -> tuple[int, int]:
    """ψ(idx, ξ) on a row-major ξ of shape ``shape`` -> (offset, count) of rav ξ (moa.h)."""
    r, q = len(shape), len(idx)
    sh = (_i64 * max(r, 1))(*shape)
    ix = (_i64 * max(q, 1))(*idx)
    off, cnt = _i64(), _i64()
    _check(_moa_psi(r, sh, q, ix, ctypes.byref(off), ctypes.byref(cnt)), "moa_psi")
    return off.value, cnt.value


def lift_rows(m: int, nparts: int, part: int) -> tuple[int, int]:
    """Row lifting: (row0, rows) owned by ``part`` of ``nparts``."""
    r0, r = _i64(), _i64()
    _check(_moa_lift_rows(m, nparts, part, ctypes.byref(r0), ctypes.byref(r)), "moa_lift_rows")
    return r0.value, r.value


def lift_panels(n: int, p: int, dtype: int = F64, nranks: int = 1) -> int:
    """Static k-panel count of the pipelined lifted exchange (moa_lift_panels)."""
    return int(_moa_lift_panels(n, p, dtype, nranks))


XPLAN_ROWS, XPLAN_ROWS_HOST, XPLAN_COLS, XPLAN_2D = 0, 1, 2, 3
XF_GATHER, XF_FUSED_GATHER, XF_PULL_B, XF_DIRECT_B = 1, 2, 4, 8
_COLL_OPS = {1: "broadcast", 2: "allgather", 3: "barrier", 4: "pull"}
_COMM_KINDS = {0: "world", 1: "pipe", 2: "row", 3: "col"}
_OPERANDS = {0: "A", 1: "B", 2: "C"}


@dataclass
class Coll:
    """One collective of a lifted call's exchange plan (moa_exchange_plan)."""
    op: str
    comm: str
    root: int
    group: int
    operand: str
    phase: int
    panel: int
    offset: int
    count: int


def exchange_plan(variant: int, m: int, n: int, p: int, dtype: int = F64, nranks: int = 1, rank: int = 0,
                  grid_rows: int = 0, grid_cols: int = 0, npanels: int = 0, flags: int = 0) -> list:
    """The ordered collectives a lifted call issues on `rank` (pure function, no GPU)."""
    need = _i32()
    cap = 64
    while True:
        arr = (_CollT * cap)()
        rc = _moa_exchange_plan(variant, m, n, p, dtype, nranks, rank, grid_rows, grid_cols, npanels, flags, arr, cap,
                                ctypes.byref(need))
        if rc != 0 and need.value > cap:
            cap = need.value
            continue
        _check(rc, "moa_exchange_plan")
        return [Coll(_COLL_OPS[o.op], _COMM_KINDS[o.comm], o.root, o.group, _OPERANDS[o.operand], o.phase, o.panel,
                     o.offset, o.count) for o in arr[:need.value]]


def pull_panels(n: int) -> list:
    """k-panel boundaries of B for the copy-engine pulled exchange (moa_pull_panels)."""
    bnd = (_i64 * 17)()
    k = int(_moa_pull_panels(n, bnd))
    return [int(b) for b in bnd[:k + 1]]


def select_block_paper(l1_budget_bytes: int, elem_bytes: int) -> int:
    b = _i64()
    _check(_moa_select_block_paper(l1_budget_bytes, elem_bytes, ctypes.byref(b)), "moa_select_block_paper")
    return b.value


@dataclass
class Plan:
    kernel: str
    bm: int
    bn: int
    bk: int
    stages: int
    threads: int
    ctas_per_sm: int
    grid: int
    tiles_m: int
    tiles_n: int
    tiles: int
    raster_group: int
    smem_bytes: int
    sms: int

    @classmethod
    def _from(cls, p: _PlanT) -> "Plan":
        return cls(KERNEL_NAMES.get(p.kernel, str(p.kernel)), p.bm, p.bn, p.bk, p.stages, p.threads, p.ctas_per_sm,
                   p.grid, p.tiles_m, p.tiles_n, p.tiles, p.raster_group, p.smem_bytes, p.sms)

    def _to(self) -> _PlanT:
        inv = {v: k for k, v in KERNEL_NAMES.items()}
        return _PlanT(inv[self.kernel], self.bm, self.bn, self.bk, self.stages, self.threads, self.ctas_per_sm,
                      self.grid, self.tiles_m, self.tiles_n, self.tiles, self.raster_group, self.smem_bytes,
                      self.sms, 0)


def plan(m: int, n: int, p: int, dtype: int = F64, device: int = -1) -> Plan:
    """The static block plan the library will use for an aligned (m, n, p) call."""
    out = _PlanT()
    _check(_moa_plan(m, n, p, dtype, device, ctypes.byref(out)), "moa_plan")
    return Plan._from(out)


# ------------------------------------------------------------------- gemm ---

def _torch():
    import torch
    return torch


_raw_stream = None


def _stream_ptr(stream, device_index=None) -> int:
    """Raw cudaStream_t of ``stream`` or of the current stream. The current stream is
    read with torch's raw getter when present (building a torch Stream object per
    call cost ~2 us of host time, tools/host_overhead.py)."""
    global _raw_stream
    if stream is not None:
        return stream.cuda_stream
    torch = _torch()
    if _raw_stream is None:
        _raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", False)
    if _raw_stream:
        return _raw_stream(torch.cuda.current_device() if device_index is None else device_index)
    return torch.cuda.current_stream().cuda_stream


def _arg(t, name: str, shape, dtype, *, cuda: Optional[bool] = True, layout: str = "contiguous",
         optional: bool = False):
    """The one validator every wrapper uses before handing raw pointers to the C ABI,
    which cannot check buffer sizes itself: `t` must be a tensor of exactly `shape`
    (None entries match any extent), of `dtype`, on the GPU (cuda=True) or host
    (cuda=False; None = either), and contiguous or row-major ("rows": unit column
    stride, any row stride >= the row length). Returns t."""
    if t is None:
        if optional:
            return None
        raise ValueError(f"{name} is required")
    torch = _torch()
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch tensor")
    if t.dim() != len(shape) or any(want is not None and have != want for have, want in zip(t.shape, shape)):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple('*' if d is None else d for d in shape)} "
                         "(Eq. 1, P:59-64)")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if cuda is not None and t.is_cuda != cuda:
        raise ValueError(f"{name} must be a {'CUDA' if cuda else 'host (CPU)'} tensor")
    if layout == "contiguous":
        if not t.is_contiguous():
            raise ValueError(f"{name} must be row-major contiguous (P:77-82)")
    elif t.numel() > 0 and (t.stride(-1) != 1 or (t.dim() == 2 and t.shape[0] > 1 and t.stride(0) < t.shape[1])):
        raise ValueError(f"{name} must be a row-major view (unit column stride, row stride >= row length)")
    return t


def _code(dtype, precision: Optional[str]) -> int:
    torch = _torch()
    if dtype == torch.float64:
        code = F64
    elif dtype == torch.float32:
        code = F32
    else:
        raise TypeError(f"unsupported dtype {dtype} (float64 or float32)")
    if precision == "3xtf32":
        if code != F32:
            raise TypeError("precision='3xtf32' needs float32 operands")
        return F32_3XTF32
    if precision not in (None, "exact"):
        raise ValueError(f"unknown precision {precision!r} (None, 'exact' or '3xtf32')")
    return code


def _ld(t) -> int:
    """Row stride (elements) of a row-major 2-D view; a view with <= 1 row has no
    meaningful stride, so its row length is passed."""
    if t.shape[0] <= 1 or t.numel() == 0:
        return max(int(t.shape[1]), 1)
    return int(t.stride(0))


def gemm(A, B, out=None, *, precision: Optional[str] = None, stream=None):
    """C := A • B on the GPU (ONF, row-major contiguous). ``precision='3xtf32'`` selects
    the TF32 tensor-core variant for float32 operands. Asynchronous on ``stream``."""
    torch = _torch()
    _arg(A, "A", (None, None), None)
    m, n = A.shape
    _arg(B, "B", (n, None), A.dtype)
    p = B.shape[1]
    if out is None:
        out = torch.empty((m, p), dtype=A.dtype, device=A.device)
    _arg(out, "out", (m, p), A.dtype)
    code = _code(A.dtype, precision)
    _check(_moa_gemm(m, n, p, A.data_ptr() or None, B.data_ptr() or None, out.data_ptr() or None, code,
                     _stream_ptr(stream, A.get_device())), "moa_gemm")
    return out


def gemm_with_plan(A, B, out, plan_: Plan, *, precision: Optional[str] = None, stream=None):
    """moa_gemm with an explicit (edited) plan: the block-size experiment."""
    _arg(A, "A", (None, None), None)
    m, n = A.shape
    _arg(B, "B", (n, None), A.dtype)
    p = B.shape[1]
    _arg(out, "out", (m, p), A.dtype)
    code = _code(A.dtype, precision)
    pt = plan_._to()
    _check(_moa_gemm_with_plan(m, n, p, A.data_ptr() or None, B.data_ptr() or None, out.data_ptr() or None, code,
                               ctypes.byref(pt), _stream_ptr(stream, A.get_device())), "moa_gemm_with_plan")
    return out


def gemm_acc(A, B, C, accumulate: bool, *, precision: Optional[str] = None, stream=None):
    """C (+)= A • B on row-major (possibly row-strided) CUDA views: A may be a column
    slice A_full[:, k0:k1], B a row panel, C any row-major view (moa_gemm_acc)."""
    _arg(A, "A", (None, None), None, layout="rows")
    m, n = A.shape
    _arg(B, "B", (n, None), A.dtype, layout="rows")
    p = B.shape[1]
    _arg(C, "C", (m, p), A.dtype, layout="rows")
    code = _code(A.dtype, precision)
    _check(_moa_gemm_acc(m, n, p, A.data_ptr() or None, _ld(A), B.data_ptr() or None, _ld(B), C.data_ptr() or None,
                         _ld(C), int(bool(accumulate)), code, _stream_ptr(stream, A.get_device())), "moa_gemm_acc")
    return C


def hadamard(A, B, out=None, *, stream=None):
    """C = A ∘ B (pointwise ×) on the GPU (moa_hadamard)."""
    torch = _torch()
    _arg(A, "A", (None, None), None)
    _arg(B, "B", tuple(A.shape), A.dtype)
    out = torch.empty_like(A) if out is None else out
    _arg(out, "out", tuple(A.shape), A.dtype)
    m, n = A.shape
    _check(_moa_hadamard(m, n, A.data_ptr() or None, B.data_ptr() or None, out.data_ptr() or None,
                         _code(A.dtype, None), _stream_ptr(stream, A.get_device())), "moa_hadamard")
    return out


def kron(A, B, out=None, *, stream=None):
    """C = A ⊗ B (outer product + ravel) on the GPU (moa_kron)."""
    torch = _torch()
    _arg(A, "A", (None, None), None)
    _arg(B, "B", (None, None), A.dtype)
    (m, n), (p, q) = A.shape, B.shape
    out = torch.empty((m * p, n * q), dtype=A.dtype, device=A.device) if out is None else out
    _arg(out, "out", (m * p, n * q), A.dtype)
    _check(_moa_kron(m, n, p, q, A.data_ptr() or None, B.data_ptr() or None, out.data_ptr() or None,
                     _code(A.dtype, None), _stream_ptr(stream, A.get_device())), "moa_kron")
    return out


def gemm_host(A_host, B_host, C_host, A_dev, B_dev, C_dev, *, precision: Optional[str] = None, stream=None):
    """End-to-end C-ABI call on host buffers (pinned torch CPU tensors): H2D, GEMM, D2H, sync."""
    _arg(A_host, "A_host", (None, None), None, cuda=False)
    m, n = A_host.shape
    _arg(B_host, "B_host", (n, None), A_host.dtype, cuda=False)
    p = B_host.shape[1]
    _arg(C_host, "C_host", (m, p), A_host.dtype, cuda=False)
    _arg(A_dev, "A_dev", (m, n), A_host.dtype)
    _arg(B_dev, "B_dev", (n, p), A_host.dtype)
    _arg(C_dev, "C_dev", (m, p), A_host.dtype)
    code = _code(A_host.dtype, precision)
    _check(_moa_gemm_host(m, n, p, A_host.data_ptr() or None, B_host.data_ptr() or None, C_host.data_ptr() or None,
                          A_dev.data_ptr() or None, B_dev.data_ptr() or None, C_dev.data_ptr() or None, code,
                          _stream_ptr(stream, A_dev.get_device())), "moa_gemm_host")
    return C_host


# ------------------------------------------------------------ multi-GPU ----

class _WindowMem:
    """__cuda_array_interface__ of a library-owned window. It holds a reference to
    its Comm, so the communicator (whose destruction frees the window) lives at least
    as long as any tensor made from it."""

    def __init__(self, comm, ptr: int, shape, typestr: str):
        self.comm = comm
        self.__cuda_array_interface__ = {"shape": tuple(int(d) for d in shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None, "stream": None}


class Comm:
    """Library-owned NCCL communicator; the 128-byte id travels over torch.distributed."""

    @staticmethod
    def exchange_unique_id(group=None, make_id=None) -> bytes:
        """Rank 0 makes the 128-byte NCCL unique id (moa_comm_get_unique_id) and every
        rank receives it over torch.distributed (any backend, e.g. gloo)."""
        import torch.distributed as dist
        rank = dist.get_rank(group)
        blob = None
        if rank == 0:
            if make_id is None:
                uid = ctypes.create_string_buffer(128)
                _check(_moa_comm_get_unique_id(uid), "moa_comm_get_unique_id")
                blob = bytes(uid.raw)
            else:
                blob = bytes(make_id())
            if len(blob) != 128:
                raise ValueError("unique id must be 128 bytes")
        obj = [blob]
        dist.broadcast_object_list(obj, src=0, group=group)
        return obj[0]

    def __init__(self, group=None, device: Optional[int] = None):
        torch = _torch()
        import torch.distributed as dist
        self._h = None
        self._windows = set()
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = torch.cuda.current_device() if device is None else device
        uid = ctypes.create_string_buffer(Comm.exchange_unique_id(group), 128)
        h = _vp()
        _check(_moa_comm_init(self.world, self.rank, uid, self.device, ctypes.byref(h)), "moa_comm_init")
        self._h = h

    @property
    def handle(self):
        if not self._h:
            raise ValueError("communicator is closed")
        return self._h

    def agree(self, local_status: int = 0) -> int:
        """COLLECTIVE: the maximum of local_status over ranks (moa_comm_agree)."""
        out = _i32()
        _check(_moa_comm_agree(self.handle, int(local_status), ctypes.byref(out)), "moa_comm_agree")
        return int(out.value)

    def alloc_window(self, shape: Sequence[int], dtype=None):
        """COLLECTIVE: a tensor of `shape` in NCCL symmetric memory registered on this
        communicator (moa_comm_alloc_window): the C_full of gemm_lifted_gather, or a B
        whose exchange is then copy-engine pulls (gemm_lifted). The library owns the
        memory; release it with free_window (collective) or close(). The tensor keeps
        this Comm alive; close() invalidates every window tensor."""
        torch = _torch()
        dtype = torch.float64 if dtype is None else dtype
        numel = 1
        for d in shape:
            numel *= int(d)
        esize = torch.empty((), dtype=dtype).element_size()
        ptr = _vp()
        _check(_moa_comm_alloc_window(self.handle, max(1, numel) * esize, ctypes.byref(ptr)), "moa_comm_alloc_window")
        typestr = {torch.float64: "<f8", torch.float32: "<f4"}[dtype]
        t = torch.as_tensor(_WindowMem(self, int(ptr.value), shape, typestr), device=torch.device("cuda", self.device))
        self._windows.add(int(ptr.value))
        return t

    def free_window(self, t) -> None:
        """COLLECTIVE: release a tensor from alloc_window (moa_comm_free_window)."""
        ptr = t.data_ptr()
        self._windows.discard(ptr)
        _check(_moa_comm_free_window(self.handle, ptr), "moa_comm_free_window")

    def window_peer(self, t, peer: int) -> int:
        """Address, in this process, of rank `peer`'s copy of window tensor t's first element."""
        out = _vp()
        _check(_moa_comm_window_peer(self.handle, t.data_ptr(), peer, ctypes.byref(out)), "moa_comm_window_peer")
        return int(out.value or 0)

    def close(self):
        if self._h:
            self._windows.clear()
            h, self._h = self._h, None
            _check(_moa_comm_destroy(h), "moa_comm_destroy")

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gemm_lifted(m: int, A_local, B, C_local, comm: Comm, C_full=None, *, precision: Optional[str] = None,
                stream=None, npanels: int = 0):
    """Row-lifted C := A • B across the communicator (collective; see moa.h). If B is a
    comm.alloc_window tensor on every rank, the exchange is copy-engine pulls."""
    _arg(B, "B", (None, None), None)
    n, p = B.shape
    r0, rows = lift_rows(m, comm.world, comm.rank)
    _arg(A_local, "A_local", (rows, n), B.dtype)
    _arg(C_local, "C_local", (rows, p), B.dtype)
    _arg(C_full, "C_full", (m, p), B.dtype, optional=True)
    code = _code(B.dtype, precision)
    _check(_moa_gemm_lifted_ex(m, n, p, A_local.data_ptr() or None, B.data_ptr() or None,
                               C_local.data_ptr() or None, None if C_full is None else (C_full.data_ptr() or None),
                               code, _stream_ptr(stream, B.get_device()), comm.handle, npanels), "moa_gemm_lifted_ex")
    return C_local


def gemm_lifted_direct(m: int, A_local, B, C_local, comm: Comm, C_full=None, *, stream=None):
    """Row-lifted C := A • B with no copy of B (moa_gemm_lifted_direct; collective): B is
    a comm.alloc_window tensor on every rank, and every rank's GEMM reads rank 0's copy
    in place over NVLink."""
    _arg(B, "B", (None, None), None)
    n, p = B.shape
    r0, rows = lift_rows(m, comm.world, comm.rank)
    _arg(A_local, "A_local", (rows, n), B.dtype)
    _arg(C_local, "C_local", (rows, p), B.dtype)
    _arg(C_full, "C_full", (m, p), B.dtype, optional=True)
    code = _code(B.dtype, None)
    _check(_moa_gemm_lifted_direct(m, n, p, A_local.data_ptr() or None, B.data_ptr() or None,
                                   C_local.data_ptr() or None, None if C_full is None else (C_full.data_ptr() or None),
                                   code, _stream_ptr(stream, B.get_device()), comm.handle), "moa_gemm_lifted_direct")
    return C_local


def gemm_lifted_host(m: int, A_host, B_host, C_host, A_dev, B_dev, C_dev, comm: Comm, *, stream=None):
    """End-to-end row-lifted GEMM on HOST buffers (moa_gemm_lifted_host; collective,
    synchronous): this rank's rows of A/C on the host, B on rank 0's host (None
    elsewhere), device buffers for the rank's rows and all of B."""
    _arg(B_dev, "B_dev", (None, None), None)
    n, p = B_dev.shape
    r0, rows = lift_rows(m, comm.world, comm.rank)
    dt = B_dev.dtype
    _arg(A_host, "A_host", (rows, n), dt, cuda=False)
    _arg(B_host, "B_host", (n, p), dt, cuda=False, optional=comm.rank != 0)
    _arg(C_host, "C_host", (rows, p), dt, cuda=False)
    _arg(A_dev, "A_dev", (rows, n), dt)
    _arg(C_dev, "C_dev", (rows, p), dt)
    _check(_moa_gemm_lifted_host(m, n, p, A_host.data_ptr() or None,
                                 None if B_host is None else (B_host.data_ptr() or None), C_host.data_ptr() or None,
                                 A_dev.data_ptr() or None, B_dev.data_ptr() or None, C_dev.data_ptr() or None,
                                 _code(dt, None), _stream_ptr(stream, B_dev.get_device()), comm.handle),
           "moa_gemm_lifted_host")
    return C_host


def gemm_lifted_gather(m: int, A_local, B, C_full, comm: Comm, *, precision: Optional[str] = None, stream=None,
                       npanels: int = 0):
    """Row-lifted C := A • B with the all-gather of C fused into the GEMM epilogue
    (moa_gemm_lifted_gather; collective). C_full (m x p) must come from
    comm.alloc_window; on return (stream order) it holds all of C on every rank."""
    _arg(B, "B", (None, None), None)
    n, p = B.shape
    r0, rows = lift_rows(m, comm.world, comm.rank)
    _arg(A_local, "A_local", (rows, n), B.dtype)
    _arg(C_full, "C_full", (m, p), B.dtype)
    _check(_moa_gemm_lifted_gather(m, n, p, A_local.data_ptr() or None, B.data_ptr() or None,
                                   C_full.data_ptr() or None, _code(B.dtype, precision), _stream_ptr(stream, B.get_device()),
                                   comm.handle, npanels), "moa_gemm_lifted_gather")
    return C_full


def gemm_scatter(A, B, out, dsts, *, accumulate: bool = False, precision: Optional[str] = None, stream=None):
    """C (+)= A • B (moa_gemm_acc semantics) whose epilogue also writes every final C
    tile to each tensor (or raw device address) in `dsts` — the fused-gather epilogue
    on one GPU (moa_gemm_scatter). A and B may be row-strided 2-D views (e.g. a
    k-panel A[:, k0:k1], B[k0:k1, :]); out and every dst tensor are m x p contiguous.
    precision='3xtf32' (float32) runs the tcgen05 variant with the same epilogue."""
    _arg(A, "A", (None, None), None, layout="rows")
    m, n = A.shape
    _arg(B, "B", (n, None), A.dtype, layout="rows")
    p = B.shape[1]
    _arg(out, "out", (m, p), A.dtype)
    addrs = []
    for i, d in enumerate(dsts):
        if isinstance(d, int):
            addrs.append(d)        # a raw device address (e.g. a peer mapping): caller-sized
        else:
            addrs.append(_arg(d, f"dsts[{i}]", (m, p), A.dtype).data_ptr())
    arr = (_vp * max(1, len(addrs)))(*[a or None for a in addrs])
    _check(_moa_gemm_scatter(m, n, p, A.data_ptr() or None, _ld(A), B.data_ptr() or None, _ld(B),
                             out.data_ptr() or None, max(1, p), 1 if accumulate else 0, len(addrs), arr,
                             _code(A.dtype, precision), _stream_ptr(stream, A.get_device())), "moa_gemm_scatter")
    return out


def gemm_lifted_cols(A, B_local, C_local, p: int, comm: Comm, C_full=None, workspace=None, *, stream=None):
    """Column-lifted C := A • B across the communicator (collective; moa_gemm_lifted_cols).
    Rank g passes its column block B_local (n x cols_g) and receives C_local (m x cols_g)."""
    _arg(A, "A", (None, None), None)
    m, n = A.shape
    c0, cols = lift_rows(p, comm.world, comm.rank)
    _arg(B_local, "B_local", (n, cols), A.dtype)
    _arg(C_local, "C_local", (m, cols), A.dtype)
    _arg(C_full, "C_full", (m, p), A.dtype, optional=True)
    if workspace is not None:
        _arg(workspace, "workspace", (None,) * workspace.dim(), A.dtype)
        if workspace.numel() < m * (-(-p // comm.world)):
            raise ValueError("workspace must hold m * ceil(p / G) elements")
    _check(_moa_gemm_lifted_cols(m, n, p, A.data_ptr() or None, B_local.data_ptr() or None,
                                 C_local.data_ptr() or None, None if C_full is None else (C_full.data_ptr() or None),
                                 None if workspace is None else (workspace.data_ptr() or None), _code(A.dtype, None),
                                 _stream_ptr(stream, A.get_device()), comm.handle), "moa_gemm_lifted_cols")
    return C_local


def gemm_lifted_2d(m: int, p: int, grid_rows: int, grid_cols: int, A_panel, B_panel, C_block, comm: Comm, *,
                   C_full=None, stream=None):
    """2-D lifted C := A • B on a grid_rows x grid_cols process grid (moa_gemm_lifted_2d);
    with C_full (a comm.alloc_window tensor) the all-gather of C is fused into the GEMM
    epilogue (moa_gemm_lifted_2d_gather)."""
    rows = cols = None   # a grid that does not match the communicator: the C ABI reports it
    if grid_rows > 0 and grid_cols > 0 and grid_rows * grid_cols == comm.world:
        r, c = divmod(comm.rank, grid_cols)
        _, rows = lift_rows(m, grid_rows, r)
        _, cols = lift_rows(p, grid_cols, c)
    _arg(A_panel, "A_panel", (rows, None), None)
    n = A_panel.shape[1]
    _arg(B_panel, "B_panel", (n, cols), A_panel.dtype)
    _arg(C_block, "C_block", (rows, cols), A_panel.dtype)
    code = _code(A_panel.dtype, None)
    sp = _stream_ptr(stream, A_panel.get_device())
    if C_full is not None:
        _arg(C_full, "C_full", (m, p), A_panel.dtype)
        _check(_moa_gemm_lifted_2d_gather(m, n, p, grid_rows, grid_cols, A_panel.data_ptr() or None,
                                          B_panel.data_ptr() or None, C_block.data_ptr() or None,
                                          C_full.data_ptr() or None, code, sp, comm.handle),
               "moa_gemm_lifted_2d_gather")
        return C_block
    _check(_moa_gemm_lifted_2d(m, n, p, grid_rows, grid_cols, A_panel.data_ptr() or None, B_panel.data_ptr() or None,
                               C_block.data_ptr() or None, code, sp, comm.handle), "moa_gemm_lifted_2d")
    return C_block
