"""ctypes binding of libbmv.so (include/bmv.h).

The product path has no CPU fallback: if the library is missing or fails to
load, every compute entry point raises DeviceError.  Arrays handed to the
*_create functions are host numpy arrays (copied by the library); value
arrays are device pointers taken from torch tensors.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .errors import DeviceError, DomainError, PatternError, ShapeError

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libbmv.so"
MAX_NODES = 5

BMV_OK, BMV_ERR_INVALID, BMV_ERR_CUDA, BMV_ERR_PATTERN = 0, 1, 2, 3

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u32p = C.POINTER(C.c_uint32)
_f64p = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)


class CellopDesc(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("wide", C.c_int32), ("n_cells", C.c_int32),
        ("code_stride", C.c_int32), ("max_groups", C.c_int32), ("n_pairs", C.c_int64),
        ("gtab_len", C.c_int64), ("pair_cell", _i32p), ("pair_gtab", _i64p),
        ("pair_ngp", _i32p), ("gtab", _i32p), ("codes", _u32p),
        ("n_breaks", C.c_int32), ("breaks", _i64p),
        ("S", C.c_double * (MAX_NODES * MAX_NODES)), ("Dco", C.c_double * (MAX_NODES * MAX_NODES)),
        ("w", C.c_double * MAX_NODES), ("kin", C.c_double * 3), ("det", C.c_double),
    ]


class ChunkDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("n_parts", C.c_int32), ("stage_bytes", C.c_int32),
        ("n_chunks", C.c_int64), ("meta_len", C.c_int64), ("part_chunk_start", _i64p),
        ("chunk_meta", _i64p), ("meta", _i32p), ("chunk_a", _i64p), ("chunk_b", _i64p),
    ]


# (name, restype, argtypes) of every exported symbol; also used by the
# CPU-side test that the library exports exactly what bmv.h declares.
SIGNATURES = [
    ("bmv_version", C.c_int, []),
    ("bmv_last_error", C.c_char_p, []),
    ("bmv_device_sm_count", C.c_int, [C.POINTER(C.c_int)]),
    ("bmv_launch_count", C.c_int, [_i64p]),
    ("bmv_cellop_create", C.c_int, [C.POINTER(CellopDesc), C.POINTER(C.c_void_p)]),
    ("bmv_cellop_destroy", C.c_int, [C.c_void_p]),
    ("bmv_cellop_apply", C.c_int,
     [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64,
      C.c_void_p]),
    ("bmv_potential_gaussian", C.c_int,
     [C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
      C.c_double, C.c_double, C.c_void_p, C.c_void_p]),
    ("bmv_cellop_launches", C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    ("bmv_cellop_apply_hm", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
      C.c_int64, C.c_void_p]),
    ("bmv_cellop_apply_pairs", C.c_int,
     [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
      C.c_void_p]),
    ("bmv_cellop_apply_hm_pairs", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
      C.c_int64, C.c_int64, C.c_void_p]),
    ("bmv_chunk_plan_create", C.c_int, [C.POINTER(ChunkDesc), C.POINTER(C.c_void_p)]),
    ("bmv_chunk_plan_destroy", C.c_int, [C.c_void_p]),
    ("bmv_tmmult_run", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    ("bmv_mmult_run", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int32, C.c_void_p]),
    ("bmv_chunk_kernel_config", C.c_int, [C.c_int32, C.c_int32, _i32p, _i32p]),
    ("bmv_index_create", C.c_int, [_i64p, C.c_int64, C.POINTER(C.c_void_p)]),
    ("bmv_index_destroy", C.c_int, [C.c_void_p]),
    ("bmv_index_size", C.c_int64, [C.c_void_p]),
    ("bmv_gather", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("bmv_scatter", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    ("bmv_zero", C.c_int, [C.c_void_p, C.c_int64, C.c_void_p]),
    ("bmv_fp64_peak_kernel", C.c_int,
     [C.c_void_p, C.c_int32, C.c_int32, _f64p, C.c_void_p]),
    ("bmv_fp64_dmma_peak_kernel", C.c_int,
     [C.c_void_p, C.c_int32, C.c_int32, _f64p, C.c_void_p]),
]

_lock = threading.Lock()
_lib = None


def load(path: str | os.PathLike | None = None):
    """Load (once) and return the ctypes library; DeviceError if absent."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        if path is None and os.environ.get("BMV_LIB"):
            path = os.environ["BMV_LIB"]  # alternative build (kernel experiments)
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise DeviceError(
                f"{p} is missing: build it with `python -m paper_1907_01005_b200.build` "
                "(no CPU fallback exists for the operator path)")
        try:
            lib = C.CDLL(str(p))
        except OSError as exc:
            raise DeviceError(f"cannot load {p}: {exc}") from exc
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int, what: str = ""):
    if rc == BMV_OK:
        return
    msg = load().bmv_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == BMV_ERR_PATTERN:
        raise PatternError(text)
    if rc == BMV_ERR_INVALID:
        raise ShapeError(text)
    raise DeviceError(text)


def ptr(arr: np.ndarray, ctype):
    """Pointer into a contiguous numpy array (caller keeps the array alive)."""
    if arr is None or arr.size == 0:
        return C.cast(None, C.POINTER(ctype))
    assert arr.flags["C_CONTIGUOUS"]
    return arr.ctypes.data_as(C.POINTER(ctype))


def dptr(tensor) -> C.c_void_p:
    """Raw device pointer of a CUDA tensor (None for empty tensors)."""
    if tensor is None:
        return C.c_void_p(None)
    if not tensor.is_cuda:
        raise DeviceError("compute kernels need CUDA tensors; this matrix lives on the CPU")
    return C.c_void_p(tensor.data_ptr() if tensor.numel() else None)


def stream_handle(device=None) -> C.c_void_p:
    import torch

    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class Handle:
    """Owning wrapper of an opaque plan pointer (destroyed with the object)."""

    def __init__(self, destroy_name: str, raw: C.c_void_p, keep=()):
        self._destroy = getattr(load(), destroy_name)
        self.raw = raw
        self._keep = keep

    def __del__(self):
        try:
            if self.raw:
                self._destroy(self.raw)
                self.raw = None
        except Exception:
            pass


def launch_count() -> int:
    """Kernels libbmv has launched so far (counted at every launch site)."""
    v = C.c_int64()
    check(load().bmv_launch_count(C.byref(v)), "bmv_launch_count")
    return int(v.value)


def require_device():
    """Fail loudly unless a CUDA device and the library are both present."""
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the operator path runs only on the GPU")
    return load()
