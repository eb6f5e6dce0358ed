"""ctypes wrapper of oracle/liboracle.so (TEST INFRASTRUCTURE ONLY; see __init__)."""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from . import numpy_oracle as NO

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
_lib = None


class Tables(C.Structure):
    _fields_ = [("n", C.c_int), ("W", C.c_int), ("kind", C.c_int),
                ("S", C.c_double * 25), ("D", C.c_double * 25), ("w3", C.c_double * 125),
                ("grad_scale", C.c_double * 3)]


def build():
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        _lib = C.CDLL(str(LIB))
        _lib.oracle_cellop_apply.restype = C.c_int
        _lib.oracle_tmmult.restype = C.c_int
        _lib.oracle_mmult.restype = C.c_int
    return _lib


def _p(a, ct):
    if a is None:
        return C.cast(None, C.POINTER(ct))
    return a.ctypes.data_as(C.POINTER(ct))


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def tables(degree, spacing, kind, lane_width):
    S, D, _, _ = NO.lagrange_tables(degree)
    n = degree + 1
    t = Tables()
    t.n, t.W, t.kind = n, lane_width, (0 if kind == "mass" else 1)
    for i in range(n * n):
        t.S[i] = S.ravel()[i]
        t.D[i] = D.ravel()[i]
    w3 = NO.weights3(degree, spacing).ravel()
    for i in range(n**3):
        t.w3[i] = w3[i]
    for k in range(3):
        t.grad_scale[k] = 0.5 / spacing[k] ** 2
    return t


def cellop_apply(degree, spacing, kind, cell_lb, cell_rib, cell_color, vq, x_meta, h_meta,
                 col_strides, col_sizes, x_data, hx_data, lane_width=8, threads=None):
    """hx_data += Op x_data over the given cells (reference Algorithm 6, all lanes)."""
    lib = load()
    t = tables(degree, spacing, kind, lane_width)
    lb, rib = _i64(cell_lb), _i64(cell_rib)
    col = None if cell_color is None else np.ascontiguousarray(cell_color, dtype=np.int32)
    vq = None if vq is None else np.ascontiguousarray(vq, dtype=np.float64)
    xr, xc, xo = (_i64(a) for a in x_meta)
    hr, hc, ho = (_i64(a) for a in h_meta)
    cs, cz = _i64(col_strides), _i64(col_sizes)
    threads = int(threads or os.cpu_count() or 1)
    rc = lib.oracle_cellop_apply(
        C.byref(t), C.c_int64(lb.shape[0]), _p(lb, C.c_int64), _p(rib, C.c_int64),
        _p(col, C.c_int32), _p(vq, C.c_double), _p(xr, C.c_int64), _p(xc, C.c_int64),
        _p(xo, C.c_int64), _p(hr, C.c_int64), _p(hc, C.c_int64), _p(ho, C.c_int64),
        _p(cs, C.c_int64), _p(cz, C.c_int64), _p(x_data, C.c_double), _p(hx_data, C.c_double),
        C.c_int(threads))
    if rc == -3:
        raise LookupError("destination pattern misses a block (PatternError)")
    if rc != 0:
        raise RuntimeError(f"oracle_cellop_apply failed ({rc})")
    return threads


def matrix_meta(m):
    """(row_start, col_index, block_offsets) host arrays of a BlockCsrMatrix."""
    return m.row_start, m.col_index, m.block_offsets
