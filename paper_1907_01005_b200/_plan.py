"""ctypes binding of libbmvplan.so (include/bmv_plan.h): the native host plan builder.

The numpy functions it replaces stay in their modules as the readable
restatement (`hashed_entries`, `ColumnSupport.owned_entries`,
`_first_occurrence_groups`); tests/test_plan_native.py pins the native
results to them bit for bit.  BMV_PLAN_NATIVE=0 selects the numpy forms.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .errors import ConsistencyError, UsageError

LIB_PATH = Path(__file__).resolve().parent / "libbmvplan.so"

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_lib = None
_lock = threading.Lock()


def enabled() -> bool:
    return os.environ.get("BMV_PLAN_NATIVE", "1") != "0"


def load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise UsageError(f"{LIB_PATH.name} is not built (python -m paper_1907_01005_b200.build)")
        lib = C.CDLL(str(LIB_PATH))
        lib.bmvp_version.restype = C.c_int
        lib.bmvp_hash_fill.argtypes = [C.c_uint64, C.c_int64, _i64p, _i64p, _i64p, _i64p,
                                       C.c_double, _f64p]
        lib.bmvp_blocks_of.argtypes = [C.c_int64, _i64p, C.c_int64, _i64p, _i64p, _i64p]
        lib.bmvp_owned_entries_count.argtypes = [C.c_int64, _i64p, _i64p, C.c_int64, C.c_int64,
                                                 _i64p]
        lib.bmvp_owned_entries_fill.argtypes = [C.c_int64, _i64p, _i64p, C.c_int64, C.c_int64,
                                                _i64p, C.c_int64, _i64p, C.c_int64, _i64p, _i64p,
                                                _i64p, _i64p, _i64p, _i64p, _i64p, _i64p]
        lib.bmvp_first_groups_count.argtypes = [C.c_int64, C.c_int32, _i64p, _i64p, _i64p]
        lib.bmvp_first_groups_fill.argtypes = [C.c_int64, C.c_int32, _i64p, _i64p, _i64p, _i64p,
                                               _i64p]
        lib.bmvp_grow_count.argtypes = [C.c_int64, C.c_int32, _i64p, C.c_int64, C.c_int64,
                                         _i64p, _i64p, _u64p, _i64p]
        lib.bmvp_grow_fill.argtypes = [C.c_int64, C.c_int64, _u64p, _i64p, _i64p]
        lib.bmvp_first_touch.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p]
        for f in ("bmvp_first_touch", "bmvp_grow_count", "bmvp_grow_fill", "bmvp_hash_fill", "bmvp_blocks_of", "bmvp_owned_entries_count", "bmvp_owned_entries_fill",
                  "bmvp_first_groups_count", "bmvp_first_groups_fill"):
            getattr(lib, f).restype = C.c_int
        _lib = lib
        return lib


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _p(a: np.ndarray | None):
    if a is None:
        return None
    if a.dtype == np.uint64:
        return a.ctypes.data_as(_u64p)
    return a.ctypes.data_as(_f64p if a.dtype == np.float64 else _i64p)


def _check(rc: int, what: str) -> None:
    if rc == 3:
        raise ConsistencyError("a support entry lies outside the multivector pattern")
    if rc != 0:
        raise UsageError(f"{what} failed (status {rc})")


def hash_fill(seed: int, rows, cols, col_map=None, flat=None, scale: float = 1.0,
              out: np.ndarray | None = None) -> np.ndarray:
    """scale * hashed_entries(seed, rows, col_map[cols]), written to out[flat] (or returned)."""
    lib = load()
    rows, cols = _i64(rows), _i64(cols)
    n = rows.size
    cmap = None if col_map is None else _i64(col_map)
    fl = None if flat is None else _i64(flat)
    if out is None:
        out = np.empty(n, dtype=np.float64)
    if out.dtype != np.float64 or not out.flags.c_contiguous:
        raise UsageError("hash_fill: out must be a contiguous float64 array")
    _check(lib.bmvp_hash_fill(C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), n, _p(rows), _p(cols),
                              _p(cmap), _p(fl), float(scale), _p(out)), "bmvp_hash_fill")
    return out


def blocks_of(starts, idx):
    """(block, offset in block) of every index; starts ascending (n_blocks + 1)."""
    lib = load()
    starts, idx = _i64(starts), _i64(idx)
    block = np.empty(idx.shape, dtype=np.int64)
    offset = np.empty(idx.shape, dtype=np.int64)
    rc = lib.bmvp_blocks_of(starts.size - 1, _p(starts), idx.size, _p(idx), _p(block), _p(offset))
    if rc != 0:
        from .errors import DomainError

        raise DomainError("index outside the blocked range")
    return block, offset


def owned_entries(support, matrix):
    """Native form of ColumnSupport.owned_entries (same arrays, same order)."""
    lib = load()
    layout = matrix.layout
    lo, hi = (int(v) for v in layout.owned_rows)
    col_ptr, col_rows = support.csr()
    n_cols = support.n_cols
    counts = np.empty(n_cols, dtype=np.int64)
    _check(lib.bmvp_owned_entries_count(n_cols, _p(col_ptr), _p(col_rows), lo, hi, _p(counts)),
           "bmvp_owned_entries_count")
    start = np.zeros(n_cols + 1, dtype=np.int64)
    np.cumsum(counts, out=start[1:])
    nnz = int(start[-1])
    flat = np.empty(nnz, dtype=np.int64)
    rows = np.empty(nnz, dtype=np.int64)
    cols = np.empty(nnz, dtype=np.int64)
    if nnz == 0:
        return flat, rows, cols
    nb_own = int(layout.n_owned_blocks)
    fb = int(layout.first_block)
    bstarts = _i64(layout.blocks.starts[fb : fb + nb_own + 1])
    cbs = _i64(matrix.col_blocks.starts)
    _check(lib.bmvp_owned_entries_fill(
        n_cols, _p(col_ptr), _p(col_rows), lo, hi, _p(start), nb_own, _p(bstarts),
        int(matrix.col_blocks.n_blocks), _p(cbs), _p(_i64(matrix.row_start)),
        _p(_i64(matrix.col_index)), _p(_i64(matrix.block_offsets)), _p(_i64(matrix.col_strides)),
        _p(flat), _p(rows), _p(cols)), "bmvp_owned_entries_fill")
    return flat, rows, cols


def first_occurrence_groups(lb: np.ndarray):
    """Native form of matfree._first_occurrence_groups (same four arrays)."""
    lib = load()
    lb = _i64(lb)
    n_cells, n3 = lb.shape
    slot_group = np.empty((n_cells, n3), dtype=np.int64)
    counts = np.empty(n_cells, dtype=np.int64)
    _check(lib.bmvp_first_groups_count(n_cells, n3, _p(lb), _p(slot_group), _p(counts)),
           "bmvp_first_groups_count")
    cell_gstart = np.zeros(n_cells + 1, dtype=np.int64)
    np.cumsum(counts, out=cell_gstart[1:])
    n_groups = int(cell_gstart[-1])
    grp_cell = np.empty(n_groups, dtype=np.int64)
    grp_block = np.empty(n_groups, dtype=np.int64)
    _check(lib.bmvp_first_groups_fill(n_cells, n3, _p(lb), _p(slot_group), _p(cell_gstart),
                                      _p(grp_cell), _p(grp_block)), "bmvp_first_groups_fill")
    return slot_group, grp_cell, grp_block, cell_gstart


def grow_pattern(cell_rb: np.ndarray, n_rb: int, n_cb: int, s_row_start, s_col_index):
    """(row_start, col_index) of inc^T (inc S) + S (grow_sparsity_for_operator)."""
    lib = load()
    cell_rb = _i64(cell_rb)
    n_cells, n3 = cell_rb.shape
    words = (n_cb + 63) // 64
    bits = np.zeros(max(n_rb * words, 1), dtype=np.uint64)
    counts = np.empty(n_rb, dtype=np.int64)
    _check(lib.bmvp_grow_count(n_cells, n3, _p(cell_rb), n_rb, n_cb, _p(_i64(s_row_start)),
                               _p(_i64(s_col_index)), _p(bits), _p(counts)), "bmvp_grow_count")
    row_start = np.zeros(n_rb + 1, dtype=np.int64)
    np.cumsum(counts, out=row_start[1:])
    col_index = np.empty(int(row_start[-1]), dtype=np.int64)
    _check(lib.bmvp_grow_fill(n_rb, n_cb, _p(bits), _p(row_start), _p(col_index)),
           "bmvp_grow_fill")
    return row_start, col_index


def first_touch(n_nodes: int, touches) -> np.ndarray:
    """first[v] = first position of v in touches (touches.size if never touched)."""
    lib = load()
    touches = _i64(touches)
    first = np.empty(n_nodes, dtype=np.int64)
    _check(lib.bmvp_first_touch(n_nodes, touches.size, _p(touches), _p(first)), "bmvp_first_touch")
    return first
