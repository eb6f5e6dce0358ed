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
                                                _i64p, C.c_int64, _i64p, _i64p, _i64p, _i64p,
                                                _i64p, _i64p, _i64p]
        lib.bmvp_support_columns_count.argtypes = [C.c_int64, _i64p, _i64p, C.c_int64, _i64p,
                                                   _i64p, C.c_int64, _i64p]
        lib.bmvp_support_columns_fill.argtypes = [C.c_int64, _i64p, _i64p, C.c_int64, _i64p,
                                                  _i64p, C.c_int64, _i64p, _i64p, _i64p]
        lib.bmvp_first_groups_count.argtypes = [C.c_int64, C.c_int32, _i64p, _i64p, _i64p]
        lib.bmvp_first_groups_fill.argtypes = [C.c_int64, C.c_int32, _i64p, _i64p, _i64p, _i64p,
                                               _i64p]
        lib.bmvp_grow_count.argtypes = [C.c_int64, C.c_int32, _i64p, C.c_int64, C.c_int64,
                                         _i64p, _i64p, _u64p, _i64p]
        lib.bmvp_grow_fill.argtypes = [C.c_int64, C.c_int64, _u64p, _i64p, _i64p]
        lib.bmvp_first_touch.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p]
        lib.bmvp_chunk_plan.restype = C.c_void_p
        lib.bmvp_chunk_plan.argtypes = [C.c_int32, C.c_int64, _i64p, _i64p, _i64p, _i64p, _i64p,
                                        _i64p, _i64p, C.c_int64, _i64p, _i64p, _i64p, _i64p,
                                        _i64p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32]
        lib.bmvp_chunk_status.argtypes = [C.c_void_p]
        lib.bmvp_chunk_status.restype = C.c_int
        lib.bmvp_chunk_sizes.argtypes = [C.c_void_p, _i64p, _i64p, _i64p]
        lib.bmvp_chunk_sizes.restype = None
        lib.bmvp_chunk_copy.argtypes = [C.c_void_p, _i64p, _i64p, C.POINTER(C.c_int32), _i64p,
                                        _i64p]
        lib.bmvp_chunk_copy.restype = None
        lib.bmvp_chunk_free.argtypes = [C.c_void_p]
        lib.bmvp_chunk_free.restype = None
        _i32p = C.POINTER(C.c_int32)
        lib.bmvp_support_transpose.argtypes = [C.c_int64, _i64p, _i64p, _i64p, C.c_int64, _i64p,
                                               _i32p]
        lib.bmvp_cell_pairs.argtypes = [C.c_int64, C.c_int32, _i64p, _i64p, _i32p, _i64p, _i32p]
        lib.bmvp_block_image.argtypes = [C.c_int64, C.c_int32, _i64p, _i64p, _i32p, C.c_int64,
                                         C.c_int64, _i64p, _i64p]
        lib.bmvp_k1_plan.argtypes = [C.c_int64, _i64p, _i64p, _i64p, _i64p, _i64p, _i64p, _i64p,
                                     _i64p, _i64p, _i64p, _i64p, _i32p, _i64p]
        for f in ("bmvp_support_transpose", "bmvp_cell_pairs", "bmvp_block_image", "bmvp_k1_plan"):
            getattr(lib, f).restype = C.c_int
        for f in ("bmvp_first_touch", "bmvp_grow_count", "bmvp_grow_fill", "bmvp_hash_fill", "bmvp_blocks_of", "bmvp_owned_entries_count", "bmvp_owned_entries_fill",
                  "bmvp_support_columns_count", "bmvp_support_columns_fill",
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
    sg = matrix.slab
    _check(lib.bmvp_owned_entries_fill(
        n_cols, _p(col_ptr), _p(col_rows), lo, hi, _p(start), nb_own, _p(bstarts),
        _p(_i64(sg.ptr)), _p(_i64(sg.cols)), _p(_i64(sg.off)), _p(flat), _p(rows), _p(cols)),
        "bmvp_owned_entries_fill")
    return flat, rows, cols


def support_columns(support, blocks, gblocks):
    """Native form of ColumnSupport.columns_for: (ptr, cols) over gblocks."""
    lib = load()
    col_ptr, col_rows = support.csr()
    gblocks = _i64(gblocks)
    n_blocks = int(blocks.n_blocks)
    sel = np.full(n_blocks, -1, dtype=np.int64)
    sel[gblocks] = np.arange(gblocks.size, dtype=np.int64)
    counts = np.empty(gblocks.size, dtype=np.int64)
    starts = _i64(blocks.starts)
    _check(lib.bmvp_support_columns_count(support.n_cols, _p(col_ptr), _p(col_rows), n_blocks,
                                          _p(starts), _p(sel), gblocks.size, _p(counts)),
           "bmvp_support_columns_count")
    ptr = np.zeros(gblocks.size + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    cols = np.empty(int(ptr[-1]), dtype=np.int64)
    cursor = np.empty(max(gblocks.size, 1), dtype=np.int64)
    _check(lib.bmvp_support_columns_fill(support.n_cols, _p(col_ptr), _p(col_rows), n_blocks,
                                         _p(starts), _p(sel), gblocks.size, _p(ptr), _p(cursor),
                                         _p(cols)), "bmvp_support_columns_fill")
    return ptr, cols


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


def chunk_plan(kind: int, rows, a, b, acb_starts, m_ltab, m, max_rows: int, max_brows: int,
               data_bytes: int, stage_bytes: int, n_parts: int) -> dict:
    """K4 / K5 chunk plan (bmv.h bmv_chunk_desc) from slab geometries a, b, m
    (objects with ptr / cols / off arrays).  Returns the descriptor arrays;
    raises PatternError (M lacks a block row), ShapeError (a row exceeds a
    stage, offsets beyond 2^31)."""
    from .errors import PatternError, ShapeError

    lib = load()
    keep = [_i64(x) for x in (rows, a.ptr, a.cols, a.off, b.ptr, b.cols, b.off, acb_starts,
                               m_ltab, m.ptr, m.cols, m.off)]
    h = lib.bmvp_chunk_plan(int(kind), keep[0].size, *[_p(x) for x in keep[:7]],
                            keep[7].size - 1, *[_p(x) for x in keep[7:]], int(max_rows),
                            int(max_brows), int(data_bytes), int(stage_bytes), int(n_parts))
    try:
        st = lib.bmvp_chunk_status(h)
        if st == 3:
            raise PatternError("the product matrix holds no block row for a column block of A")
        if st == 4:
            raise ShapeError("a single row of the product does not fit a K4/K5 stage")
        if st == 5:
            raise ShapeError("K4/K5 offsets exceed 2^31 elements")
        if st != 0:
            raise UsageError(f"bmvp_chunk_plan failed (status {st})")
        n = C.c_int64()
        ml = C.c_int64()
        dm = C.c_int64()
        lib.bmvp_chunk_sizes(h, C.byref(n), C.byref(ml), C.byref(dm))
        n_chunks, meta_len = n.value, ml.value
        out = {
            "part_chunk_start": np.empty(n_parts + 1, dtype=np.int64),
            "chunk_meta": np.empty(n_chunks + 1, dtype=np.int64),
            "meta": np.empty(max(meta_len, 1), dtype=np.int32),
            "chunk_a": np.empty(max(2 * n_chunks, 1), dtype=np.int64),
            "chunk_b": np.empty(max(2 * n_chunks, 1), dtype=np.int64) if kind == 4 else None,
        }
        lib.bmvp_chunk_copy(h, _p(out["part_chunk_start"]), _p(out["chunk_meta"]),
                            out["meta"].ctypes.data_as(C.POINTER(C.c_int32)), _p(out["chunk_a"]),
                            _p(out["chunk_b"]) if kind == 4 else None)
        out.update(kind=kind, n_chunks=n_chunks, meta_len=meta_len, dmma=dm.value,
                   n_parts=n_parts, stage_bytes=stage_bytes)
        return out
    finally:
        lib.bmvp_chunk_free(h)


def _p32(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def support_transpose(support, row_sel: np.ndarray, n_sel: int):
    """Row -> columns CSR of a ColumnSupport over the selected rows
    (row_sel: global row -> selected index or -1); columns ascending."""
    lib = load()
    col_ptr, col_rows = support.csr()
    row_sel = _i64(row_sel)
    ptr = np.zeros(n_sel + 1, dtype=np.int64)
    _check(lib.bmvp_support_transpose(support.n_cols, _p(col_ptr), _p(col_rows), _p(row_sel),
                                      n_sel, _p(ptr), None), "bmvp_support_transpose")
    cols = np.empty(max(int(ptr[-1]), 1), dtype=np.int32)
    _check(lib.bmvp_support_transpose(support.n_cols, _p(col_ptr), _p(col_rows), _p(row_sel),
                                      n_sel, _p(ptr), _p32(cols)), "bmvp_support_transpose")
    return ptr, cols[: int(ptr[-1])]


def cell_pairs(cell_rows: np.ndarray, row_ptr: np.ndarray, row_cols: np.ndarray):
    """Per cell the sorted union of the columns of its rows (cell_rows (n, n3)
    indices into the row CSR, -1 = none).  (ptr, cols int32)."""
    lib = load()
    cell_rows = _i64(cell_rows)
    n, n3 = cell_rows.shape
    ptr = np.zeros(n + 1, dtype=np.int64)
    row_ptr = _i64(row_ptr)
    row_cols = np.ascontiguousarray(row_cols, dtype=np.int32)
    rc = row_cols if row_cols.size else np.zeros(1, dtype=np.int32)
    _check(lib.bmvp_cell_pairs(n, n3, _p(cell_rows), _p(row_ptr), _p32(rc), _p(ptr), None),
           "bmvp_cell_pairs")
    cols = np.empty(max(int(ptr[-1]), 1), dtype=np.int32)
    _check(lib.bmvp_cell_pairs(n, n3, _p(cell_rows), _p(row_ptr), _p32(rc), _p(ptr), _p32(cols)),
           "bmvp_cell_pairs")
    return ptr, cols[: int(ptr[-1])]


def block_image(cell_blocks: np.ndarray, pair_ptr, pair_cols, n_blocks: int, n_cols: int):
    """image(b) = union of the cells' pair columns over the cells touching b
    (cell_blocks (n, n3): selected block index or -1).  (ptr, cols int64)."""
    lib = load()
    cell_blocks = _i64(cell_blocks)
    n, n3 = cell_blocks.shape
    pair_ptr = _i64(pair_ptr)
    pc = np.ascontiguousarray(pair_cols, dtype=np.int32)
    pc = pc if pc.size else np.zeros(1, dtype=np.int32)
    ptr = np.zeros(n_blocks + 1, dtype=np.int64)
    _check(lib.bmvp_block_image(n, n3, _p(cell_blocks), _p(pair_ptr), _p32(pc), n_blocks, n_cols,
                                _p(ptr), None), "bmvp_block_image")
    cols = np.empty(max(int(ptr[-1]), 1), dtype=np.int64)
    _check(lib.bmvp_block_image(n, n3, _p(cell_blocks), _p(pair_ptr), _p32(pc), n_blocks, n_cols,
                                _p(ptr), _p(cols)), "bmvp_block_image")
    return ptr, cols[: int(ptr[-1])]


def k1_gtab(pair_cell, pair_col, cell_gstart, grp_block, src, dst, pair_gtab, gtab_len: int):
    """K1 group tables (see bmv_plan.h bmvp_k1_plan); returns (gtab, bad pair or -1)."""
    lib = load()
    gtab = np.empty(max(gtab_len, 2), dtype=np.int32)
    bad = C.c_int64(-1)
    keep = [_i64(a) for a in (pair_cell, pair_col, cell_gstart, grp_block, src.ptr, src.cols,
                               src.off, dst.ptr, dst.cols, dst.off, pair_gtab)]
    rc = lib.bmvp_k1_plan(keep[0].size, *[_p(a) for a in keep], _p32(gtab), C.byref(bad))
    if rc not in (0, 3):
        raise UsageError(f"bmvp_k1_plan failed (status {rc})")
    return gtab[:gtab_len], int(bad.value)
