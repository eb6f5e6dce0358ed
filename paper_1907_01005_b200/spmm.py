"""Plans of the K4 / K5 kernels (csrc/bmv_spmm.cu) on slab storage.

The reference multiplies stored block pairs in Python loops: tmmult
(`bcsr.py:631-667`, S_kl += A_ik^T B_il over the owned block rows i) and
mmult (`bcsr.py:587-628`, Y_ij += A_ik C_kj kept where Y stores (i, j)).
Here the owned rows of A are cut into CHUNKS of consecutive rows (the native
planner bmvp_chunk_plan, include/bmv_plan.h); a chunk is one contiguous
range of A's (and, for K4, B's) slab values, multiplied densely over the
union of its rows' stored columns on the FP64 tensor cores.  Plans are
cached on the first operand, keyed by the operands' slab geometries (kept
alive by the cache entry, so a recycled id() cannot alias), with a bounded
number of entries.
"""

from __future__ import annotations

import os
from collections import OrderedDict

import numpy as np
import torch

from . import _lib, _plan
from .errors import PatternError, ShapeError

# chunk shape: the kernels (bmv_spmm.cu) give every warp private buffers of
# bmv_chunk_kernel_config() bytes, the largest chunk [meta | A | B];
# BMV_SPMM_STAGE / BMV_SPMM_DATA / BMV_SPMM_ROWS override for tuning runs
K4_MAX_ROWS = K5_MAX_ROWS = int(os.environ.get("BMV_SPMM_ROWS", 256))
MAX_BLOCK_ROWS = 16
META_ALLOWANCE = 1536        # bytes left for the chunk meta when cutting chunks


SHORT_ROWS = 32              # mean rows per block row below which K4 takes its second shape


def chunk_bytes(kind: int, variant: int = 0) -> tuple[int, int]:
    """(largest chunk, staged values per chunk) in bytes for K4 / K5 (kind 4 / 5);
    variant 1: the kernel shape for short block rows (larger chunks)."""
    if "BMV_SPMM_STAGE" in os.environ:
        stage = int(os.environ["BMV_SPMM_STAGE"])
    else:
        C = _lib.C
        warps, buf = C.c_int32(), C.c_int32()
        _lib.check(_lib.load().bmv_chunk_kernel_config(int(kind), int(variant), C.byref(warps),
                                                       C.byref(buf)))
        stage = int(buf.value)
    data = int(os.environ.get("BMV_SPMM_DATA", max(stage - META_ALLOWANCE, stage // 2)))
    return stage, data


_CACHE_ENTRIES = 8


class ChunkPlan:
    def __init__(self, arrays: dict, flops: int, zero_begin: int = 0):
        self.arrays = arrays
        self.flops = flops
        self.zero_begin = zero_begin
        self.n_chunks = int(arrays["n_chunks"])
        self.dmma = int(arrays["dmma"])
        lib = _lib.load()
        d = _lib.ChunkDesc()
        d.kind = int(arrays["kind"])
        d.n_parts = int(arrays["n_parts"])
        d.stage_bytes = int(arrays["stage_bytes"])
        d.n_chunks = self.n_chunks
        d.meta_len = int(arrays["meta_len"])
        C = _lib.C
        d.part_chunk_start = _lib.ptr(arrays["part_chunk_start"], C.c_int64)
        d.chunk_meta = _lib.ptr(arrays["chunk_meta"], C.c_int64)
        d.meta = _lib.ptr(arrays["meta"], C.c_int32)
        d.chunk_a = _lib.ptr(arrays["chunk_a"], C.c_int64)
        d.chunk_b = _lib.ptr(arrays["chunk_b"], C.c_int64) if arrays["chunk_b"] is not None \
            else C.cast(None, C.POINTER(C.c_int64))
        raw = C.c_void_p()
        _lib.check(lib.bmv_chunk_plan_create(C.byref(d), C.byref(raw)), "bmv_chunk_plan_create")
        self.handle = _lib.Handle("bmv_chunk_plan_destroy", raw)


def _n_parts(device) -> int:
    if device is not None and torch.device(device).type == "cuda" and torch.cuda.is_available():
        return int(torch.cuda.get_device_properties(torch.device(device)).multi_processor_count)
    return 148


def _cache_get(a, key, refs):
    cache = a.__dict__.setdefault("_spmm_plans", OrderedDict())
    hit = cache.get(key)
    if hit is not None and all(x is y for x, y in zip(hit[1], refs)):
        cache.move_to_end(key)
        return hit[0]
    return None


def _cache_put(a, key, refs, plan):
    cache = a.__dict__.setdefault("_spmm_plans", OrderedDict())
    cache[key] = (plan, refs)
    while len(cache) > _CACHE_ENTRIES:
        cache.popitem(last=False)


class _Owned:
    """Slab geometry restricted to the owned block rows (planner input)."""

    def __init__(self, m):
        n = m.n_owned_blocks
        sg = m.slab
        self.ptr = sg.ptr[: n + 1]
        self.cols = sg.cols[: int(sg.ptr[n])]
        self.off = sg.off[: n + 1]


def _local_table(layout, n_global: int) -> np.ndarray:
    tab = np.full(n_global, -1, dtype=np.int64)
    gl = layout.global_blocks_of_locals()
    tab[gl] = np.arange(gl.size, dtype=np.int64)
    return tab


def _check_tmmult_blocks(a, b, c):
    """PatternError when c lacks a block (k, l) with a_ik and b_il stored in
    one owned block row i (the reference's check, bcsr.py:653-659)."""
    from scipy import sparse

    n = a.n_owned_blocks
    na = int(a.row_start[n])
    nb = int(b.row_start[n])
    pa = sparse.csr_matrix((np.ones(na, dtype=np.int32), a.col_index[:na], a.row_start[: n + 1]),
                           shape=(n, a.col_blocks.n_blocks))
    pb = sparse.csr_matrix((np.ones(nb, dtype=np.int32), b.col_index[:nb], b.row_start[: n + 1]),
                           shape=(n, b.col_blocks.n_blocks))
    need = (pa.T @ pb).tocoo()
    if need.nnz == 0:
        return
    ltab = _local_table(c.layout, c.layout.blocks.n_blocks)
    lk = ltab[need.row]
    if (lk < 0).any():
        raise PatternError(f"rank {c.layout.rank} holds no row of S for column block "
                           f"{int(need.row[lk < 0][0])}")
    keys = c.local_keys()
    k = lk * c.col_blocks.n_blocks + need.col
    p = np.searchsorted(keys, k)
    ok = (p < keys.size) & (keys[np.minimum(p, max(keys.size - 1, 0))] == k)
    if not ok.all():
        i = int(np.flatnonzero(~ok)[0])
        raise PatternError(f"tmmult destination misses block ({int(need.row[i])}, {int(need.col[i])})")


def tmmult_plan(a, b, c) -> ChunkPlan:
    """K4 plan of c = a^T b (c: rows = a's columns, columns = b's columns)."""
    refs = (a.slab, b.slab, c.slab)
    key = ("tm", id(b.slab), id(c.slab))
    plan = _cache_get(a, key, refs)
    if plan is not None:
        return plan
    _check_tmmult_blocks(a, b, c)
    n = a.n_owned_blocks
    rows = a.local_row_sizes[:n]
    # short block rows: the S flush per chunk weighs as much as the product;
    # the second kernel shape has fewer warps and larger chunks
    variant = 1 if n and float(np.mean(rows)) < SHORT_ROWS else 0
    stage, data = chunk_bytes(4, variant)
    arrays = _plan.chunk_plan(
        4, a.local_row_sizes[:n], _Owned(a), _Owned(b), a.col_blocks.starts,
        _local_table(c.layout, c.layout.blocks.n_blocks), c.slab,
        K4_MAX_ROWS, MAX_BLOCK_ROWS, data, stage, _n_parts(c.device))
    flops = int(2 * np.sum(rows * a.slab.width[:n] * b.slab.width[:n]))
    plan = ChunkPlan(arrays, flops)
    _cache_put(a, key, refs, plan)
    return plan


def mmult_plan(a, b, c) -> ChunkPlan:
    """K5 plan of c = alpha a b (b: rows = a's columns; c: a's rows, b's columns)."""
    refs = (a.slab, b.slab, c.slab)
    key = ("mm", id(b.slab), id(c.slab))
    plan = _cache_get(a, key, refs)
    if plan is not None:
        return plan
    n = a.n_owned_blocks
    # every column block of a needs a complete row block of b (ghosted if remote)
    na = int(a.row_start[n])
    kcols = np.unique(a.col_index[:na])
    btab = _local_table(b.layout, b.layout.blocks.n_blocks)
    kb = btab[kcols]
    if (kb < 0).any():
        raise PatternError(f"rank {b.layout.rank} holds no ghost of block row {int(kcols[kb < 0][0])}")
    if (b.local_row_sizes[kb] != a.col_blocks.sizes[kcols]).any():
        bad = int(kcols[b.local_row_sizes[kb] != a.col_blocks.sizes[kcols]][0])
        raise ShapeError(f"row block {bad} of b is incomplete (split ghost group)")
    arrays = _plan.chunk_plan(
        5, a.local_row_sizes[:n], _Owned(a), _Owned(c), a.col_blocks.starts, btab, b.slab,
        K5_MAX_ROWS, MAX_BLOCK_ROWS, chunk_bytes(5)[1], chunk_bytes(5)[0], _n_parts(c.device))
    rows = a.local_row_sizes[:n]
    flops = int(2 * np.sum(rows * a.slab.width[:n] * c.slab.width[:n]))
    plan = ChunkPlan(arrays, flops, zero_begin=c._ghost_data_begin)
    _cache_put(a, key, refs, plan)
    return plan
