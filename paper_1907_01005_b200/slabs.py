"""Slab storage of multivector values in HBM (the B200 layout behind BlockCsrMatrix).

The reference stores every stored block (block row i, column block k) as a
dense rows x stride array padded to the lane width, blocks one after the
other (`bcsr.py:233-318`).  For the sparse multivectors of this path those
blocks are 21-35 % full: inside one block row only the orbitals whose
support reaches the row's DoFs hold values.  Here each local block row i
stores ONE row-major slab

    slab_i[r][j],  r < rows_i,  j < K_i,

over its *stored columns* cols_i (ascending global column ids): all columns
of its stored blocks by default, or only the active ones when the matrix is
built from a column support (entry-level declaration, support.py) or as the
image of the operator (matfree.ImageColumns).  The stored columns of a
block row are a property of the GLOBAL block row (rank independent), so a
ghost copy of block row i has the owner's K_i and the exchange moves whole
slab rows.  Slabs are laid out in local block-row order (owned, then
ghosts), each starting on a 16-byte boundary, so

* the values of consecutive block rows are one contiguous byte range (K4 /
  K5 stage a chunk of rows with one bulk copy),
* the active columns of one DoF row are adjacent (K1 pairs of one cell read
  and reduce neighbouring doubles), and
* storage is 1.10-1.21x the structural nonzeros at the BASELINE configs
  instead of 3.5-4.8x.

Entry (local block lb, row r, global column c) lives at
    slab_off[lb] + r * K[lb] + slot(lb, c),   slot = position of c in cols_lb.
"""

from __future__ import annotations

import numpy as np

from .errors import ConsistencyError


class FullColumns:
    """Every column of every stored block (the reference's storage set)."""

    def columns_for(self, pattern, gblocks: np.ndarray):
        gblocks = np.asarray(gblocks, dtype=np.int64)
        cb = pattern.col_blocks
        cnt = pattern.row_start[gblocks + 1] - pattern.row_start[gblocks]
        owner = np.repeat(np.arange(gblocks.size, dtype=np.int64), cnt)
        first = np.concatenate([[0], np.cumsum(cnt)])[:-1]
        pos = pattern.row_start[gblocks][owner] + (np.arange(int(cnt.sum())) - first[owner])
        k = pattern.col_index[pos]
        w = cb.sizes[k]
        ptr = np.zeros(gblocks.size + 1, dtype=np.int64)
        np.add.at(ptr, owner + 1, w)
        ptr = np.cumsum(ptr)
        own2 = np.repeat(np.arange(k.size, dtype=np.int64), w)
        f2 = np.concatenate([[0], np.cumsum(w)])[:-1]
        cols = cb.starts[k][own2] + (np.arange(int(w.sum())) - f2[own2])
        return ptr, cols.astype(np.int64)

    def key(self):
        return ("full",)


FULL = FullColumns()


def _expand(counts: np.ndarray):
    counts = np.asarray(counts, dtype=np.int64)
    owner = np.repeat(np.arange(counts.size, dtype=np.int64), counts)
    start = np.concatenate([[0], np.cumsum(counts)])[:-1]
    return owner, np.arange(int(counts.sum()), dtype=np.int64) - start[owner]


class SlabGeometry:
    """Offsets of the slabs of one rank-local matrix.

    ptr / cols: stored columns per local block row (CSR over local blocks);
    rows: rows per local block row; pattern positions (row_start, col_index)
    give, per stored block, its first slot and number of stored lanes.
    """

    def __init__(self, ptr, cols, rows, row_start, col_index, col_blocks, n_owned):
        self.ptr = np.asarray(ptr, dtype=np.int64)
        self.cols = np.asarray(cols, dtype=np.int64)
        self.width = np.diff(self.ptr)
        rows = np.asarray(rows, dtype=np.int64)
        size = rows * self.width
        size = size + (size & 1)  # 16-byte aligned slabs
        self.off = np.concatenate([[0], np.cumsum(size)]).astype(np.int64)
        self.n_local = rows.size
        self.n_cols_total = int(col_blocks.total)
        self.row_of_slot = np.repeat(np.arange(self.n_local, dtype=np.int64), self.width)
        self.keys = self.row_of_slot * self.n_cols_total + self.cols
        if self.keys.size > 1 and not np.all(np.diff(self.keys) > 0):
            raise ConsistencyError("slab columns must be strictly ascending per block row")
        # stored blocks: slots [pos_slot, pos_slot + pos_nslot) of their block row
        pos_row = np.repeat(np.arange(self.n_local, dtype=np.int64), np.diff(row_start))
        k = np.asarray(col_index, dtype=np.int64)
        lo = pos_row * self.n_cols_total + col_blocks.starts[k]
        hi = pos_row * self.n_cols_total + col_blocks.starts[k + 1]
        a = np.searchsorted(self.keys, lo)
        b = np.searchsorted(self.keys, hi)
        self.pos_slot = a - self.ptr[pos_row]
        self.pos_nslot = b - a
        if int(self.pos_nslot.sum()) != self.cols.size:
            raise ConsistencyError("a stored column lies outside the stored blocks of its row")
        self.pos_full = self.pos_nslot == col_blocks.sizes[k]
        self.block_offsets = self.off[pos_row] + self.pos_slot
        self.ghost_begin = int(self.off[n_owned])

    def slots(self, lb, gcol) -> np.ndarray:
        """Slot of global column gcol in local block row lb (-1 if not stored)."""
        lb = np.asarray(lb, dtype=np.int64)
        key = lb * self.n_cols_total + np.asarray(gcol, dtype=np.int64)
        if self.keys.size == 0:
            return np.full(key.shape, -1, dtype=np.int64)
        p = np.searchsorted(self.keys, key)
        pc = np.minimum(p, self.keys.size - 1)
        ok = (p < self.keys.size) & (self.keys[pc] == key)
        return np.where(ok, p - self.ptr[lb], -1)

    def offsets(self, lb, r, gcol) -> np.ndarray:
        """Element offsets of entries (lb, r, gcol); -1 where the column is not stored."""
        lb = np.asarray(lb, dtype=np.int64)
        s = self.slots(lb, gcol)
        return np.where(s >= 0, self.off[lb] + np.asarray(r, dtype=np.int64) * self.width[lb] + s, -1)

    def row_entries(self, lb: int, rows: np.ndarray) -> np.ndarray:
        """Offsets of every stored entry of rows `rows` of block row lb, row-major."""
        k = int(self.width[lb])
        return (int(self.off[lb]) + np.asarray(rows, dtype=np.int64)[:, None] * k
                + np.arange(k, dtype=np.int64)[None, :]).ravel()

    def block_entries(self, lbs: np.ndarray, rows_per: np.ndarray):
        """(offsets, local block, row, slot) of every entry of block rows lbs
        (all their rows_per rows), block row by block row, row-major."""
        lbs = np.asarray(lbs, dtype=np.int64)
        cnt = np.asarray(rows_per, dtype=np.int64) * self.width[lbs]
        owner, t = _expand(cnt)
        lb = lbs[owner]
        k = self.width[lb]
        r = t // np.maximum(k, 1)
        s = t - r * k
        return self.off[lb] + t, lb, r, s
