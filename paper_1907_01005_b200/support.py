"""Entry-level column supports of a sparse multivector.

The reference stores X as dense padded blocks (`bcsr.py:233-318`) and its
cell loop computes all W lanes of every visited column block, including
the lanes whose orbital has no support on the cell (`matfree.py:500-513`;
SURVEY section 3.1: 3.4x extra work at the Q2 config).  The a-priori
support of every column is known from the localisation patches
(`localization.py:184-204`).  Attaching it to a matrix declares that its
entries outside the support are structural zeros; the B200 operator then
runs only the active (cell, column) pairs.  Skipping a pair whose input is
identically zero on the cell changes no output value, so results are the
same as the all-lanes computation whenever the declaration holds.

`check=True` (default) verifies the declaration on the host when the
support is attached to a filled matrix.
"""

from __future__ import annotations

import numpy as np
from scipy import sparse

from .errors import ConsistencyError


class ColumnSupport:
    """For every column (storage order), the sorted global rows it may occupy."""

    def __init__(self, n_rows: int, col_ptr: np.ndarray, rows: np.ndarray):
        self.n_rows = int(n_rows)
        self.col_ptr = np.asarray(col_ptr, dtype=np.int64)
        self.rows = np.asarray(rows, dtype=np.int64)
        self.n_cols = self.col_ptr.size - 1

    @classmethod
    def from_localization(cls, loc_layout, supports, n_rows: int) -> "ColumnSupport":
        """From per-centre supports (column_supports) and the column order."""
        centre = loc_layout.centers_of_new_cols()
        parts = [np.asarray(supports[int(c)], dtype=np.int64) for c in centre]
        counts = np.asarray([p.size for p in parts], dtype=np.int64)
        ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        rows = np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)
        return cls(n_rows, ptr, rows)

    @property
    def nnz(self) -> int:
        return int(self.rows.size)

    def local_mask(self, layout) -> sparse.csr_matrix:
        """Boolean (local rows x columns) CSR; local rows = owned then ghosts."""
        key = ("mask", id(layout))
        cache = self.__dict__.setdefault("_cache", {})
        hit = cache.get(key)
        if hit is not None:
            return hit
        lo, hi = layout.owned_rows
        n_own = hi - lo
        col = np.repeat(np.arange(self.n_cols, dtype=np.int64), np.diff(self.col_ptr))
        r = self.rows
        own = (r >= lo) & (r < hi)
        loc = np.full(r.size, -1, dtype=np.int64)
        loc[own] = r[own] - lo
        flat = layout.ghost_rows_flat
        if flat.size:
            rest = ~own
            pos = np.searchsorted(flat, r[rest])
            hit_g = (pos < flat.size) & (flat[np.minimum(pos, flat.size - 1)] == r[rest])
            tmp = np.full(pos.size, -1, dtype=np.int64)
            tmp[hit_g] = n_own + pos[hit_g]
            loc[rest] = tmp
        keep = loc >= 0
        n_local = n_own + flat.size
        m = sparse.csr_matrix((np.ones(int(keep.sum()), dtype=np.int8), (loc[keep], col[keep])),
                              shape=(n_local, self.n_cols))
        m.sum_duplicates()
        m.sort_indices()
        cache[key] = m
        return m

    def owned_entries(self, matrix):
        """(flat storage offsets, global rows, columns) of the support entries
        in the matrix's owned rows, column-major (column, then row) order.

        This is the compact value order used by `upload_support_values`.
        Cached per (pattern, layout, lane width).
        """
        key = ("owned", id(matrix.pattern), id(matrix.layout), matrix.lane_width)
        cache = self.__dict__.setdefault("_cache", {})
        hit = cache.get(key)
        if hit is not None:
            return hit
        layout = matrix.layout
        lo, hi = layout.owned_rows
        cols = np.repeat(np.arange(self.n_cols, dtype=np.int64), np.diff(self.col_ptr))
        rows = self.rows
        keep = (rows >= lo) & (rows < hi)
        rows, cols = rows[keep], cols[keep]
        if rows.size == 0:
            hit = (rows, rows, cols)
            cache[key] = hit
            return hit
        blocks = layout.blocks
        nb_own = layout.n_owned_blocks
        own_sizes = blocks.sizes[layout.first_block : layout.first_block + nb_own]
        lb = np.repeat(np.arange(nb_own, dtype=np.int64), own_sizes)[rows - lo]
        rib = rows - blocks.starts[layout.first_block + lb]
        cbk = np.repeat(np.arange(matrix.col_blocks.n_blocks, dtype=np.int64),
                        matrix.col_blocks.sizes)[cols]
        n_cb = matrix.col_blocks.n_blocks
        n_own_pos = int(matrix.row_start[nb_own])
        if nb_own * n_cb <= 64_000_000:
            table = np.full(nb_own * n_cb, -1, dtype=np.int64)
            table[matrix.pos_row[:n_own_pos] * n_cb + matrix.col_index[:n_own_pos]] = \
                np.arange(n_own_pos, dtype=np.int64)
            pos = table[lb * n_cb + cbk]
        else:
            keys = matrix.local_keys()[:n_own_pos]
            k = lb * n_cb + cbk
            pos = np.searchsorted(keys, k)
            pos = np.where((pos < keys.size) & (keys[np.minimum(pos, keys.size - 1)] == k), pos, -1)
        if (pos < 0).any():
            raise ConsistencyError("a support entry lies outside the multivector pattern")
        flat = (matrix.block_offsets[pos] + rib * matrix.col_strides[cbk]
                + (cols - matrix.col_blocks.starts[cbk]))
        hit = (flat, rows, cols)
        cache[key] = hit
        return hit

    def check_matrix(self, matrix) -> None:
        """Raise ConsistencyError if an owned entry outside the support is nonzero."""
        dense_rows = matrix.layout.owned_rows
        flat, grow, gcol = matrix._valid_owned_index()
        if flat.size == 0:
            return
        vals = matrix.data.detach().cpu().numpy()[flat]
        nz = vals != 0.0
        if not nz.any():
            return
        grow, gcol = grow[nz], gcol[nz]
        key = gcol * self.n_rows + grow
        col = np.repeat(np.arange(self.n_cols, dtype=np.int64), np.diff(self.col_ptr))
        skey = np.sort(col * self.n_rows + self.rows)
        pos = np.searchsorted(skey, key)
        inside = (pos < skey.size) & (skey[np.minimum(pos, max(skey.size - 1, 0))] == key)
        if not inside.all():
            i = int(np.flatnonzero(~inside)[0])
            raise ConsistencyError(
                f"entry ({int(grow[i])}, {int(gcol[i])}) is nonzero but outside the declared "
                f"column support (owned rows {dense_rows})")


def attach_support(matrix, support: ColumnSupport, check: bool = True):
    """Declare matrix entries outside `support` structural zeros."""
    if support.n_cols != matrix.col_blocks.total:
        raise ConsistencyError("support column count differs from the matrix")
    if check:
        support.check_matrix(matrix)
    matrix.support = support
    return matrix
