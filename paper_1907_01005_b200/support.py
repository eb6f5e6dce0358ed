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

A support also decides the STORAGE of a matrix built with it
(`BlockCsrMatrix(..., columns=support)`, slabs.py): a block row stores only
the columns whose support reaches one of its rows, so entries outside the
support take no memory and no HBM traffic.  `attach_support` re-lays-out an
existing matrix the same way.

`check=True` (default) verifies the declaration on the host when the
support is attached to a filled matrix.
"""

from __future__ import annotations

import numpy as np
from scipy import sparse

from .errors import ConsistencyError


class ColumnSupport:
    """For every column (storage order), the sorted global rows it may occupy.

    Holds one sorted row array per column (shared with the per-centre
    support arrays, no copy); rank-local views only touch the columns whose
    row range intersects the rank's rows.
    """

    def __init__(self, n_rows: int, col_rows: list):
        self.n_rows = int(n_rows)
        self.col_rows = [np.asarray(r, dtype=np.int64) for r in col_rows]
        self.n_cols = len(self.col_rows)
        self._lo = np.asarray([r[0] if r.size else np.iinfo(np.int64).max for r in self.col_rows])
        self._hi = np.asarray([r[-1] if r.size else -1 for r in self.col_rows])

    @classmethod
    def from_localization(cls, loc_layout, supports, n_rows: int) -> "ColumnSupport":
        """From per-centre supports (column_supports) and the column order."""
        centre = loc_layout.centers_of_new_cols()
        return cls(n_rows, [supports[int(c)] for c in centre])

    def csr(self):
        """(col_ptr, col_rows): the columns' rows concatenated (cached; native builder input)."""
        hit = self.__dict__.get("_csr")
        if hit is None:
            ptr = np.zeros(self.n_cols + 1, dtype=np.int64)
            np.cumsum([r.size for r in self.col_rows], out=ptr[1:])
            rows = np.concatenate(self.col_rows) if self.n_cols else np.zeros(0, dtype=np.int64)
            hit = self._csr = (ptr, np.ascontiguousarray(rows, dtype=np.int64))
        return hit

    @property
    def nnz(self) -> int:
        return int(sum(r.size for r in self.col_rows))

    def columns_touching(self, lo: int, hi: int) -> np.ndarray:
        """Columns with at least one support row in [lo, hi)."""
        return np.flatnonzero((self._lo < hi) & (self._hi >= lo))

    def entries_in(self, lo: int, hi: int, extra_rows: np.ndarray | None = None):
        """(rows, cols) of support entries with rows in [lo, hi) or in extra_rows (sorted)."""
        rows, cols = [], []
        cand = set(self.columns_touching(lo, hi).tolist())
        if extra_rows is not None and extra_rows.size:
            cand |= set(np.flatnonzero((self._lo <= extra_rows[-1])
                                       & (self._hi >= extra_rows[0])).tolist())
        for c in sorted(cand):
            r = self.col_rows[c]
            a, b = np.searchsorted(r, [lo, hi])
            keep = [r[a:b]]
            if extra_rows is not None and extra_rows.size:
                pos = np.searchsorted(extra_rows, r)
                hit = (pos < extra_rows.size) & (extra_rows[np.minimum(pos, extra_rows.size - 1)] == r)
                hit[a:b] = False
                keep.append(r[hit])
            rr = np.concatenate(keep)
            rows.append(rr)
            cols.append(np.full(rr.size, c, dtype=np.int64))
        if not rows:
            z = np.zeros(0, dtype=np.int64)
            return z, z
        return np.concatenate(rows), np.concatenate(cols)

    def local_mask(self, layout) -> sparse.csr_matrix:
        """Boolean (local rows x columns) CSR; local rows = owned then ghosts."""
        key = ("mask", id(layout))
        cache = self.__dict__.setdefault("_cache", {})
        hit = cache.get(key)
        if hit is not None:
            return hit
        lo, hi = layout.owned_rows
        n_own = hi - lo
        flat = layout.ghost_rows_flat
        r, col = self.entries_in(lo, hi, flat)
        own = (r >= lo) & (r < hi)
        loc = np.empty(r.size, dtype=np.int64)
        loc[own] = r[own] - lo
        if flat.size and (~own).any():
            loc[~own] = n_own + np.searchsorted(flat, r[~own])
        n_local = n_own + flat.size
        m = sparse.csr_matrix((np.ones(r.size, dtype=np.int8), (loc, col)),
                              shape=(n_local, self.n_cols))
        m.sum_duplicates()
        m.sort_indices()
        cache[key] = m
        return m

    def columns_for(self, pattern, gblocks: np.ndarray):
        """Stored columns (slab columns, slabs.py) of global block rows `gblocks`:
        the columns whose support has a row in the block row.  (ptr, cols)."""
        from . import _plan

        blocks = pattern.row_blocks
        gblocks = np.asarray(gblocks, dtype=np.int64)
        if _plan.enabled():
            return _plan.support_columns(self, blocks, gblocks)
        sel = np.full(blocks.n_blocks, -1, dtype=np.int64)
        sel[gblocks] = np.arange(gblocks.size, dtype=np.int64)
        keys = []
        for c in range(self.n_cols):
            r = self.col_rows[c]
            if r.size == 0:
                continue
            g = np.unique(blocks.blocks_of(r))
            s_ = sel[g]
            s_ = s_[s_ >= 0]
            keys.append(s_ * self.n_cols + c)
        k = np.sort(np.concatenate(keys)) if keys else np.zeros(0, dtype=np.int64)
        ptr = np.searchsorted(k // max(self.n_cols, 1) if k.size else k,
                              np.arange(gblocks.size + 1), side="left").astype(np.int64)
        return ptr, (k % max(self.n_cols, 1)).astype(np.int64)

    def key(self):
        return ("support", id(self))

    def owned_entries(self, matrix):
        """(flat storage offsets, global rows, columns) of the support entries
        in the matrix's owned rows, column-major (column, then row) order.

        This is the compact value order used by `upload_support_values`.
        Cached per matrix geometry.
        """
        key = ("owned", id(matrix.slab))
        cache = self.__dict__.setdefault("_cache", {})
        hit = cache.get(key)
        if hit is not None and hit[0] is matrix.slab:
            return hit[1]
        from . import _plan

        out = _plan.owned_entries(self, matrix) if _plan.enabled() \
            else self._owned_entries_numpy(matrix)
        cache[key] = (matrix.slab, out)
        return out

    def _owned_entries_numpy(self, matrix):
        """numpy restatement of owned_entries (the native builder is pinned to it)."""
        layout = matrix.layout
        lo, hi = layout.owned_rows
        rows, cols = self.entries_in(lo, hi)
        if rows.size == 0:
            return rows, rows, cols
        blocks = layout.blocks
        nb_own = layout.n_owned_blocks
        own_sizes = blocks.sizes[layout.first_block : layout.first_block + nb_own]
        lb = np.repeat(np.arange(nb_own, dtype=np.int64), own_sizes)[rows - lo]
        rib = rows - blocks.starts[layout.first_block + lb]
        flat = matrix.slab.offsets(lb, rib, cols)
        if (flat < 0).any():
            raise ConsistencyError("a support entry lies outside the multivector pattern")
        return flat, rows, cols

    def check_matrix(self, matrix) -> None:
        """Raise ConsistencyError if an owned entry outside the support is nonzero."""
        flat, grow, gcol = matrix._valid_owned_index()
        if flat.size == 0:
            return
        vals = matrix.data.detach().cpu().numpy()[flat]
        nz = vals != 0.0
        if not nz.any():
            return
        grow, gcol = grow[nz], gcol[nz]
        lo, hi = matrix.layout.owned_rows
        r, c = self.entries_in(lo, hi)
        skey = np.sort(c * self.n_rows + r)
        key = gcol * self.n_rows + grow
        pos = np.searchsorted(skey, key)
        inside = (pos < skey.size) & (skey[np.minimum(pos, max(skey.size - 1, 0))] == key)
        if not inside.all():
            i = int(np.flatnonzero(~inside)[0])
            raise ConsistencyError(
                f"entry ({int(grow[i])}, {int(gcol[i])}) is nonzero but outside the declared "
                f"column support (owned rows {(lo, hi)})")


def attach_support(matrix, support: ColumnSupport, check: bool = True):
    """Declare matrix entries outside `support` structural zeros.

    If the matrix does not already store exactly the support's columns, it is
    re-laid-out (slabs.py): values inside the new slabs are kept, entries
    outside the support are dropped (check=True first verifies they are 0)."""
    if support.n_cols != matrix.col_blocks.total:
        raise ConsistencyError("support column count differs from the matrix")
    if check:
        support.check_matrix(matrix)
    matrix.relayout(support)
    return matrix
