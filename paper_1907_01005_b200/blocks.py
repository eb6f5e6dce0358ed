"""Blockings of index ranges and block-level sparsity patterns (host side).

Same public surface as the reference (`bcsrmv/blocks.py:10-157`): a
`BlockIndices` partition of [0, total) and a CSR-indexed
`BlockSparsityPattern` whose per-row column ids are strictly ascending, so
the CSR position of a block is its linear storage index.  Construction is
vectorised (no per-row Python loop when built from CSR arrays) because the
weak-scaling patterns have millions of block rows.
"""

from __future__ import annotations

import numpy as np

from .errors import ConfigurationError, DomainError, PatternError


class BlockIndices:
    """Contiguous blocks of positive size covering [0, total)."""

    def __init__(self, sizes):
        sizes = np.asarray(sizes, dtype=np.int64)
        if sizes.ndim != 1:
            raise ConfigurationError("block sizes must be a 1-d sequence")
        if sizes.size and int(sizes.min()) <= 0:
            raise ConfigurationError("block sizes must be positive")
        self.sizes = sizes
        self.starts = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)

    @property
    def n_blocks(self) -> int:
        return int(self.sizes.size)

    @property
    def total(self) -> int:
        return int(self.starts[-1])

    def block_start(self, b: int) -> int:
        return int(self.starts[b])

    def block_size(self, b: int) -> int:
        return int(self.sizes[b])

    def global_to_block(self, i: int) -> tuple[int, int]:
        if i < 0 or i >= self.total:
            raise DomainError(f"index {i} outside [0, {self.total})")
        b = int(np.searchsorted(self.starts, i, side="right")) - 1
        return b, i - int(self.starts[b])

    def blocks_of(self, indices) -> np.ndarray:
        idx = np.asarray(indices, dtype=np.int64)
        if idx.size and (int(idx.min()) < 0 or int(idx.max()) >= self.total):
            raise DomainError("index outside the blocked range")
        return np.searchsorted(self.starts, idx, side="right") - 1

    def __eq__(self, other) -> bool:
        if self is other:
            return True
        return isinstance(other, BlockIndices) and np.array_equal(self.sizes, other.sizes)

    def __hash__(self):
        return hash((self.sizes.size, self.total))

    def __repr__(self) -> str:
        return f"BlockIndices(n_blocks={self.n_blocks}, total={self.total})"


class BlockSparsityPattern:
    """Block pattern over independent row/column blockings (CSR, sorted)."""

    def __init__(self, row_blocks: BlockIndices, col_blocks: BlockIndices, rows):
        rows = list(rows)
        if len(rows) != row_blocks.n_blocks:
            raise PatternError("one column list required per block row")
        counts = np.fromiter((len(r) for r in rows), dtype=np.int64, count=len(rows))
        cols = (
            np.concatenate([np.asarray(r, dtype=np.int64).ravel() for r in rows])
            if rows
            else np.zeros(0, dtype=np.int64)
        )
        row_start = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        self._init_csr(row_blocks, col_blocks, row_start, cols.astype(np.int64))

    @classmethod
    def from_csr(cls, row_blocks, col_blocks, row_start, col_index):
        """Build from CSR arrays directly (validated, vectorised)."""
        obj = cls.__new__(cls)
        obj._init_csr(
            row_blocks,
            col_blocks,
            np.asarray(row_start, dtype=np.int64),
            np.asarray(col_index, dtype=np.int64),
        )
        return obj

    def _init_csr(self, row_blocks, col_blocks, row_start, col_index):
        n = row_blocks.n_blocks
        if row_start.size != n + 1 or row_start[0] != 0 or row_start[-1] != col_index.size:
            raise PatternError("one column list required per block row")
        if col_index.size:
            if int(col_index.min()) < 0 or int(col_index.max()) >= col_blocks.n_blocks:
                bad = int(np.flatnonzero((col_index < 0) | (col_index >= col_blocks.n_blocks))[0])
                r = int(np.searchsorted(row_start, bad, side="right")) - 1
                raise PatternError(f"column id out of range in block row {r}")
            d = np.diff(col_index)
            same_row = np.ones(col_index.size - 1, dtype=bool)
            starts = row_start[1:-1]
            starts = starts[(starts > 0) & (starts < col_index.size)]
            same_row[starts - 1] = False
            bad = np.flatnonzero(same_row & (d <= 0))
            if bad.size:
                r = int(np.searchsorted(row_start, int(bad[0]) + 1, side="right")) - 1
                raise PatternError(f"column ids of block row {r} not ascending")
        self.row_blocks = row_blocks
        self.col_blocks = col_blocks
        self.row_start = row_start
        self.col_index = col_index

    @property
    def n_stored_blocks(self) -> int:
        return int(self.col_index.size)

    def row_cols(self, r: int) -> np.ndarray:
        return self.col_index[self.row_start[r] : self.row_start[r + 1]]

    def block_pos(self, r: int, c: int) -> int:
        lo, hi = int(self.row_start[r]), int(self.row_start[r + 1])
        k = lo + int(np.searchsorted(self.col_index[lo:hi], c))
        if k < hi and self.col_index[k] == c:
            return k
        return -1

    def has(self, r: int, c: int) -> bool:
        return self.block_pos(r, c) >= 0

    def block_rows(self) -> np.ndarray:
        """Block-row id of every stored block (CSR expansion)."""
        return np.repeat(
            np.arange(self.row_blocks.n_blocks, dtype=np.int64), np.diff(self.row_start)
        )

    def keys(self) -> np.ndarray:
        """Sorted int64 keys row * n_col_blocks + col of the stored blocks."""
        return self.block_rows() * self.col_blocks.n_blocks + self.col_index

    def to_bool_csr(self):
        from scipy import sparse

        return sparse.csr_matrix(
            (np.ones(self.col_index.size, dtype=bool), self.col_index.copy(), self.row_start.copy()),
            shape=(self.row_blocks.n_blocks, self.col_blocks.n_blocks),
        )

    @classmethod
    def from_bool_csr(cls, mat, row_blocks: BlockIndices, col_blocks: BlockIndices):
        mat = mat.tocsr()
        mat.sum_duplicates()
        mat.sort_indices()
        # explicit zeros (False) never arise from boolean products here
        return cls.from_csr(row_blocks, col_blocks, mat.indptr.astype(np.int64), mat.indices.astype(np.int64))

    def entry_mask(self) -> np.ndarray:
        mask = np.zeros((self.row_blocks.total, self.col_blocks.total), dtype=bool)
        rb, cb = self.row_blocks, self.col_blocks
        for r, c in zip(self.block_rows().tolist(), self.col_index.tolist()):
            mask[rb.starts[r] : rb.starts[r + 1], cb.starts[c] : cb.starts[c + 1]] = True
        return mask

    def contains(self, other: "BlockSparsityPattern") -> bool:
        if self.row_blocks != other.row_blocks or self.col_blocks != other.col_blocks:
            return False
        theirs = other.keys()
        if theirs.size == 0:
            return True
        mine = self.keys()
        pos = np.searchsorted(mine, theirs)
        pos = np.minimum(pos, max(mine.size - 1, 0))
        return bool(mine.size) and bool(np.all(mine[pos] == theirs))

    def __eq__(self, other) -> bool:
        if self is other:
            return True
        return (
            isinstance(other, BlockSparsityPattern)
            and self.row_blocks == other.row_blocks
            and self.col_blocks == other.col_blocks
            and np.array_equal(self.row_start, other.row_start)
            and np.array_equal(self.col_index, other.col_index)
        )

    def __hash__(self):
        return hash((self.row_blocks.n_blocks, self.col_blocks.n_blocks, self.col_index.size))
