"""Shared builders for the parity tests (product API on one side, oracle on the other)."""

from __future__ import annotations

import numpy as np

from paper_1907_01005_b200.bcsr import BlockCsrMatrix
from paper_1907_01005_b200.localization import (
    build_support_sparsity,
    column_supports,
    grow_sparsity_for_operator,
    order_and_block_columns,
)
from paper_1907_01005_b200.matfree import CellOperator, make_dof_layout
from paper_1907_01005_b200.mesh import build_mesh, enumerate_dofs, partition_and_order_cells
from paper_1907_01005_b200.problem import hashed_entries
from paper_1907_01005_b200.support import ColumnSupport, attach_support


class Small:
    """Acceptance-style small problem (reference tests/_utils.py:35-59 shape)."""

    def __init__(self, extents, spacing, level, degree, centers, radius, block_size=3, vectors=2,
                 n_ranks=1):
        self.mesh = build_mesh(extents, spacing, level)
        self.partition = partition_and_order_cells(self.mesh, n_ranks)
        self.numbering = enumerate_dofs(self.mesh, self.partition, degree)
        self.layout = order_and_block_columns(self.mesh, self.partition, centers, radius, vectors,
                                              block_size)
        self.supports = column_supports(self.mesh, self.numbering, self.layout)
        self.pattern = build_support_sparsity(self.mesh, self.partition, self.numbering,
                                              self.layout, self.supports)
        self.grown = grow_sparsity_for_operator(self.pattern, self.mesh, self.numbering)
        self.n_ranks = n_ranks
        self.degree = degree
        self.support = ColumnSupport.from_localization(self.layout, self.supports,
                                                       self.numbering.n_dofs)
        keys = np.concatenate([c * self.numbering.n_dofs + s for c, s in enumerate(self.supports)])
        self._keys = np.sort(keys)

    def in_support(self, rows, new_cols):
        centre = self.layout.old_col_of_new[new_cols] // self.layout.vectors_per_center
        key = centre * self.numbering.n_dofs + rows
        pos = np.searchsorted(self._keys, key)
        return (pos < self._keys.size) & (self._keys[np.minimum(pos, self._keys.size - 1)] == key)

    def fill(self, m: BlockCsrMatrix, seed: int, scale: float = 1.0, attach=True):
        old = self.layout.old_col_of_new
        m.fill_owned_entries(lambda r, c: np.where(self.in_support(r, c),
                                                   scale * hashed_entries(seed, r, old[c]), 0.0))
        if attach:
            attach_support(m, self.support, check=True)
        return m

    def operands(self, ctx, device):
        rl = make_dof_layout(ctx, self.mesh, self.partition, self.numbering)
        op = CellOperator(self.mesh, self.partition, self.numbering, rl)
        x = BlockCsrMatrix(self.pattern, rl, ctx, 8, device)
        hx = BlockCsrMatrix(self.grown, rl, ctx, 8, device)
        return rl, op, x, hx


def cosine(seed):
    def v(points):
        return np.cos(np.atleast_2d(points) @ np.asarray([0.8, 1.4, 0.5]) + seed)

    return v


def to_original_columns(dense, layout):
    out = np.zeros_like(dense)
    out[:, layout.old_col_of_new] = dense
    return out
