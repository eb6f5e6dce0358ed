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

    def operands(self, ctx, device, lane_width=8):
        rl = make_dof_layout(ctx, self.mesh, self.partition, self.numbering)
        op = CellOperator(self.mesh, self.partition, self.numbering, rl)
        x = BlockCsrMatrix(self.pattern, rl, ctx, lane_width, device)
        hx = BlockCsrMatrix(self.grown, rl, ctx, lane_width, device)
        return rl, op, x, hx

    def projection_operands(self, ctx, device, rl, lane_width=8, seed=77):
        """(s, c, xc): projection target, a filled column-space matrix, X C target."""
        from paper_1907_01005_b200.energy import (column_space_ghost_blocks, make_column_layout,
                                                  projected_pattern)

        proj = projected_pattern(self.pattern, self.grown)
        ghosts = column_space_ghost_blocks(self.grown, proj, rl, self.layout.rank_block_start,
                                           ctx.rank)
        clayout = make_column_layout(ctx, self.layout.column_blocks, self.layout.rank_block_start,
                                     ghosts)
        s = BlockCsrMatrix(proj, clayout, ctx, lane_width, device)
        c = BlockCsrMatrix(proj, clayout, ctx, lane_width, device)
        c.fill_owned_entries(lambda r, col: hashed_entries(seed, r, col))
        xc = BlockCsrMatrix(self.pattern, rl, ctx, lane_width, device)
        return s, c, xc


def cosine(seed):
    def v(points):
        return np.cos(np.atleast_2d(points) @ np.asarray([0.8, 1.4, 0.5]) + seed)

    return v


def to_original_columns(dense, layout):
    out = np.zeros_like(dense)
    out[:, layout.old_col_of_new] = dense
    return out


def emulated_apply(op, potential, kind, src, dst):
    """CPU emulation of CellOperator.apply for CPU-resident matrices (tests only).

    The product's own sequence (CellOperator._overlapped: zero dst, src ghost
    update in flight during the interior part A of the cell loop, boundary
    cells, dst compress in flight during part B, release src ghosts) over
    the K1 plan's (cell, column) pairs, with the cell integral taken from the
    numpy oracle.  Exercises the host plan and the rank-context exchange in
    the overlapped order without a GPU.
    """
    import torch

    from oracle import numpy_oracle as O
    from paper_1907_01005_b200.matfree import _CellPlan

    deg = op.shape.degree
    n3 = (deg + 1) ** 3
    dst.ensure_owned()
    plan = _CellPlan(op, src, dst, upload=False)
    a = plan.arrays

    def run(p0, p1):
        if p1 <= p0:
            return
        cell = a["pair_cell"][p0:p1].astype(np.int64)
        codes = a["codes"].reshape(-1, plan.code_stride)[cell].astype(np.int64)
        if plan.wide:
            w0, w1 = codes[:, 0 : 2 * n3 : 2], codes[:, 1 : 2 * n3 : 2]
            g, rx, rh = w0 >> 27, w0 & 0x7FFFFFF, w1
        else:
            c = codes[:, :n3]
            g, rx, rh = c >> 27, (c >> 14) & 0x1FFF, c & 0x3FFF
        gt = a["gtab"].astype(np.int64)
        base = a["pair_gtab"][p0:p1, None] + 2 * g
        xo, ho = gt[base], gt[base + 1]
        X = src.data.numpy()
        u = np.where(xo >= 0, X[np.maximum(xo, 0) + rx], 0.0)
        vq = None
        if kind != "mass" and potential is not None:
            vq = O.sample_potential(potential, op.cell_origins[cell], deg, op.mesh.spacing)
        out = O.cell_integrals(deg, op.mesh.spacing, kind, u[:, :, None], vq)[:, :, 0]
        H = dst.data.numpy().copy()
        np.add.at(H, (ho + rh).ravel(), out.ravel())
        dst.data.copy_(torch.from_numpy(H))

    op._overlapped(plan, src, (dst,), run)
    return plan
