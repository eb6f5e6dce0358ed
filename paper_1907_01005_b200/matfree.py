"""Matrix-free mass / Hamiltonian application on GPU-resident BCSR multivectors.

Drop-in for the reference `bcsrmv/matfree.py` (same names and semantics).
`CellOperator.apply` keeps the reference's contract (`matfree.py:458-527`):
checks -> dst zeroed -> src ghosts updated -> cell loop -> src ghosts
released -> dst compressed.  The cell loop itself is one launch of a K1
kernel (csrc/bmv_k1.cu) over a precomputed plan on slab storage (slabs.py):

* per cell: the (group, row-in-block) slot of each of its (p+1)^3 DoFs,
  groups being the distinct local block rows in first-occurrence order
  (the reference CellDoFMap, `matfree.py:58-130`), encoded with the row
  offsets r * K of src and dst;
* the work list: (cell, column) pairs -- with a ColumnSupport declared on
  src only the columns whose support reaches the cell (support.py),
  otherwise every column src stores in the cell's block rows -- and per
  pair and group the slab positions of the column in src and dst; a column
  dst does not store raises PatternError like the reference's
  `advance_to` (`matfree.py:207-219`).

A destination built with `columns=op.image_columns(spec_of_src)`
(ImageColumns) stores exactly the columns the operator can reach.

The potential is sampled once per (operator, potential) at the cell
quadrature points (`matfree.py:35-40,491-495`): Gaussian-sum potentials on
the device, arbitrary callables on the host in cell chunks.

`CellOperator.apply_h_and_mass` computes H X and M X with one gather and
one interpolation (the two products compute_energy forms,
`energy.py:144-145`).
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch
from scipy import sparse

from . import _lib
from .bcsr import BlockCsrMatrix, RankLayout, _zero_range, build_rank_layout, serial_layout
from .blocks import BlockSparsityPattern
from .counters import OpCounters
from .errors import ConsistencyError, PatternError, ShapeError
from .localization import grow_sparsity_for_operator
from .mesh import CellPartition, DofNumbering, StructuredMesh, cells_nodes
from .shapes import ShapeInfo, collocation_derivative, shape_info

MASS = "mass"
HAMILTONIAN = "hamiltonian"
SUMFAC = "sumfac"
GEMM = "gemm"


@dataclass(frozen=True)
class OperatorSpec:
    kind: str
    potential: object = None  # None, a constant, or a callable of (n, 3) points

    def sample_potential(self, points: np.ndarray) -> np.ndarray:
        if self.potential is None:
            return np.zeros(points.shape[0])
        if callable(self.potential):
            return np.asarray(self.potential(points), dtype=float)
        return np.full(points.shape[0], float(self.potential))

    @property
    def potential_is_constant(self) -> bool:
        return not callable(self.potential)


def mass_operator() -> OperatorSpec:
    return OperatorSpec(MASS)


def hamiltonian_operator(potential=None) -> OperatorSpec:
    return OperatorSpec(HAMILTONIAN, potential)


class GaussianPotential:
    """V(x) = scale * sum_c exp(-|x - c|^2 / sigma^2), evaluable on host and device.

    BASELINE configs use scale = -1 over all orbital centres.  Calling the
    object evaluates on the host (numpy); the operator evaluates it on the
    GPU at the quadrature points.
    """

    def __init__(self, centers, sigma: float, scale: float = -1.0):
        self.centers = np.atleast_2d(np.asarray(centers, dtype=float))
        self.sigma = float(sigma)
        self.scale = float(scale)

    @property
    def inv_sigma2(self) -> float:
        return 1.0 / (self.sigma * self.sigma)

    def __call__(self, points):
        pts = np.atleast_2d(np.asarray(points, dtype=float))
        out = np.zeros(pts.shape[0])
        for c in self.centers:
            d = pts - c
            out += np.exp(-(d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1] + d[:, 2] * d[:, 2]) * self.inv_sigma2)
        return self.scale * out


# -- cell DoF map --------------------------------------------------------------


@dataclass(frozen=True)
class CellDoFMap:
    """Reference-format cell DoF map (`matfree.py:58-87`)."""

    dof_indices: np.ndarray   # (n, 2): (row in block, dof in cell), grouped by block
    block_indices: np.ndarray  # (m, 2): (local block, group size), first occurrence order
    cell_offsets: np.ndarray  # (n_cells + 1, 2)
    n_cell_dofs: int

    @property
    def n_cells(self) -> int:
        return self.cell_offsets.shape[0] - 1

    def cell_groups(self, cell: int):
        d0, b0 = self.cell_offsets[cell]
        _, b1 = self.cell_offsets[cell + 1]
        out, off = [], int(d0)
        for block, count in self.block_indices[int(b0) : int(b1)]:
            pairs = self.dof_indices[off : off + int(count)]
            out.append((int(block), pairs[:, 0], pairs[:, 1]))
            off += int(count)
        return out


def _first_occurrence_groups(lb: np.ndarray):
    """Native builder (libbmvplan) unless BMV_PLAN_NATIVE=0; same arrays as the numpy form."""
    from . import _plan

    lb = np.asarray(lb)
    if _plan.enabled() and lb.shape[0] > 0:
        return _plan.first_occurrence_groups(lb)
    return _first_occurrence_groups_numpy(lb)


def _first_occurrence_groups_numpy(lb: np.ndarray):
    """Group the DoFs of each cell by local block, groups in first-occurrence order.

    lb: (n_cells, n3) local block per cell DoF.  Returns
      slot_group (n_cells, n3) local group index of every DoF,
      grp_cell, grp_block (groups ordered by cell then first occurrence),
      cell_gstart (n_cells + 1).
    """
    n_cells, n3 = lb.shape
    if n_cells == 0:
        z = np.zeros(0, dtype=np.int64)
        return np.zeros((0, n3), dtype=np.int64), z, z, np.zeros(1, dtype=np.int64)
    width = int(lb.max()) + 1
    key = (np.arange(n_cells, dtype=np.int64)[:, None] * width + lb).ravel()
    order = np.argsort(key, kind="stable")  # by key, then DoF (stable)
    ks = key[order]
    first = np.ones(ks.size, dtype=bool)
    first[1:] = ks[1:] != ks[:-1]
    gid = np.cumsum(first) - 1
    n_groups = int(gid[-1]) + 1
    g_first_d = (order % n3)[first]
    g_cell = ks[first] // width
    g_block = ks[first] % width
    gorder = np.lexsort((g_first_d, g_cell))
    rank = np.empty(n_groups, dtype=np.int64)
    rank[gorder] = np.arange(n_groups)
    grp_cell = g_cell[gorder]
    cell_gstart = np.searchsorted(grp_cell, np.arange(n_cells + 1)).astype(np.int64)
    local = rank - cell_gstart[g_cell]
    slot_group = np.empty(ks.size, dtype=np.int64)
    slot_group[order] = local[gid]
    return slot_group.reshape(n_cells, n3), grp_cell, g_block[gorder], cell_gstart


def build_cell_dof_map_from_rows(cell_rows, map_rows) -> CellDoFMap:
    """Reference arrays (`matfree.py:90-116`), computed without a per-DoF loop."""
    cell_rows = np.asarray(cell_rows, dtype=np.int64)
    if cell_rows.ndim == 1:
        cell_rows = cell_rows[None, :]
    n_cells = cell_rows.shape[0]
    n3 = cell_rows.shape[1] if n_cells else 0
    lb, rib = map_rows(cell_rows.ravel())
    lb = np.asarray(lb).reshape(n_cells, n3)
    rib = np.asarray(rib).reshape(n_cells, n3)
    slot_group, grp_cell, grp_block, cell_gstart = _first_occurrence_groups(lb)
    d = np.tile(np.arange(n3), n_cells)
    cell = np.repeat(np.arange(n_cells), n3)
    gflat = slot_group.ravel()
    order = np.lexsort((d, gflat, cell))
    dof_indices = np.stack([rib.ravel()[order], d[order]], axis=1).astype(np.int64)
    counts = np.bincount(cell_gstart[cell] + gflat, minlength=grp_cell.size)
    block_indices = np.stack([grp_block, counts], axis=1).astype(np.int64)
    offsets = np.stack([np.arange(n_cells + 1) * n3, cell_gstart], axis=1).astype(np.int64)
    return CellDoFMap(dof_indices.reshape(-1, 2), block_indices.reshape(-1, 2), offsets, n3)


def build_cell_dof_map(mesh, numbering, layout, cells) -> CellDoFMap:
    return build_cell_dof_map_from_rows(cells_nodes(mesh, numbering, cells), layout.map_rows)


def owned_cell_ghost_rows(mesh, numbering, partition, rank) -> np.ndarray:
    cells = partition.cells_of_rank(rank)
    nodes = cells_nodes(mesh, numbering, cells).ravel()
    mark = np.zeros(int(nodes.max()) + 1 if nodes.size else 0, dtype=bool)
    mark[nodes] = True
    touched = np.flatnonzero(mark)  # == np.unique(nodes), without the sort
    lo, hi = numbering.owned_ranges[rank]
    return touched[(touched < lo) | (touched >= hi)]


def make_dof_layout(ctx, mesh, partition, numbering) -> RankLayout:
    ghost = owned_cell_ghost_rows(mesh, numbering, partition, ctx.rank)
    return build_rank_layout(ctx, numbering.row_blocks, numbering.rank_block_start, ghost)


# -- block-row accessor (host, API parity and diagnostics) ---------------------

_EXHAUSTED = np.iinfo(np.int64).max


class RowsBlockAccessor:
    """k-way merge over the column lists of a cell's block rows (`matfree.py:159-237`)."""

    def __init__(self, matrix: BlockCsrMatrix, cell_map: CellDoFMap):
        self.matrix = matrix
        self.cell_map = cell_map
        self._groups, self._cursor, self._end, self._col = [], [], [], []
        self.current_col = None

    def _column_at(self, g):
        if self._cursor[g] >= self._end[g]:
            return _EXHAUSTED
        return int(self.matrix.col_index[self._cursor[g]])

    def _refresh(self):
        c = min(self._col) if self._col else _EXHAUSTED
        self.current_col = None if c == _EXHAUSTED else c
        return self.current_col

    def reinit(self, cell):
        self._groups = self.cell_map.cell_groups(cell)
        rs = self.matrix.row_start
        self._cursor = [int(rs[b]) for b, _, _ in self._groups]
        self._end = [int(rs[b + 1]) for b, _, _ in self._groups]
        self._col = [self._column_at(g) for g in range(len(self._groups))]
        return self._refresh()

    def advance(self):
        if self.current_col is None:
            return None
        lim = self.current_col + 1
        for g in range(len(self._groups)):
            if self._cursor[g] < self._end[g] and self._col[g] < lim:
                self._cursor[g] += 1
                self._col[g] = self._column_at(g)
        return self._refresh()

    def advance_to(self, col):
        for g in range(len(self._groups)):
            while self._cursor[g] < self._end[g] and self._col[g] < col:
                self._cursor[g] += 1
                self._col[g] = self._column_at(g)
            if self._col[g] != col:
                raise PatternError(f"destination pattern misses column block {col} in local "
                                   f"block row {self._groups[g][0]}")
        self.current_col = col

    def active_groups(self):
        c = self.current_col
        return [(rows, dofs, self.matrix.block_values(self._cursor[g]))
                for g, (block, rows, dofs) in enumerate(self._groups) if self._col[g] == c]

    def emitted_columns(self, cell):
        out, c = [], self.reinit(cell)
        while c is not None:
            out.append(c)
            c = self.advance()
        return out


# -- per-mesh tables -------------------------------------------------------------


class _CellKernels:
    """1D/3D tables shared by all cells (`matfree.py:248-271`)."""

    def __init__(self, shape: ShapeInfo, spacing):
        self.shape = shape
        hx, hy, hz = (float(h) for h in spacing)
        self.det = hx * hy * hz
        w = shape.weights
        self.w3 = (w[:, None, None] * w[None, :, None] * w[None, None, :]) * self.det
        self.grad_scale = (0.5 / hx**2, 0.5 / hy**2, 0.5 / hz**2)
        pts = shape.points
        gz, gy, gx = np.meshgrid(pts * hz, pts * hy, pts * hx, indexing="ij")
        self.quad_offsets = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)

    def cell_quad_points(self, cell_origin) -> np.ndarray:
        return np.asarray(cell_origin) + self.quad_offsets


def sumfac_flops_per_lane(n: int, kind: str, with_potential: bool) -> int:
    """Reference-formulation flops of one cell integral per lane (`matfree.py:274-367`)."""
    if kind == MASS:
        return 12 * n**4 + n**3
    if with_potential:
        return 36 * n**4 + 8 * n**3
    return 34 * n**4 + 5 * n**3


def implemented_flops_per_pair(n: int, kind: str, with_potential: bool) -> int:
    """Flops the K1 kernel issues per pair (collocation form, FMA = 2)."""
    if kind == MASS:
        return 12 * n**4 + n**3
    return 24 * n**4 + (8 if with_potential else 6) * n**3


# -- the operator ------------------------------------------------------------------


def _expand(counts: np.ndarray):
    counts = np.asarray(counts, dtype=np.int64)
    owner = np.repeat(np.arange(counts.size, dtype=np.int64), counts)
    start = np.concatenate([[0], np.cumsum(counts)])[:-1]
    return owner, np.arange(int(counts.sum()), dtype=np.int64) - start[owner]


def _bool_csr(m) -> sparse.csr_matrix:
    m = m.tocsr()
    m.sum_duplicates()
    m.sort_indices()
    m.data[:] = 1
    return m


class ImageColumns:
    """Stored columns of an operator image H X (the `columns=` of a
    destination BlockCsrMatrix, slabs.py).

    Block row i stores column alpha iff some cell touching a row of i has the
    active pair (cell, alpha), i.e. the pair K1 computes when it applies the
    operator to a source with stored-column spec `source`: a ColumnSupport
    (entry level: the cell has a node in supp(alpha)) or any other spec
    (every stored column of the block rows the cell touches).  Defined per
    GLOBAL block row (the owner and every ghost copy agree), computed from
    the cells touching the requested block rows.
    """

    def __init__(self, op: "CellOperator", source):
        self.op = op
        self.source = source

    def key(self):
        return ("image", id(self.op), id(self.source))

    def columns_for(self, pattern, gblocks: np.ndarray):
        from . import _plan

        if _plan.enabled():
            return self._columns_native(pattern, gblocks)
        return self._columns_numpy(pattern, gblocks)

    def _columns_native(self, pattern, gblocks: np.ndarray):
        from . import _plan
        from .support import ColumnSupport

        op = self.op
        blocks = op.numbering.row_blocks
        gblocks = np.asarray(gblocks, dtype=np.int64)
        cells = op.cells_touching_blocks(gblocks)
        nodes = cells_nodes(op.mesh, op.numbering, cells)
        nb, _ = _plan.blocks_of(blocks.starts, nodes)
        if isinstance(self.source, ColumnSupport):
            row_sel, rptr, rcols = op.support_rows(self.source, nodes)
            pptr, pcols = _plan.cell_pairs(row_sel[nodes], rptr, rcols)
        else:
            touched = np.unique(nb)
            sptr, scols = self.source.columns_for(pattern, touched)
            pptr, pcols = _plan.cell_pairs(np.searchsorted(touched, nb), sptr, scols)
        sel = np.full(blocks.n_blocks, -1, dtype=np.int64)
        sel[gblocks] = np.arange(gblocks.size, dtype=np.int64)
        return _plan.block_image(sel[nb], pptr, pcols, gblocks.size, pattern.col_blocks.total)

    def _columns_numpy(self, pattern, gblocks: np.ndarray):
        """numpy restatement of the native image (sparse products)."""
        from .support import ColumnSupport

        op = self.op
        mesh, numbering = op.mesh, op.numbering
        blocks = numbering.row_blocks
        gblocks = np.asarray(gblocks, dtype=np.int64)
        n_cols = pattern.col_blocks.total
        cells = op.cells_touching_blocks(gblocks)
        nodes = cells_nodes(mesh, numbering, cells)  # (nc, n3) global rows
        nc, n3 = nodes.shape
        cell_of = np.repeat(np.arange(nc, dtype=np.int64), n3)
        flat = nodes.ravel()
        if isinstance(self.source, ColumnSupport):
            ptr, rows = self.source.csr()
            # support restricted to the rows these cells touch
            mark = np.full(numbering.n_dofs, -1, dtype=np.int64)
            uniq = np.unique(flat)
            mark[uniq] = np.arange(uniq.size, dtype=np.int64)
            col_of = np.repeat(np.arange(self.source.n_cols, dtype=np.int64), np.diff(ptr))
            sel = mark[rows] >= 0
            xm = sparse.csr_matrix((np.ones(int(sel.sum()), dtype=np.int32),
                                    (mark[rows[sel]], col_of[sel])), shape=(uniq.size, n_cols))
            a = sparse.csr_matrix((np.ones(flat.size, dtype=np.int32), (cell_of, mark[flat])),
                                  shape=(nc, uniq.size))
            act = _bool_csr(a @ xm)
        else:
            gb = blocks.blocks_of(flat)
            touched = np.unique(gb)
            sptr, scols = self.source.columns_for(pattern, touched)
            tpos = np.searchsorted(touched, gb)
            inc = _bool_csr(sparse.csr_matrix((np.ones(flat.size, dtype=np.int32),
                                               (cell_of, tpos)), shape=(nc, touched.size)))
            s = sparse.csr_matrix((np.ones(scols.size, dtype=np.int32), scols, sptr),
                                  shape=(touched.size, n_cols))
            act = _bool_csr(inc @ s)
        # cell -> requested block rows it touches
        sel = np.full(blocks.n_blocks, -1, dtype=np.int64)
        sel[gblocks] = np.arange(gblocks.size, dtype=np.int64)
        sb = sel[blocks.blocks_of(flat)]
        ok = sb >= 0
        touch = _bool_csr(sparse.csr_matrix((np.ones(int(ok.sum()), dtype=np.int32),
                                             (sb[ok], cell_of[ok])), shape=(gblocks.size, nc)))
        img = _bool_csr(touch @ act)
        return img.indptr.astype(np.int64), img.indices.astype(np.int64)


class _CellPlan:
    """Device plan of K1 (csrc/bmv_k1.cu) for one (src, dst) geometry couple."""

    def __init__(self, op: "CellOperator", src: BlockCsrMatrix, dst: BlockCsrMatrix,
                 upload: bool = True):
        n = op.shape.degree + 1
        n3 = n**3
        n_cells = op.slot_group.shape[0]
        ng = np.diff(op.cell_gstart)
        # work list: (cell, column) pairs, cells in Hilbert order, columns ascending
        if src.support is not None:
            act = op.active_pairs(src.support)
            self.support_based = True
        else:
            inc = _bool_csr(sparse.csr_matrix(
                (np.ones(op.grp_cell.size, dtype=np.int32), (op.grp_cell, op.grp_block)),
                shape=(n_cells, src.n_local_blocks)))
            sg = src.slab
            s = sparse.csr_matrix((np.ones(sg.cols.size, dtype=np.int32), sg.cols, sg.ptr),
                                  shape=(src.n_local_blocks, src.col_blocks.total))
            act = _bool_csr(inc @ s)
            self.support_based = False
        # pair order: interior cells part A | cells with a ghost row | interior part B,
        # so apply() runs A during the halo exchange of src and B during the compress
        cnt = np.diff(act.indptr).astype(np.int64)
        ghost = (op._lb >= op.layout.n_owned_blocks).any(axis=1) if n_cells else \
            np.zeros(0, dtype=bool)
        interior = np.flatnonzero(~ghost)
        cum = np.cumsum(cnt[interior])
        half = int(np.searchsorted(cum, cum[-1] // 2)) + 1 if interior.size and ghost.any() \
            else interior.size
        order = np.concatenate([interior[:half], np.flatnonzero(ghost), interior[half:]])
        owner_c, k = _expand(cnt[order])
        p_cell = order[owner_c]
        p_col = act.indices[act.indptr[order][owner_c] + k].astype(np.int64)
        n_pairs = p_col.size
        n_a = int(cnt[interior[:half]].sum())
        self.split = (n_a, n_a + int(cnt[ghost].sum()))
        # per (pair, group): {src slab offset + slot | -1, dst slab offset + slot}
        pg = ng[p_cell]
        ngp = pg + (pg & 1)
        if ngp.size and int(ngp.max()) > 32:
            raise ConsistencyError("a cell touches more than 32 block rows")
        if max(int(src.slab.off[-1]), int(dst.slab.off[-1])) >= 2**31:
            raise ShapeError("K1 offsets exceed 2^31 elements")
        pair_gtab = np.concatenate([[0], np.cumsum(2 * ngp)]).astype(np.int64)
        from . import _plan

        if _plan.enabled():
            gtab, bad = _plan.k1_gtab(p_cell, p_col, op.cell_gstart, op.grp_block, src.slab,
                                      dst.slab, pair_gtab[:-1], int(pair_gtab[-1]))
            if bad >= 0:
                raise PatternError(f"destination does not store column {int(p_col[bad])} in a "
                                   f"block row reached by cell {int(p_cell[bad])}")
        else:
            owner, g = _expand(pg)
            lb = op.grp_block[op.cell_gstart[p_cell][owner] + g]
            col = p_col[owner]
            zero = np.zeros(lb.size, dtype=np.int64)
            xo = src.slab.offsets(lb, zero, col)
            ho = dst.slab.offsets(lb, zero, col)
            if (ho < 0).any():
                bad = int(np.flatnonzero(ho < 0)[0])
                raise PatternError(f"destination does not store column {int(col[bad])} in local "
                                   f"block row {int(lb[bad])} (reached by cell "
                                   f"{int(p_cell[owner[bad]])})")
            gtab = np.zeros(int(pair_gtab[-1]), dtype=np.int32)
            gtab[0::2] = -1
            at = pair_gtab[:-1][owner] + 2 * g
            gtab[at] = xo
            gtab[at + 1] = ho
        # per (cell, DoF) codes: group, r * K_src, r * K_dst
        sgp = op.slot_group
        lbd, rib = op._lb, op._rib
        rkx = rib * src.slab.width[lbd]
        rkh = rib * dst.slab.width[lbd]
        wide = bool(n_cells and (int(sgp.max()) >= 32 or int(rkx.max()) >= 1 << 13
                                 or int(rkh.max()) >= 1 << 14))
        if os.environ.get("BMV_K1_WIDE") == "1":  # tests: force the 64-bit code rows
            wide = True
        if wide:
            if n_cells and (int(rkx.max()) >= 1 << 27 or int(rkh.max()) >= 1 << 31):
                raise ShapeError("K1 codes: block rows too large for 32-bit row offsets")
            stride = (2 * n3 + 3) // 4 * 4
            codes = np.zeros((n_cells, stride), dtype=np.uint32)
            codes[:, 0 : 2 * n3 : 2] = (sgp << 27) | rkx
            codes[:, 1 : 2 * n3 : 2] = rkh
        else:
            stride = (n3 + 3) // 4 * 4
            codes = np.zeros((n_cells, stride), dtype=np.uint32)
            codes[:, :n3] = (sgp << 27) | (rkx << 14) | rkh
        self.n = n
        self.n_cells = n_cells
        self.n_pairs = int(n_pairs)
        self.wide = wide
        self.max_groups = int(ngp.max()) if ngp.size else 2
        self.cells_visited = int(np.count_nonzero(np.diff(act.indptr)))
        # reference accounting (OpCounters): visits = (cell, column block) couples
        # of the RowsBlockAccessor over src's block pattern
        inc_b = _bool_csr(sparse.csr_matrix(
            (np.ones(op.grp_cell.size, dtype=np.int32), (op.grp_cell, op.grp_block)),
            shape=(n_cells, src.n_local_blocks)))
        xp = sparse.csr_matrix((np.ones(src.col_index.size, dtype=np.int32), src.col_index,
                                src.row_start), shape=(src.n_local_blocks, src.col_blocks.n_blocks))
        vis = _bool_csr(inc_b @ xp)
        visit_col = vis.indices.astype(np.int64)
        self.n_visits = int(visit_col.size)
        self.lane_groups = int(np.sum((src.col_strides[visit_col] + src.lane_width - 1)
                                      // src.lane_width))
        self.dof_lane_slots = int(n3 * np.sum(src.col_strides[visit_col]))
        self.arrays = dict(
            pair_cell=np.ascontiguousarray(p_cell, dtype=np.int32),
            pair_gtab=np.ascontiguousarray(pair_gtab[:-1], dtype=np.int64),
            pair_ngp=np.ascontiguousarray(ngp, dtype=np.int32),
            gtab=gtab,
            codes=np.ascontiguousarray(codes.ravel()),
        )
        self.code_stride = stride
        self.handle = None
        self.launches = 0
        if upload:
            self.upload(op)

    def upload(self, op):
        n, arrs = self.n, self.arrays
        lib = _lib.load()
        d = _lib.CellopDesc()
        d.n, d.wide, d.n_cells = n, 1 if self.wide else 0, self.n_cells
        d.code_stride, d.max_groups = self.code_stride, self.max_groups
        d.n_pairs, d.gtab_len = self.n_pairs, int(arrs["gtab"].size)
        d.pair_cell = _lib.ptr(arrs["pair_cell"], C.c_int32)
        d.pair_gtab = _lib.ptr(arrs["pair_gtab"], C.c_int64)
        d.pair_ngp = _lib.ptr(arrs["pair_ngp"], C.c_int32)
        d.gtab = _lib.ptr(arrs["gtab"], C.c_int32)
        d.codes = _lib.ptr(arrs["codes"], C.c_uint32)
        breaks = np.ascontiguousarray(sorted(set(int(b) for b in self.split)), dtype=np.int64)
        d.n_breaks = int(breaks.size)
        d.breaks = _lib.ptr(breaks, C.c_int64)
        sh = op.shape
        dco = collocation_derivative(sh)
        for i in range(n):
            d.w[i] = float(sh.weights[i])
            for j in range(n):
                d.S[i * n + j] = float(sh.values[i, j])
                d.Dco[i * n + j] = float(dco[i, j])
        ker = op.kernels
        for k in range(3):
            d.kin[k] = ker.det * ker.grad_scale[k]
        d.det = ker.det
        raw = C.c_void_p()
        _lib.check(lib.bmv_cellop_create(C.byref(d), C.byref(raw)), "bmv_cellop_create")
        self.handle = _lib.Handle("bmv_cellop_destroy", raw)
        nl = C.c_int32()
        _lib.check(lib.bmv_cellop_launches(self.handle.raw, C.byref(nl)))
        self.launches = int(nl.value)


class CellOperator:
    """Rank-local matrix-free operator bound to a mesh and a row layout."""

    def __init__(self, mesh: StructuredMesh, partition: CellPartition,
                 numbering: DofNumbering, layout: RankLayout):
        self.mesh = mesh
        self.partition = partition
        self.numbering = numbering
        self.layout = layout
        self.cells = partition.cells_of_rank(layout.rank)
        self.shape = shape_info(numbering.degree)
        self.kernels = _CellKernels(self.shape, mesh.spacing)
        rows = cells_nodes(mesh, numbering, self.cells)
        n3 = (numbering.degree + 1) ** 3
        rows = rows.reshape(len(self.cells), n3)
        self._cell_rows = rows  # global DoF rows of the rank's cells (reused by the planners)
        lb, rib = layout.map_rows(rows.ravel())
        lb = lb.reshape(rows.shape)
        rib = rib.reshape(rows.shape)
        self.slot_group, self.grp_cell, self.grp_block, self.cell_gstart = \
            _first_occurrence_groups(lb)
        if self.slot_group.size and (int(self.slot_group.max()) > 255 or int(rib.max()) >= 1 << 24):
            raise ConsistencyError("cell touches more than 256 block rows or a block row > 2^24 rows")
        self.cell_slots = (self.slot_group << 24) | rib
        self._lb, self._rib = lb, rib
        self._cell_map = None
        if len(self.cells):
            ijk = mesh.cells_ijk(self.cells)
            self.cell_origins = np.asarray(mesh.origin) + ijk * np.asarray(mesh.spacing)
            self.cell_color = (ijk[:, 0] & 1) + 2 * (ijk[:, 1] & 1) + 4 * (ijk[:, 2] & 1)
        else:
            self.cell_origins = np.zeros((0, 3))
            self.cell_color = np.zeros(0, dtype=np.int64)
        self._plans: dict = {}
        self._coefs: dict = {}
        self._act: dict = {}
        self._rows: dict = {}
        self._images: dict = {}
        self._dev_tables = None
        self._node_of_dof = None

    @property
    def cell_map(self) -> CellDoFMap:
        if self._cell_map is None:
            self._cell_map = build_cell_dof_map(self.mesh, self.numbering, self.layout, self.cells)
        return self._cell_map

    def cell_local_rows_matrix(self, n_local_rows: int) -> sparse.csr_matrix:
        starts = np.concatenate([[0], np.cumsum(self.layout.local_row_counts())]).astype(np.int64)
        loc = starts[self._lb] + self._rib
        n_cells, n3 = loc.shape
        return sparse.csr_matrix((np.ones(loc.size, dtype=np.int32), loc.ravel(),
                                  np.arange(0, loc.size + 1, n3)), shape=(n_cells, n_local_rows))

    # -- supports, images and plans ---------------------------------------------

    def active_pairs(self, support) -> sparse.csr_matrix:
        """(owned cells x columns) bool CSR: the cell has a node in the column's support."""
        from . import _plan

        hit = self._act.get(id(support))
        if hit is not None and hit[0] is support:
            return hit[1]
        if _plan.enabled():
            nodes = self._cell_rows
            row_sel, rptr, rcols = self.support_rows(support, nodes)
            ptr, cols = _plan.cell_pairs(row_sel[nodes], rptr, rcols)
            act = sparse.csr_matrix((np.ones(cols.size, dtype=np.int8), cols.astype(np.int64), ptr),
                                    shape=(len(self.cells), support.n_cols))
        else:
            mask = support.local_mask(self.layout)
            a_cell = self.cell_local_rows_matrix(mask.shape[0])
            act = _bool_csr(a_cell @ mask.astype(np.int32))
        self._act[id(support)] = (support, act)
        return act

    def support_rows(self, support, nodes: np.ndarray):
        """(row_sel, ptr, cols): the support's row -> columns CSR over the rows
        of the cells touching this rank's block rows (native transpose; cached
        per support).  `nodes` must lie in those rows."""
        from . import _plan

        hit = self._rows.get(id(support))
        if hit is None or hit[0] is not support:
            cells = self.cells_touching_blocks(self.layout.global_blocks_of_locals())
            rows = cells_nodes(self.mesh, self.numbering, cells).ravel()
            row_sel = np.full(self.numbering.n_dofs, -1, dtype=np.int64)
            row_sel[rows] = 0
            sel = np.flatnonzero(row_sel == 0)
            row_sel[sel] = np.arange(sel.size, dtype=np.int64)
            ptr, cols = _plan.support_transpose(support, row_sel, sel.size)
            hit = (support, row_sel, ptr, cols)
            self._rows[id(support)] = hit
        if (hit[1][nodes] < 0).any():
            raise ConsistencyError("support_rows: rows outside the rank's neighbourhood")
        return hit[1], hit[2], hit[3]

    def image_columns(self, source) -> ImageColumns:
        """Stored-column spec of H X for a source X stored with spec `source`
        (`BlockCsrMatrix(grown_pattern, layout, ctx, columns=op.image_columns(support))`)."""
        hit = self._images.get(id(source))
        if hit is None or hit.source is not source:
            hit = ImageColumns(self, source)
            self._images[id(source)] = hit
        return hit

    def cells_touching_blocks(self, gblocks: np.ndarray) -> np.ndarray:
        """Global ids of the cells with a node in one of the global block rows."""
        mesh, numbering = self.mesh, self.numbering
        blocks = numbering.row_blocks
        gblocks = np.asarray(gblocks, dtype=np.int64)
        if gblocks.size == blocks.n_blocks:
            return np.arange(mesh.n_cells, dtype=np.int64)
        if self._node_of_dof is None:
            inv = np.empty(numbering.n_dofs, dtype=np.int64)
            inv[numbering.new_index_of_node] = np.arange(numbering.n_dofs, dtype=np.int64)
            self._node_of_dof = inv
        sz = blocks.sizes[gblocks]
        owner = np.repeat(np.arange(gblocks.size, dtype=np.int64), sz)
        first = np.concatenate([[0], np.cumsum(sz)])[:-1]
        rows = blocks.starts[gblocks][owner] + (np.arange(int(sz.sum())) - first[owner])
        node = self._node_of_dof[rows]
        p = numbering.degree
        sx, sy, _ = mesh.node_grid_shape(p)
        ex, ey, ez = mesh.extents
        idx = (node % sx, (node // sx) % sy, node // (sx * sy))
        cand = []
        for axis_lo in range(8):
            ok = np.ones(node.size, dtype=bool)
            c = []
            for ax, (v, e) in enumerate(zip(idx, (ex, ey, ez))):
                lo = (axis_lo >> ax) & 1
                ci = v // p - lo
                good = (ci >= 0) & (ci < e)
                if lo:
                    good &= (v % p) == 0
                ok &= good
                c.append(ci)
            cand.append((c[0] + ex * (c[1] + ey * c[2]))[ok])
        return np.unique(np.concatenate(cand))

    def plan_for(self, src: BlockCsrMatrix, dst: BlockCsrMatrix) -> _CellPlan:
        key = (id(src.slab), id(src.support), id(dst.slab))
        hit = self._plans.get(key)
        if hit is not None and hit[1] is src.slab and hit[2] is src.support and hit[3] is dst.slab:
            return hit[0]
        plan = _CellPlan(self, src, dst)
        self._plans[key] = (plan, src.slab, src.support, dst.slab)
        while len(self._plans) > 8:
            self._plans.pop(next(iter(self._plans)))
        return plan

    def _device_tables(self, device):
        if self._dev_tables is None:
            f = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=device)
            self._dev_tables = (f(self.cell_origins.reshape(-1, 3)), f(self.kernels.quad_offsets),
                                f(self.kernels.w3.ravel()))
        return self._dev_tables

    def coefficient(self, spec: OperatorSpec, device):
        """(device tensor or None, cell stride) of the quadrature coefficient.

        Rows are padded to q3p = q^3 rounded up to even (16-byte rows, staged
        by TMA in K1); the stride is q3p for a per-cell coefficient and 0 for
        one shared by every cell."""
        q3 = self.shape.n_q ** 3
        q3p = q3 + (q3 & 1)
        if spec.kind == MASS:
            key = ("mass",)
        elif spec.kind == HAMILTONIAN:
            if spec.potential is None:
                return None, 0
            key = ("pot", id(spec.potential)) if callable(spec.potential) else ("const", float(spec.potential))
        else:
            raise ShapeError(f"unknown operator kind {spec.kind!r}")
        hit = self._coefs.get(key)
        if hit is not None and (key[0] != "pot" or hit[2] is spec.potential):
            return hit[0], hit[1]
        w3 = self.kernels.w3.ravel()

        def padded_row(v):
            return torch.as_tensor(np.concatenate([v, np.zeros(q3p - q3)]), device=device)

        if key[0] == "mass":
            coef, stride = padded_row(w3), 0
        elif key[0] == "const":
            coef, stride = padded_row(w3 * float(spec.potential)), 0
        elif isinstance(spec.potential, GaussianPotential):
            pot = spec.potential
            n_cells = len(self.cells)
            org, qoff, w3d = self._device_tables(device)
            cen = torch.as_tensor(pot.centers, dtype=torch.float64, device=device)
            acc = torch.zeros(max(n_cells, 1) * q3, dtype=torch.float64, device=device)
            lib = _lib.require_device()
            chunk = 4096
            for c0 in range(0, max(pot.centers.shape[0], 1), chunk):
                part = cen[c0 : c0 + chunk]
                tmp = torch.empty_like(acc)
                _lib.check(lib.bmv_potential_gaussian(
                    n_cells, q3, _lib.dptr(org), _lib.dptr(qoff), _lib.dptr(w3d), _lib.dptr(part),
                    int(part.shape[0]), pot.inv_sigma2, pot.scale, _lib.dptr(tmp),
                    _lib.stream_handle(device)), "bmv_potential_gaussian")
                acc += tmp
            coef = torch.zeros(max(n_cells, 1), q3p, dtype=torch.float64, device=device)
            coef[:, :q3] = acc.view(-1, q3)
            coef = coef.view(-1)
            stride = q3p
        else:
            n_cells = len(self.cells)
            vals = np.zeros((n_cells, q3p))
            step = 4096
            for c0 in range(0, n_cells, step):
                pts = (self.cell_origins[c0 : c0 + step, None, :]
                       + self.kernels.quad_offsets[None, :, :]).reshape(-1, 3)
                vals[c0 : c0 + step, :q3] = spec.sample_potential(pts).reshape(-1, q3) * w3[None, :]
            coef, stride = torch.as_tensor(vals.ravel(), device=device), q3p
        self._coefs[key] = (coef, stride, spec.potential)
        return coef, stride

    # -- apply ------------------------------------------------------------------

    def _check_operands(self, spec, src, dst, variant):
        if src.layout is not self.layout or dst.layout is not self.layout:
            raise ShapeError("operator and operands must share one rank layout")
        if src.col_blocks != dst.col_blocks or src.lane_width != dst.lane_width:
            raise ShapeError("src and dst must share column blocking and lanes")
        if variant not in (SUMFAC, GEMM):
            raise ShapeError(f"unknown operator variant {variant!r}")
        if spec.kind not in (MASS, HAMILTONIAN):
            raise ShapeError(f"unknown operator kind {spec.kind!r}")

    def apply(self, spec: OperatorSpec, src: BlockCsrMatrix, dst: BlockCsrMatrix,
              variant: str = SUMFAC, counters: OpCounters | None = None):
        """dst = Op(spec) @ src over the rank's cells, then compress dst
        (reference matfree.py:458-527).  With ghost rows the exchanges overlap
        the cell loop: src's ghost update is in flight while the cells
        touching no ghost row (part A) run, the compress of dst while part B
        runs; the cells with ghost rows run in between."""
        self._check_operands(spec, src, dst, variant)
        lib = _lib.require_device()
        dst.ensure_owned()
        plan = self.plan_for(src, dst)
        if variant == GEMM:
            self._apply_gemm(spec, plan, src, dst)
            if counters is not None:
                self._count(spec, variant, plan, src, dst, counters)
            return
        coef, stride = self.coefficient(spec, dst.device)
        kin = 1 if spec.kind == HAMILTONIAN else 0
        cp = _lib.dptr(coef) if coef is not None else C.c_void_p(None)
        stream = _lib.stream_handle(dst.device)

        def run(p0, p1):
            _lib.check(lib.bmv_cellop_apply_pairs(
                plan.handle.raw, kin, cp, stride, _lib.dptr(src.data), _lib.dptr(dst.data), p0, p1,
                stream), "bmv_cellop_apply_pairs")

        self._overlapped(plan, src, (dst,), run)
        if counters is not None:
            self._count(spec, variant, plan, src, dst, counters)

    # -- element-matrix variant (comparison point) -------------------------------

    def _base_element_matrix(self, kind: str) -> np.ndarray:
        """Cell-independent part of the element matrix (reference
        `element_matrices`, matfree.py:375-397): the kinetic term by direct
        quadrature on the tensor-product tables (x fastest), or 0 for mass."""
        n3 = (self.shape.degree + 1) ** 3
        if kind != HAMILTONIAN:
            return np.zeros((n3, n3))
        S, D = self.shape.values, self.shape.derivatives
        w = self.kernels.w3.ravel()
        g3 = (np.kron(S, np.kron(S, D)), np.kron(S, np.kron(D, S)), np.kron(D, np.kron(S, S)))
        out = np.zeros((n3, n3))
        for g, c in zip(g3, self.kernels.grad_scale):
            out += g.T @ ((w * c)[:, None] * g)
        return out

    def _apply_gemm(self, spec, plan, src, dst, cells_per_chunk: int = 512):
        """variant='gemm' (reference matfree.py:375-397, 496, 509-511): per cell
        the dense element matrix A_c = K + N3^T diag(w3 V_c) N3 times the
        gathered block of the cell's active columns.  The paper's comparison
        point ("FE op. (BCSR gemm)"), not the hot path: batched cuBLAS products
        (torch.bmm) over cell chunks, gather / scatter index lists built on the
        host from the K1 plan's codes and group tables at every call."""
        dev = dst.device
        arr = plan.arrays
        n = plan.n
        n3 = n ** 3
        S = self.shape.values
        nn3 = torch.as_tensor(np.kron(S, np.kron(S, S)), device=dev)           # (q3, n3)
        base = torch.as_tensor(self._base_element_matrix(spec.kind), device=dev)
        coef, stride = self.coefficient(spec, dev)
        q3 = self.shape.n_q ** 3
        p_cell = arr["pair_cell"].astype(np.int64)
        codes = arr["codes"].reshape(plan.n_cells, plan.code_stride)
        gtab = arr["gtab"].astype(np.int64)
        pgt = arr["pair_gtab"]
        _zero_range(dst.data, 0, dst.data.numel())
        src.update_ghost_values()
        # cells in plan order; a cell's pairs are consecutive
        starts = np.flatnonzero(np.r_[True, p_cell[1:] != p_cell[:-1]]) if p_cell.size else \
            np.zeros(0, dtype=np.int64)
        ends = np.r_[starts[1:], p_cell.size]
        for c0 in range(0, starts.size, cells_per_chunk):
            ps, pe = starts[c0 : c0 + cells_per_chunk], ends[c0 : c0 + cells_per_chunk]
            cells = p_cell[ps]
            cnt = pe - ps
            kmax = int(cnt.max())
            pairs = np.arange(int(ps[0]), int(pe[-1]), dtype=np.int64)
            pc = p_cell[pairs]
            row = codes[pc]                                   # (pairs, stride) code rows
            if plan.wide:
                g = (row[:, 0 : 2 * n3 : 2] >> 27).astype(np.int64)
                rkx = (row[:, 0 : 2 * n3 : 2] & 0x7FFFFFF).astype(np.int64)
                rkh = row[:, 1 : 2 * n3 : 2].astype(np.int64)
            else:
                g = (row[:, :n3] >> 27).astype(np.int64)
                rkx = ((row[:, :n3] >> 14) & 0x1FFF).astype(np.int64)
                rkh = (row[:, :n3] & 0x3FFF).astype(np.int64)
            at = pgt[pairs][:, None] + 2 * g
            xo = gtab[at]
            ho = gtab[at + 1]
            x_off = np.where(xo >= 0, xo + rkx, -1)           # (pairs, n3)
            h_off = ho + rkh
            xt = torch.as_tensor(np.maximum(x_off, 0), device=dev)
            u = src.data[xt] * torch.as_tensor(x_off >= 0, device=dev)
            # pack the pairs of each cell into a padded block (cells, n3, kmax)
            slot = pairs - np.repeat(ps, cnt)
            cidx = np.repeat(np.arange(cells.size), cnt)
            blk = torch.zeros(cells.size, kmax, n3, dtype=torch.float64, device=dev)
            ci, si = torch.as_tensor(cidx, device=dev), torch.as_tensor(slot, device=dev)
            blk[ci, si] = u
            if coef is None:
                a_c = base.expand(cells.size, n3, n3)
            else:
                cw = coef.view(-1, stride)[:, :q3] if stride else coef[:q3].view(1, q3)
                cc = cw[torch.as_tensor(cells, device=dev)] if stride else cw.expand(cells.size, q3)
                a_c = base + torch.einsum("qi,cq,qj->cij", nn3, cc, nn3)
            out = torch.bmm(a_c, blk.transpose(1, 2))          # (cells, n3, kmax)
            vals = out.transpose(1, 2)[ci, si]                  # (pairs, n3)
            dst.data.index_add_(0, torch.as_tensor(h_off.ravel(), device=dev), vals.reshape(-1))
        src.release_ghosts()
        dst.support = None
        dst.compress()

    def _overlapped(self, plan, src, dsts, run):
        """zero dsts | src ghost update || part A | boundary | compress dsts || part B."""
        for d in dsts:
            _zero_range(d.data, 0, d.data.numel())
        a_end, b_beg = plan.split
        src.update_ghost_values_start()
        run(0, a_end)
        src.update_ghost_values_finish()
        run(a_end, b_beg)
        for d in dsts:
            d.support = None
            d.compress_start()
        run(b_beg, plan.n_pairs)
        src.release_ghosts()
        for d in dsts:
            d.compress_finish()

    def apply_h_and_mass(self, spec: OperatorSpec, src: BlockCsrMatrix, hdst: BlockCsrMatrix,
                         mdst: BlockCsrMatrix, counters: OpCounters | None = None):
        """hdst = H(spec) @ src and mdst = M @ src (the two products
        compute_energy forms, reference energy.py:129-174), fused: one gather
        of src and one interpolation to the quadrature points feed both
        (bmv_cellop_apply_hm_pairs).  When the destinations store different
        entries it runs the two applies instead; the choice depends only on
        the operands' storage, which every rank shares, so all ranks run the
        same exchange sequence."""
        if spec.kind != HAMILTONIAN:
            raise ShapeError("apply_h_and_mass takes the Hamiltonian spec")
        for d in (hdst, mdst):
            self._check_operands(spec, src, d, SUMFAC)
        same = (hdst.pattern is mdst.pattern and hdst.columns is mdst.columns)
        if not same:
            self.apply(spec, src, hdst, counters=counters)
            self.apply(mass_operator(), src, mdst, counters=counters)
            return
        lib = _lib.require_device()
        plan = self.plan_for(src, hdst)
        hdst.ensure_owned()
        mdst.ensure_owned()
        coef, stride = self.coefficient(spec, hdst.device)
        mcoef, _ = self.coefficient(mass_operator(), hdst.device)
        cp = _lib.dptr(coef) if coef is not None else C.c_void_p(None)
        stream = _lib.stream_handle(hdst.device)

        def run(p0, p1):
            _lib.check(lib.bmv_cellop_apply_hm_pairs(
                plan.handle.raw, cp, stride, _lib.dptr(mcoef), _lib.dptr(src.data),
                _lib.dptr(hdst.data), _lib.dptr(mdst.data), p0, p1, stream),
                "bmv_cellop_apply_hm_pairs")

        self._overlapped(plan, src, (hdst, mdst), run)
        if counters is not None:
            self._count(spec, SUMFAC, plan, src, hdst, counters)
            self._count(mass_operator(), SUMFAC, plan, src, mdst, counters)

    def _count(self, spec, variant, plan, src, dst, counters):
        n = plan.n
        w = src.lane_width
        with_v = spec.kind == HAMILTONIAN and spec.potential is not None
        if variant == GEMM:  # reference accounting: 2 (n^3)^2 per lane (matfree.py:509-511)
            counters.flops += plan.lane_groups * 2 * (n ** 3) ** 2 * w
        else:
            counters.flops += plan.lane_groups * sumfac_flops_per_lane(n, spec.kind, with_v) * w
        counters.cells_visited += plan.cells_visited
        counters.col_blocks_visited += plan.n_visits
        counters.dof_lane_slots += plan.dof_lane_slots
        ghost_vals = int(src.slab.off[-1] - src.slab.ghost_begin)
        counters.bytes_moved += 8 * (src.data.numel() + 2 * dst.data.numel()) + 16 * ghost_vals
        counters.add_extra("pairs", plan.n_pairs)
        counters.add_extra("flops_implemented",
                           plan.n_pairs * implemented_flops_per_pair(n, spec.kind, with_v))
        counters.add_extra("kernel_launches", plan.launches)


def flop_report(variant, mesh, spec, pattern, partition, numbering, lane_width=8) -> dict:
    """Analytic accounting of one serial application (`matfree.py:578-611`); no launch."""
    layout = serial_layout(numbering.row_blocks)
    grown = grow_sparsity_for_operator(pattern, mesh, numbering)
    op = CellOperator(mesh, partition, numbering, layout)
    src = BlockCsrMatrix(pattern, layout, None, lane_width, device="cpu")
    visits = 0
    slots = 0
    lane_groups = 0
    for ci in range(len(op.cells)):
        cols = RowsBlockAccessor(src, op.cell_map).emitted_columns(ci)
        visits += len(cols)
        strides = src.col_strides[np.asarray(cols, dtype=np.int64)] if cols else np.zeros(0, np.int64)
        slots += int(op.cell_map.n_cell_dofs * strides.sum())
        lane_groups += int(((strides + lane_width - 1) // lane_width).sum())
    n = numbering.degree + 1
    with_v = spec.kind == HAMILTONIAN and spec.potential is not None
    if variant == GEMM:
        flops = lane_groups * 2 * (n**3) ** 2 * lane_width
    else:
        flops = lane_groups * sumfac_flops_per_lane(n, spec.kind, with_v) * lane_width
    dst_vals = BlockCsrMatrix(grown, layout, None, lane_width, device="cpu").data.numel()
    return {"variant": variant, "kind": spec.kind, "flops": flops, "dof_lane_slots": slots,
            "flops_per_dof": flops / slots if slots else 0.0, "col_blocks_visited": visits,
            "cells_visited": int(len(op.cells)),
            "bytes_est": 8 * (src.data.numel() + 2 * dst_vals)}
