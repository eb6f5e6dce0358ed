"""BASELINE workloads: configs, seeded inputs, per-rank operand setup.

The five configs of BASELINE.json, built with this package's (bit-exact)
setup functions and the choices of SURVEY section 0.1: coarse level 0,
column blocks of B = 8, one vector per centre (M1-M3), values
2 * hashed_values(seed, row, original column) masked by the support (M4,
the reference's splitmix64 counter hash, `bench/problem.py:85-131`),
Y = second multivector with seed 2 (M5), Y = X C on X's own pattern (M6),
C on the projected pattern with entries only where supports overlap (M7),
weak-scaling lattice offset of half a spacing (M8), reference Hilbert
partition (M9).  The potential is -sum_c exp(-|x-c|^2/sigma^2) over all
centres.  Inputs are synthetic (no public dataset exists for this path).

Fills are vectorised: one hash per support entry written straight to its
storage offset, identical to the reference's masked per-block `np.isin`
fill.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
from scipy import sparse

from .bcsr import BlockCsrMatrix, _IndexList
from .blocks import BlockSparsityPattern
from .energy import column_space_ghost_blocks, make_column_layout, projected_pattern
from .localization import (
    build_support_sparsity,
    column_supports,
    grow_sparsity_for_operator,
    order_and_block_columns,
    patch_fine_cells,
)
from .matfree import CellOperator, GaussianPotential, make_dof_layout, hamiltonian_operator
from .mesh import build_mesh, cells_nodes, enumerate_dofs, partition_and_order_cells
from .support import ColumnSupport, attach_support

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def hashed_entries(seed: int, rows, cols) -> np.ndarray:
    """Elementwise hashed value in [-0.5, 0.5) of (seed, row, col) triples."""
    r = np.asarray(rows, dtype=np.int64).astype(np.uint64)
    c = np.asarray(cols, dtype=np.int64).astype(np.uint64)
    with np.errstate(over="ignore"):
        h = _mix64(r * np.uint64(0x9E3779B97F4A7C15) + c * np.uint64(0xD1B54A32D192ED03)
                   + np.uint64(seed & 0xFFFFFFFFFFFFFFFF))
    return h.astype(np.float64) / float(2**64) - 0.5


def hashed_values(seed: int, rows, cols) -> np.ndarray:
    """Outer-product form (rows x cols), same values as the reference helper."""
    r = np.asarray(rows, dtype=np.int64)
    c = np.asarray(cols, dtype=np.int64)
    return hashed_entries(seed, np.repeat(r, c.size), np.tile(c, r.size)).reshape(r.size, c.size)


@dataclass
class ProblemConfig:
    name: str
    extents: tuple
    degree: int
    centers: np.ndarray
    radius: float
    sigma: float
    spacing: tuple | None = None
    dirichlet: bool = False
    kernels: tuple = ("apply_h",)
    block_size: int = 8
    lane_width: int = 8
    vectors_per_center: int = 1
    coarse_level: int = 0
    seed_x: int = 1
    seed_y: int = 2
    seed_c: int = 7
    note: str = ""

    def __post_init__(self):
        if self.spacing is None:
            self.spacing = tuple(1.0 / self.extents[0] for _ in range(3))


def lattice(counts, spacing, offset) -> np.ndarray:
    """Centres offset + spacing * (i, j, k), x fastest."""
    nx, ny, nz = counts
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    ijk = np.stack([i.ravel(), j.ravel(), k.ravel()], axis=1).astype(float)
    return np.asarray(offset, dtype=float) + ijk * np.asarray(spacing, dtype=float)


def baseline_config(name: str, n_ranks: int = 1) -> ProblemConfig:
    """BASELINE.json configs[0..4] ('smoke', 'q2', 'q4', 'proj', 'weak')."""
    if name == "smoke":
        c = lattice((2, 2, 2), 0.5, 0.25)
        return ProblemConfig("smoke", (8, 8, 8), 2, c, 0.3, 0.2, dirichlet=True,
                             kernels=("apply_h", "tmmult", "mmult"),
                             note="CPU-oracle smoke: 8^3 Q2, M=8, r=0.3, sigma=0.2")
    if name in ("q2", "q4"):
        c = lattice((4, 4, 4), 0.25, 0.125)
        deg = 2 if name == "q2" else 4
        return ProblemConfig(name, (32, 32, 32), deg, c, 0.25, 0.1,
                             note=f"32^3 Q{deg}, M=64 lattice 0.25 offset 0.125, r=0.25, sigma=0.1")
    if name == "proj":
        c = lattice((8, 8, 8), 1.0 / 8, 1.0 / 16)
        return ProblemConfig("proj", (64, 64, 64), 2, c, 1.5 / 8, 0.1,
                             kernels=("apply_h", "tmmult", "mmult"),
                             note="64^3 Q2, M=512 lattice 1/8, r=1.5/8, sigma=0.1")
    if name.startswith("weak"):
        g = int(name[4:]) if len(name) > 4 else int(n_ranks)
        h = 1.0 / 64
        c = lattice((8, 8, 8 * g), 8 * h, 4 * h)
        return ProblemConfig(f"weak{g}", (64, 64, 64 * g), 4, c, 8 * h, 2 * h,
                             spacing=(h, h, h), kernels=("apply_h", "tmmult", "mmult"),
                             note=f"weak G={g}: 64x64x{64 * g} Q4, M={512 * g}, r=8h, sigma=2h")
    raise ValueError(f"unknown config {name!r}")


@dataclass
class Problem:
    cfg: ProblemConfig
    mesh: object
    partition: object
    numbering: object
    loc_layout: object
    supports: list
    pattern: BlockSparsityPattern
    grown: BlockSparsityPattern
    potential: GaussianPotential
    n_ranks: int
    _proj: BlockSparsityPattern | None = None
    _support: ColumnSupport | None = None
    _overlap: sparse.csr_matrix | None = None
    extra: dict = field(default_factory=dict)

    @property
    def proj_pattern(self) -> BlockSparsityPattern:
        if self._proj is None:
            self._proj = projected_pattern(self.pattern, self.grown)
        return self._proj

    @property
    def column_support(self) -> ColumnSupport:
        if self._support is None:
            self._support = ColumnSupport.from_localization(self.loc_layout, self.supports,
                                                            self.numbering.n_dofs)
        return self._support

    def spec_h(self):
        return hamiltonian_operator(self.potential)

    def support_overlap(self) -> sparse.csr_matrix:
        """(M x M) bool CSR, new column order: True where two supports share a row.

        Supports are the nodes of cell patches; two node sets intersect iff a
        cell of one patch and a cell of the other share a node, i.e. iff the
        one-cell dilation of the first patch meets the second.  Candidate
        pairs are pruned by centre distance, then tested exactly on cell ids.
        """
        if self._overlap is not None:
            return self._overlap
        lay = self.loc_layout
        mesh = self.mesh
        nc = lay.centers.shape[0]
        nx, ny, nz = mesh.extents
        patches = [patch_fine_cells(mesh, lay, c) for c in range(nc)]
        plen = np.asarray([p_.size for p_ in patches], dtype=np.int64)
        n_cells = mesh.n_cells
        pmat = sparse.csr_matrix(
            (np.ones(int(plen.sum()), dtype=np.int32),
             np.concatenate(patches) if nc else np.zeros(0, dtype=np.int64),
             np.concatenate([[0], np.cumsum(plen)])), shape=(nc, n_cells))
        pmat.sum_duplicates()
        pmat.data[:] = 1
        # cell adjacency (27-point, cells sharing a node) as a sparse matrix
        ijk = mesh.cells_ijk(np.arange(n_cells))
        rows_a, cols_a = [], []
        for dz in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    q = ijk + np.asarray([dx, dy, dz])
                    ok = ((q[:, 0] >= 0) & (q[:, 0] < nx) & (q[:, 1] >= 0) & (q[:, 1] < ny)
                          & (q[:, 2] >= 0) & (q[:, 2] < nz))
                    rows_a.append(np.flatnonzero(ok))
                    qo = q[ok]
                    cols_a.append(qo[:, 0] + nx * (qo[:, 1] + ny * qo[:, 2]))
        adj = sparse.csr_matrix((np.ones(sum(r.size for r in rows_a), dtype=np.int32),
                                 (np.concatenate(rows_a), np.concatenate(cols_a))),
                                shape=(n_cells, n_cells))
        touch = ((pmat @ adj) @ pmat.T).tocoo()  # patch a dilated by one cell meets patch b
        rr = [np.arange(nc), touch.row.astype(np.int64)]
        cc = [np.arange(nc), touch.col.astype(np.int64)]
        r_c = np.concatenate(rr)
        c_c = np.concatenate(cc)
        v = lay.vectors_per_center
        new_of_center = lay.new_col_of_old.reshape(nc, v)
        rr = np.repeat(new_of_center[r_c], v, axis=1).ravel()
        cc = np.tile(new_of_center[c_c], (1, v)).ravel()
        out = sparse.csr_matrix((np.ones(rr.size, dtype=bool), (rr, cc)), shape=(nc * v, nc * v))
        out.sum_duplicates()
        out.sort_indices()
        self._overlap = out
        return out


def build_problem(cfg: ProblemConfig | str, n_ranks: int = 1) -> Problem:
    if isinstance(cfg, str):
        cfg = baseline_config(cfg, n_ranks)
    mesh = build_mesh(cfg.extents, cfg.spacing, cfg.coarse_level)
    partition = partition_and_order_cells(mesh, n_ranks)
    numbering = enumerate_dofs(mesh, partition, cfg.degree)
    lay = order_and_block_columns(mesh, partition, cfg.centers, cfg.radius,
                                  cfg.vectors_per_center, cfg.block_size)
    supports = column_supports(mesh, numbering, lay)
    pattern = build_support_sparsity(mesh, partition, numbering, lay, supports)
    grown = grow_sparsity_for_operator(pattern, mesh, numbering)
    pot = GaussianPotential(cfg.centers, cfg.sigma, -1.0)
    return Problem(cfg, mesh, partition, numbering, lay, supports, pattern, grown, pot, n_ranks)


def _support_entries(matrix: BlockCsrMatrix, prob: Problem):
    """(flat offsets, global rows, new cols) of the support entries in owned rows."""
    return prob.column_support.owned_entries(matrix)


def fill_multivector(matrix: BlockCsrMatrix, prob: Problem, seed: int, attach: bool = True):
    """X[r, c] = 2 * hash(seed, r, old(c)) on the support of c, else 0 (owned rows).

    With `attach` (default) the matrix is (re)laid out to store exactly the
    support's columns (support.attach_support; slabs.py) and the values go up
    as the compact support vector (8 bytes per structural nonzero), scattered
    on the device.  Equals the reference's masked per-block fill
    (`bench/problem.py:113-131`) on every stored entry.
    """
    import torch

    from . import _plan

    matrix._require("owned-writable")
    sup = prob.column_support
    if attach and matrix.support is not sup:
        matrix.relayout(sup)
    flat, rows, cols = sup.owned_entries(matrix)
    old = prob.loc_layout.old_col_of_new
    if _plan.enabled():
        vals = _plan.hash_fill(seed, rows, cols, old, None, 2.0)
    else:
        vals = 2.0 * hashed_entries(seed, rows, old[cols])
    if attach:
        matrix.upload_support_values(torch.from_numpy(vals))
    else:
        _zero_owned(matrix)
        matrix._write_host(flat, vals)
    return matrix


def _zero_owned(matrix: BlockCsrMatrix):
    from .bcsr import _zero_range

    _zero_range(matrix.data, 0, matrix.n_owned_values)


def fill_projected(matrix: BlockCsrMatrix, prob: Problem, seed: int):
    """C[a, b] = 2 * hash(seed, old(a), old(b)) where supports of a, b overlap."""
    old = prob.loc_layout.old_col_of_new
    ov = prob.support_overlap()

    def values(grow, gcol):
        v = 2.0 * hashed_entries(seed, old[grow], old[gcol])
        key = grow * ov.shape[1] + gcol
        okeys = np.repeat(np.arange(ov.shape[0], dtype=np.int64), np.diff(ov.indptr)) * ov.shape[1] \
            + ov.indices
        pos = np.searchsorted(okeys, key)
        hit = (pos < okeys.size) & (okeys[np.minimum(pos, okeys.size - 1)] == key)
        return np.where(hit, v, 0.0)

    matrix.fill_owned_entries(values)
    return matrix


def dirichlet_rows(prob: Problem) -> np.ndarray:
    """Global rows of the nodes on the boundary of the box."""
    mesh, p = prob.mesh, prob.numbering.degree
    sx, sy, sz = mesh.node_grid_shape(p)
    k, j, i = np.meshgrid(np.arange(sz), np.arange(sy), np.arange(sx), indexing="ij")
    bnd = ((i == 0) | (i == sx - 1) | (j == 0) | (j == sy - 1) | (k == 0) | (k == sz - 1)).ravel()
    return np.sort(prob.numbering.new_index_of_node[np.flatnonzero(bnd)])


class DirichletMask:
    """Zero the boundary rows of a multivector (optional mask)."""

    def __init__(self, matrix: BlockCsrMatrix, rows: np.ndarray):
        lo, hi = matrix.layout.owned_rows
        rows = np.asarray(rows, dtype=np.int64)
        rows = rows[(rows >= lo) & (rows < hi)]
        lb, rib = matrix.layout.map_rows(rows)
        sg = matrix.slab
        k = sg.width[lb]
        owner = np.repeat(np.arange(lb.size, dtype=np.int64), k)
        first = np.concatenate([[0], np.cumsum(k)])[:-1]
        idx = sg.off[lb][owner] + rib[owner] * k[owner] + (np.arange(int(k.sum())) - first[owner])
        self.index = _IndexList(idx.astype(np.int64), matrix.device)
        self._zeros = None

    def apply(self, matrix: BlockCsrMatrix):
        import torch

        if self._zeros is None or self._zeros.device != matrix.data.device:
            self._zeros = torch.zeros(self.index.size, dtype=torch.float64, device=matrix.data.device)
        self.index.scatter(self._zeros, matrix.data, add=False)


@dataclass
class RankSetup:
    """Per-rank operands of one workload."""

    prob: Problem
    ctx: object
    layout: object
    op: CellOperator
    x: BlockCsrMatrix
    hx: BlockCsrMatrix
    y: BlockCsrMatrix | None = None
    hy: BlockCsrMatrix | None = None
    s: BlockCsrMatrix | None = None
    c: BlockCsrMatrix | None = None
    xc: BlockCsrMatrix | None = None
    dirichlet: tuple | None = None


def make_rank_setup(ctx, prob: Problem, projection: bool | None = None, device=None,
                    with_y: bool | None = None, compact_xc: bool = True) -> RankSetup:
    """Operands of one workload on this rank, in slab storage (slabs.py):
    X (and Y) store their support columns, H X (H Y) the operator image of
    that support, S and C (projected pattern) every column of their blocks,
    X C the support columns of X (X's own storage; compact_xc=False
    keeps the reference's block-level truncation instead)."""
    cfg = prob.cfg
    layout = make_dof_layout(ctx, prob.mesh, prob.partition, prob.numbering)
    op = CellOperator(prob.mesh, prob.partition, prob.numbering, layout)
    w = cfg.lane_width
    sup = prob.column_support
    img = op.image_columns(sup)
    x = fill_multivector(BlockCsrMatrix(prob.pattern, layout, ctx, w, device, columns=sup),
                         prob, cfg.seed_x)
    hx = BlockCsrMatrix(prob.grown, layout, ctx, w, device, columns=img)
    st = RankSetup(prob, ctx, layout, op, x, hx)
    if cfg.dirichlet:
        rows = dirichlet_rows(prob)
        st.dirichlet = (DirichletMask(x, rows), DirichletMask(hx, rows))
    if projection is None:
        projection = "tmmult" in cfg.kernels or "mmult" in cfg.kernels
    if projection:
        lay = prob.loc_layout
        proj = prob.proj_pattern
        ghosts = column_space_ghost_blocks(prob.grown, proj, layout, lay.rank_block_start, ctx.rank)
        clayout = make_column_layout(ctx, lay.column_blocks, lay.rank_block_start, ghosts)
        if with_y is None:
            with_y = cfg.name == "proj"
        if with_y:
            st.y = fill_multivector(BlockCsrMatrix(prob.pattern, layout, ctx, w, device,
                                                   columns=sup), prob, cfg.seed_y)
            st.hy = BlockCsrMatrix(prob.grown, layout, ctx, w, device, columns=img)
        st.s = BlockCsrMatrix(proj, clayout, ctx, w, device)
        st.c = fill_projected(BlockCsrMatrix(proj, clayout, ctx, w, device), prob, cfg.seed_c)
        st.xc = BlockCsrMatrix(prob.pattern, layout, ctx, w, device,
                               columns=sup if compact_xc else None)
    return st
