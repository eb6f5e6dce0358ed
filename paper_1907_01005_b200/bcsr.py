"""Block-CSR multivectors resident in GPU memory, ghost exchange, SpMM.

Drop-in for the reference `bcsrmv/bcsr.py` (same names, signatures, state
machine and errors).  What changes is where the values live and who
computes:

* `BlockCsrMatrix.data` is a torch float64 tensor on the rank's GPU in SLAB
  layout (slabs.py) instead of the reference's padded per-block arrays
  (`bcsr.py:233-318`): each local block row stores one row-major
  rows x K slab over its stored columns, owned block rows then ghosts.  By
  default the stored columns are every column of the row's stored blocks
  (the reference's storage set, without the lane padding); a matrix built
  with `columns=` a column support (support.py) or an operator image
  (matfree.ImageColumns) stores only the active ones -- 1.1-1.2x the
  structural nonzeros of the BASELINE multivectors instead of 3.5-4.8x.
  `value_bytes` / `load_value_bytes` convert to and from the reference's
  byte layout; `block_values(pos)` is a (rows x block columns) view when the
  block stores all its columns, else a dense copy.
* ghost update / compress (`bcsr.py:401-519`) pack and unpack whole slab
  rows with the libbmv gather/scatter kernels and move buffers with the
  rank context (NCCL point-to-point between GPUs); compress adds in
  ascending source rank order, like the reference.
* `tmmult` / `mmult` (`bcsr.py:587-667`) run the K4 / K5 chunk kernels
  (csrc/bmv_spmm.cu, plans in spmm.py).
* the OM glue (`scale_add`, `copy_pattern_subset`, `add_scaled_identity`,
  `tr_tmmult`, `tr_mult`; `bcsr.py:526-577,670-725`) runs as element-wise
  device ops on cached index maps.

Matrices may also live on the CPU (`device="cpu"`): layout and exchange
logic then run with torch index ops so the multi-rank protocol can be
tested with gloo, but every compute kernel refuses CPU storage
(DeviceError) -- there is no CPU fallback of the operator path.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, _plan, spmm
from .blocks import BlockIndices, BlockSparsityPattern
from .counters import OpCounters
from .slabs import FULL, SlabGeometry
from .errors import (
    ConsistencyError,
    DomainError,
    PatternError,
    ProtocolError,
    ShapeError,
    StateError,
)

OWNED = "owned-writable"
GHOSTED = "ghost-readable"
GHOST_XCHG = "ghost-update-in-flight"
COMPRESS_XCHG = "compress-in-flight"


def default_device():
    if torch.cuda.is_available():
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def group_rows_by_block(rows, blocks: BlockIndices) -> list:
    """(block id, sorted rows) groups, ascending block order."""
    rows = np.unique(np.asarray(rows, dtype=np.int64))
    if rows.size == 0:
        return []
    b = blocks.blocks_of(rows)
    cut = np.flatnonzero(np.diff(b)) + 1
    return [(int(bb[0]), rr) for bb, rr in zip(np.split(b, cut), np.split(rows, cut))]


@dataclass(frozen=True)
class GhostGroup:
    owner: int
    block: int
    rows: np.ndarray
    rows_in_block: np.ndarray


@dataclass(frozen=True)
class ImportGroup:
    peer: int
    block: int
    rows_in_block: np.ndarray


class RankLayout:
    """Row ownership of one rank, its ghost groups and export plan."""

    def __init__(self, rank, n_ranks, blocks, rank_block_start, ghost_groups, import_groups):
        self.rank = int(rank)
        self.n_ranks = int(n_ranks)
        self.blocks = blocks
        self.rank_block_start = np.asarray(rank_block_start, dtype=np.int64)
        self.ghost_groups = list(ghost_groups)
        self.import_groups = list(import_groups)
        self.first_block = int(self.rank_block_start[rank])
        self.n_owned_blocks = int(self.rank_block_start[rank + 1]) - self.first_block
        self.owned_rows = (int(blocks.starts[self.first_block]),
                           int(blocks.starts[self.first_block + self.n_owned_blocks]))
        self._ghost_local = {g.block: self.n_owned_blocks + i for i, g in enumerate(self.ghost_groups)}
        if self.ghost_groups:
            self.ghost_rows_flat = np.concatenate([g.rows for g in self.ghost_groups])
            counts = np.asarray([len(g.rows) for g in self.ghost_groups], dtype=np.int64)
        else:
            self.ghost_rows_flat = np.zeros(0, dtype=np.int64)
            counts = np.zeros(0, dtype=np.int64)
        self.ghost_offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)

    @property
    def n_local_blocks(self) -> int:
        return self.n_owned_blocks + len(self.ghost_groups)

    @property
    def n_local_rows(self) -> int:
        return (self.owned_rows[1] - self.owned_rows[0]) + int(self.ghost_rows_flat.size)

    def owner_of_block(self, gb: int) -> int:
        return int(np.searchsorted(self.rank_block_start, gb, side="right")) - 1

    def owns_block(self, gb: int) -> bool:
        return self.first_block <= gb < self.first_block + self.n_owned_blocks

    def local_block_of_global(self, gb: int) -> int:
        if self.owns_block(gb):
            return gb - self.first_block
        lb = self._ghost_local.get(int(gb))
        if lb is None:
            raise PatternError(f"rank {self.rank} holds no ghost of block row {gb}")
        return lb

    def global_block_of_local(self, lb: int) -> int:
        if lb < self.n_owned_blocks:
            return self.first_block + lb
        return self.ghost_groups[lb - self.n_owned_blocks].block

    def global_blocks_of_locals(self) -> np.ndarray:
        ghosts = np.asarray([g.block for g in self.ghost_groups], dtype=np.int64)
        return np.concatenate([np.arange(self.first_block, self.first_block + self.n_owned_blocks,
                                         dtype=np.int64), ghosts])

    def local_row_count(self, lb: int) -> int:
        if lb < self.n_owned_blocks:
            return self.blocks.block_size(self.first_block + lb)
        return len(self.ghost_groups[lb - self.n_owned_blocks].rows)

    def local_row_counts(self) -> np.ndarray:
        own = self.blocks.sizes[self.first_block : self.first_block + self.n_owned_blocks]
        return np.concatenate([own, np.diff(self.ghost_offsets)]).astype(np.int64)

    def map_rows(self, rows):
        """(local block, row in block) of global rows; ConsistencyError if unmapped."""
        rows = np.asarray(rows, dtype=np.int64)
        lb = np.empty(rows.shape, dtype=np.int64)
        rib = np.empty(rows.shape, dtype=np.int64)
        lo, hi = self.owned_rows
        own = (rows >= lo) & (rows < hi)
        if own.all() and rows.size > 100_000 and _plan.enabled():
            g, rib = _plan.blocks_of(self.blocks.starts, rows)  # native, OpenMP
            return g - self.first_block, rib
        if own.any():
            g = self.blocks.blocks_of(rows[own])
            lb[own] = g - self.first_block
            rib[own] = rows[own] - self.blocks.starts[g]
        rest = ~own
        if rest.any():
            r = rows[rest]
            flat = self.ghost_rows_flat
            if flat.size == 0:
                raise ConsistencyError(f"rank {self.rank} touches unmapped row {int(r.flat[0])}")
            pos = np.searchsorted(flat, r)
            bad = (pos >= flat.size) | (flat[np.minimum(pos, flat.size - 1)] != r)
            if bad.any():
                raise ConsistencyError(f"rank {self.rank} touches unmapped row {int(r[bad].flat[0])}")
            grp = np.searchsorted(self.ghost_offsets, pos, side="right") - 1
            lb[rest] = self.n_owned_blocks + grp
            rib[rest] = pos - self.ghost_offsets[grp]
        return lb, rib


def serial_layout(blocks: BlockIndices) -> RankLayout:
    return RankLayout(0, 1, blocks, [0, blocks.n_blocks], [], [])


def build_rank_layout(ctx, blocks: BlockIndices, rank_block_start, ghost_rows) -> RankLayout:
    """Collective: group ghost rows by owner block, request them, verify echoes.

    Same two-message protocol as the reference (`bcsr.py:159-230`) so a
    malformed request raises ProtocolError on the owner.
    """
    rank_block_start = np.asarray(rank_block_start, dtype=np.int64)
    me = ctx.rank
    lid = ctx.next_matrix_id()
    ghost_groups, per_owner = [], {}
    for block, rows in group_rows_by_block(ghost_rows, blocks):
        owner = int(np.searchsorted(rank_block_start, block, side="right")) - 1
        if owner == me:
            raise ConsistencyError(f"rank {me} lists its own row as ghost")
        ghost_groups.append(GhostGroup(owner, block, rows, rows - blocks.starts[block]))
        per_owner.setdefault(owner, []).append((block, rows))
    for peer in range(ctx.n_ranks):
        if peer != me:
            req = per_owner.get(peer, [])
            ctx.isend(peer, ("ghost_req", lid),
                      (np.asarray([b for b, _ in req], dtype=np.int64), [r for _, r in req]))
    import_groups, echoes = [], {}
    for peer in range(ctx.n_ranks):
        if peer == me:
            continue
        req_blocks, req_rows = ctx.irecv(peer, ("ghost_req", lid)).wait()
        for b, rows in zip(req_blocks, req_rows):
            b = int(b)
            lo, hi = int(blocks.starts[b]), int(blocks.starts[b + 1])
            owner = int(np.searchsorted(rank_block_start, b, side="right")) - 1
            rows = np.asarray(rows, dtype=np.int64)
            if owner != me or rows.min() < lo or rows.max() >= hi:
                raise ProtocolError(f"rank {me}: peer {peer} requested rows outside my block {b}")
            import_groups.append(ImportGroup(peer, b, rows - lo))
        echoes[peer] = (np.asarray(req_blocks, dtype=np.int64).copy(),
                        np.asarray([len(r) for r in req_rows], dtype=np.int64))
    for peer, echo in echoes.items():
        ctx.isend(peer, ("ghost_ack", lid), echo)
    for peer in range(ctx.n_ranks):
        if peer == me:
            continue
        b_echo, c_echo = ctx.irecv(peer, ("ghost_ack", lid)).wait()
        req = per_owner.get(peer, [])
        if not (np.array_equal(b_echo, np.asarray([b for b, _ in req], dtype=np.int64))
                and np.array_equal(c_echo, np.asarray([len(r) for _, r in req], dtype=np.int64))):
            raise ProtocolError(f"rank {me}: ghost plan with rank {peer} is inconsistent")
    import_groups.sort(key=lambda g: (g.peer, g.block))
    return RankLayout(me, ctx.n_ranks, blocks, rank_block_start, ghost_groups, import_groups)


class _IndexList:
    """Element index list; a libbmv device plan for CUDA data, a tensor on CPU."""

    def __init__(self, idx: np.ndarray, device):
        self.size = int(idx.size)
        self.device = torch.device(device)
        if self.device.type == "cuda":
            lib = _lib.load()
            raw = _lib.C.c_void_p()
            arr = np.ascontiguousarray(idx, dtype=np.int64)
            _lib.check(lib.bmv_index_create(_lib.ptr(arr, _lib.C.c_int64), arr.size,
                                            _lib.C.byref(raw)), "bmv_index_create")
            self.handle = _lib.Handle("bmv_index_destroy", raw)
            self.tensor = None
        else:
            self.handle = None
            self.tensor = torch.from_numpy(np.ascontiguousarray(idx, dtype=np.int64))

    def gather(self, src: torch.Tensor) -> torch.Tensor:
        if self.handle is None:
            return src[self.tensor].clone()
        out = torch.empty(self.size, dtype=torch.float64, device=src.device)
        if self.size:
            _lib.check(_lib.load().bmv_gather(self.handle.raw, _lib.dptr(src), _lib.dptr(out),
                                              _lib.stream_handle(src.device)), "bmv_gather")
        return out

    def scatter(self, buf: torch.Tensor, dst: torch.Tensor, add: bool):
        if self.size == 0:
            return
        if self.handle is None:
            if add:
                dst.index_add_(0, self.tensor, buf)
            else:
                dst[self.tensor] = buf
            return
        _lib.check(_lib.load().bmv_scatter(self.handle.raw, _lib.dptr(buf), _lib.dptr(dst),
                                           1 if add else 0, _lib.stream_handle(dst.device)),
                   "bmv_scatter")


def _zero_range(data: torch.Tensor, begin: int, end: int):
    if end <= begin:
        return
    if data.is_cuda:
        view = data[begin:end]
        _lib.check(_lib.load().bmv_zero(_lib.dptr(view), end - begin,
                                        _lib.stream_handle(data.device)), "bmv_zero")
    else:
        data[begin:end] = 0.0


def _local_block_table(layout: RankLayout, n_global: int) -> np.ndarray:
    """Local block id of every global block (-1 when neither owned nor ghost)."""
    tab = np.full(n_global, -1, dtype=np.int64)
    gl = layout.global_blocks_of_locals()
    tab[gl] = np.arange(gl.size, dtype=np.int64)
    return tab


class BlockCsrMatrix:
    """Rank-local BCSR matrix; values on the GPU in slab layout (slabs.py).

    `columns` selects the stored columns of every block row: None = all
    columns of the stored blocks (the reference's storage set), a
    ColumnSupport = the columns its support reaches (entries outside it are
    structural zeros, `.support` keeps the entry-level declaration), or any
    object with `columns_for(pattern, global_blocks)` (matfree.ImageColumns).
    """

    def __init__(self, pattern: BlockSparsityPattern, layout: RankLayout, ctx=None,
                 lane_width: int = 8, device=None, columns=None):
        if pattern.row_blocks != layout.blocks:
            raise ShapeError("pattern row blocking does not match the layout")
        if lane_width < 1:
            raise DomainError("lane width must be positive")
        if ctx is None and layout.n_ranks > 1:
            raise ShapeError("multi-rank matrices need a rank context")
        self.pattern = pattern
        self.layout = layout
        self.ctx = ctx
        self.lane_width = int(lane_width)
        self.col_blocks = pattern.col_blocks
        w = self.lane_width
        # the reference's padded block widths (value_bytes / load_value_bytes format)
        self.col_strides = ((self.col_blocks.sizes + w - 1) // w * w).astype(np.int64)
        gblocks = layout.global_blocks_of_locals()
        counts = (pattern.row_start[gblocks + 1] - pattern.row_start[gblocks]).astype(np.int64)
        self.local_row_sizes = layout.local_row_counts()
        self.row_start = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        if gblocks.size:
            starts = pattern.row_start[gblocks]
            idx = np.repeat(starts - self.row_start[:-1], counts) + np.arange(int(self.row_start[-1]))
            self.col_index = pattern.col_index[idx].astype(np.int64)
        else:
            self.col_index = np.zeros(0, dtype=np.int64)
        self.pos_row = np.repeat(np.arange(gblocks.size, dtype=np.int64), counts)
        if device is None:
            device = getattr(ctx, "device", None) or default_device()
        self.device = torch.device(device)
        self._set_geometry(columns)
        self.data = torch.zeros(int(self.slab.off[-1]), dtype=torch.float64, device=self.device)
        self.state = OWNED
        self._mid = ctx.next_matrix_id() if ctx is not None else 0
        self._pending = None
        self._xplan = None

    # -- geometry ----------------------------------------------------------------

    def _set_geometry(self, columns):
        from .support import ColumnSupport

        spec = FULL if columns is None else columns
        if isinstance(spec, ColumnSupport) and spec.n_cols != self.col_blocks.total:
            raise ConsistencyError("support column count differs from the matrix")
        self.columns = spec
        self.support = spec if isinstance(spec, ColumnSupport) else None
        ptr, cols = spec.columns_for(self.pattern, self.layout.global_blocks_of_locals())
        self.slab = SlabGeometry(ptr, cols, self.local_row_sizes, self.row_start, self.col_index,
                                 self.col_blocks, self.layout.n_owned_blocks)
        self.block_offsets = self.slab.block_offsets
        self._ghost_data_begin = self.slab.ghost_begin
        self._xplan = None
        self._plans = {}

    def relayout(self, columns):
        """Store `columns` instead (slabs.py); values of columns stored in both
        layouts are kept, the others dropped."""
        if columns is self.columns:
            return self
        old_slab, old = self.slab, self.data
        self._set_geometry(columns)
        new = torch.zeros(int(self.slab.off[-1]), dtype=torch.float64, device=self.device)
        n_loc = self.layout.n_local_blocks
        off, lb, r, s = self.slab.block_entries(np.arange(n_loc), self.local_row_sizes)
        gcol = self.slab.cols[self.slab.ptr[lb] + s]
        src = old_slab.offsets(lb, r, gcol)
        ok = src >= 0
        if ok.any():
            di = torch.as_tensor(off[ok], device=self.device)
            si = torch.as_tensor(src[ok], device=self.device)
            new[di] = old[si]
        self.data = new
        return self

    # -- views and metadata ---------------------------------------------------

    @property
    def n_owned_blocks(self) -> int:
        return self.layout.n_owned_blocks

    @property
    def n_local_blocks(self) -> int:
        return self.layout.n_local_blocks

    @property
    def n_owned_values(self) -> int:
        return self._ghost_data_begin

    def row_cols_local(self, lb: int) -> np.ndarray:
        return self.col_index[self.row_start[lb] : self.row_start[lb + 1]]

    def block_values(self, pos: int) -> torch.Tensor:
        """(rows x block columns): a view when the block stores every column,
        else a dense copy with zeros in the columns it does not store."""
        lb = int(self.pos_row[pos])
        rows = int(self.local_row_sizes[lb])
        cb = int(self.col_index[pos])
        size = int(self.col_blocks.sizes[cb])
        k = int(self.slab.width[lb])
        off = int(self.slab.block_offsets[pos])
        ns = int(self.slab.pos_nslot[pos])
        view = self.data.as_strided((rows, ns), (k, 1), self.data.storage_offset() + off)
        if self.slab.pos_full[pos]:
            return view
        out = torch.zeros(rows, size, dtype=torch.float64, device=self.device)
        s0 = int(self.slab.ptr[lb] + self.slab.pos_slot[pos])
        lanes = self.slab.cols[s0 : s0 + ns] - self.col_blocks.starts[cb]
        out[:, torch.as_tensor(lanes, device=self.device)] = view
        return out

    def block_valid(self, pos: int) -> torch.Tensor:
        return self.block_values(pos)

    def block_pos_local(self, lb: int, col: int) -> int:
        lo, hi = int(self.row_start[lb]), int(self.row_start[lb + 1])
        k = lo + int(np.searchsorted(self.col_index[lo:hi], col))
        if k < hi and self.col_index[k] == col:
            return k
        return -1

    def local_keys(self) -> np.ndarray:
        """Sorted keys local_block * n_col_blocks + col of the stored blocks."""
        return self.pos_row * self.col_blocks.n_blocks + self.col_index

    def _require(self, *states):
        if self.state not in states:
            raise StateError(f"operation requires state in {states}, matrix is {self.state}")

    def ensure_owned(self):
        if self.state == GHOSTED:
            self.release_ghosts()
        else:
            self._require(OWNED)

    def _owned_local(self, grow: np.ndarray):
        """(local block, row in block) of owned global rows."""
        lay = self.layout
        g = lay.blocks.blocks_of(grow)
        return g - lay.first_block, grow - lay.blocks.starts[g]

    def _valid_owned_index(self):
        """(flat offsets, global rows, global cols) of every owned stored entry."""
        n_own = self.n_owned_blocks
        if n_own == 0:
            z = np.zeros(0, dtype=np.int64)
            return z, z, z
        off, lb, r, s = self.slab.block_entries(np.arange(n_own), self.local_row_sizes[:n_own])
        grow = self.layout.blocks.starts[self.layout.first_block + lb] + r
        gcol = self.slab.cols[self.slab.ptr[lb] + s]
        return off, grow, gcol

    # -- elementwise ---------------------------------------------------------------

    def zero_out(self):
        self._require(OWNED)
        _zero_range(self.data, 0, self.data.numel())

    def zero_ghost_blocks(self):
        _zero_range(self.data, self._ghost_data_begin, self.data.numel())

    def release_ghosts(self):
        self._require(GHOSTED)
        self.zero_ghost_blocks()
        self.state = OWNED

    def copy(self) -> "BlockCsrMatrix":
        """Same pattern, layout and stored columns (so the same structural
        zeros: a support declaration is part of the storage), values copied."""
        out = BlockCsrMatrix.__new__(BlockCsrMatrix)
        out.__dict__.update(self.__dict__)
        out.data = self.data.clone()
        out._pending = None
        out._plans = {}
        return out

    def _write_host(self, flat: np.ndarray, vals: np.ndarray):
        if flat.size:
            self.data[torch.as_tensor(flat, device=self.device)] = \
                torch.as_tensor(np.asarray(vals, dtype=np.float64), device=self.device)

    def fill_owned(self, fn):
        """Set every owned block to fn(global_rows, global_cols) (host callback);
        values of columns the block does not store must be 0."""
        self._require(OWNED)
        flat, vals = [], []
        for pos in range(int(self.row_start[self.n_owned_blocks])):
            lb = int(self.pos_row[pos])
            gb = self.layout.global_block_of_local(lb)
            r0 = int(self.layout.blocks.starts[gb])
            rows = np.arange(r0, r0 + int(self.local_row_sizes[lb]))
            c = int(self.col_index[pos])
            c0 = int(self.col_blocks.starts[c])
            cols = np.arange(c0, c0 + int(self.col_blocks.sizes[c]))
            v = np.asarray(fn(rows, cols), dtype=np.float64).reshape(rows.size, cols.size)
            s0 = int(self.slab.ptr[lb] + self.slab.pos_slot[pos])
            ns = int(self.slab.pos_nslot[pos])
            lanes = self.slab.cols[s0 : s0 + ns] - c0
            keep = np.zeros(cols.size, dtype=bool)
            keep[lanes] = True
            if np.any(v[:, ~keep] != 0.0):
                raise ConsistencyError(f"fill_owned: nonzero value in a column block {c} "
                                       f"column that block row {gb} does not store")
            k = int(self.slab.width[lb])
            base = int(self.slab.block_offsets[pos])
            flat.append((base + np.arange(rows.size)[:, None] * k + np.arange(ns)[None, :]).ravel())
            vals.append(v[:, lanes].ravel())
        if flat:
            self._write_host(np.concatenate(flat), np.concatenate(vals))
        self.support = None

    def fill_owned_entries(self, fn_flat):
        """Vectorised fill: fn_flat(global_rows, global_cols) -> values per stored entry."""
        self._require(OWNED)
        flat, grow, gcol = self._valid_owned_index()
        if flat.size == 0:
            return
        self._write_host(flat, fn_flat(grow, gcol))
        self.support = None

    def to_dense_owned(self) -> np.ndarray:
        out = np.zeros((self.layout.blocks.total, self.col_blocks.total))
        flat, grow, gcol = self._valid_owned_index()
        if flat.size:
            host = self.data.detach().cpu().numpy()
            out[grow, gcol] = host[flat]
        return out

    def norm_owned_sq(self) -> float:
        v = self.data[: self._ghost_data_begin]
        return float(torch.dot(v, v).item())

    def _entry_offset(self, row: int, col: int):
        lb, rib = self.layout.map_rows([row])
        cb, _ = self.col_blocks.global_to_block(col)
        if self.block_pos_local(int(lb[0]), cb) < 0:
            return None, False
        off = int(self.slab.offsets(lb, rib, [col])[0])
        return (None if off < 0 else off), True

    def get_entry(self, row: int, col: int) -> float:
        off, _ = self._entry_offset(row, col)
        return 0.0 if off is None else float(self.data[off].item())

    def add_entry(self, row: int, col: int, value: float):
        off, block = self._entry_offset(row, col)
        if not block:
            raise PatternError(f"block for entry ({row}, {col}) not stored")
        if off is None:
            raise PatternError(f"entry ({row}, {col}) lies outside the stored columns of its block row")
        self.data[off] += value
        self.support = None

    # -- compact support values (B200 transfer format) ---------------------------

    def _support_index(self):
        if self.support is None:
            raise StateError("no column support declared (support.attach_support)")
        key = ("support_index", id(self.support), id(self.slab))
        cache = _plan_cache(self)
        hit = cache.get(key)
        if hit is None or hit[2] is not self.support:
            flat, _, _ = self.support.owned_entries(self)
            hit = (_IndexList(flat, self.device), int(flat.size), self.support)
            cache[key] = hit
        return hit[0], hit[1]

    def n_support_values(self) -> int:
        return self._support_index()[1]

    def upload_support_values(self, values: torch.Tensor):
        """Owned values from the compact support order (column, then row).

        `values` (host, ideally pinned, or device) holds only the support
        entries.  The owned region is zeroed first; ghost slabs are untouched.
        """
        self._require(OWNED)
        idx, n = self._support_index()
        if values.numel() != n:
            raise ShapeError(f"{values.numel()} values for {n} support entries")
        dev = values.to(self.device, non_blocking=True) if values.device != self.device else values
        if n != self.n_owned_values:  # slab slots outside the support stay 0
            _zero_range(self.data, 0, self.n_owned_values)
        idx.scatter(dev.reshape(-1).to(torch.float64), self.data, add=False)

    def download_support_values(self, out: torch.Tensor | None = None) -> torch.Tensor:
        """Owned support entries in the compact order (device tensor, or copied into `out`)."""
        idx, n = self._support_index()
        vals = idx.gather(self.data)
        if out is not None:
            out.copy_(vals, non_blocking=True)
            return out
        return vals

    # -- ghost exchange -------------------------------------------------------

    def _exchange_plan(self):
        """Per-peer element index lists (whole slab rows), built once per matrix."""
        if self._xplan is not None:
            return self._xplan
        lay = self.layout
        imports: dict = {}
        for g in lay.import_groups:
            imports.setdefault(g.peer, []).append(g)
        ghosts: dict = {}
        for i, g in enumerate(lay.ghost_groups):
            ghosts.setdefault(g.owner, []).append(i)
        send_owned, recv_ghost = {}, {}
        z = np.zeros(0, dtype=np.int64)
        for peer, groups in sorted(imports.items()):
            parts = [self.slab.row_entries(g.block - lay.first_block, np.asarray(g.rows_in_block))
                     for g in groups]
            send_owned[peer] = _IndexList(np.concatenate(parts) if parts else z, self.device)
        for owner, gids in sorted(ghosts.items()):
            parts = []
            for gi in gids:
                lb = lay.n_owned_blocks + gi
                parts.append(self.slab.row_entries(lb, np.arange(int(self.local_row_sizes[lb]))))
            recv_ghost[owner] = _IndexList(np.concatenate(parts) if parts else z, self.device)
        self._xplan = (send_owned, recv_ghost)
        return self._xplan

    def update_ghost_values_start(self):
        if self.state in (GHOST_XCHG, COMPRESS_XCHG):
            raise StateError(f"exchange already in flight ({self.state})")
        self._require(OWNED)
        sends = []
        if self.ctx is not None and self.layout.n_ranks > 1:
            send_owned, recv_ghost = self._exchange_plan()
            sends = [(peer, il.gather(self.data)) for peer, il in send_owned.items()]
            recvs = [(owner, torch.empty(il.size, dtype=torch.float64, device=self.device))
                     for owner, il in recv_ghost.items()]
            self._pending = (recvs, self.ctx.exchange_start(sends, recvs, ("ghost", self._mid)))
        else:
            self._pending = None
        self.state = GHOST_XCHG

    def update_ghost_values_finish(self):
        if self.state != GHOST_XCHG:
            raise StateError("no ghost update in flight")
        if self._pending is not None:
            recvs, handle = self._pending
            self.ctx.exchange_finish(handle)
            _, recv_ghost = self._exchange_plan()
            for owner, buf in recvs:
                recv_ghost[owner].scatter(buf, self.data, add=False)
        self._pending = None
        self.state = GHOSTED

    def update_ghost_values(self):
        self.update_ghost_values_start()
        self.update_ghost_values_finish()

    def compress_start(self):
        if self.state in (GHOST_XCHG, COMPRESS_XCHG):
            raise StateError(f"exchange already in flight ({self.state})")
        self._require(OWNED)
        if self.ctx is not None and self.layout.n_ranks > 1:
            send_owned, recv_ghost = self._exchange_plan()
            sends = [(owner, il.gather(self.data)) for owner, il in recv_ghost.items()]
            recvs = [(peer, torch.empty(il.size, dtype=torch.float64, device=self.device))
                     for peer, il in send_owned.items()]
            self._pending = (recvs, self.ctx.exchange_start(sends, recvs, ("compress", self._mid)))
        else:
            self._pending = None
        self.state = COMPRESS_XCHG

    def compress_finish(self):
        """Owners add the partials in ascending source-rank order."""
        if self.state != COMPRESS_XCHG:
            raise StateError("no compress in flight")
        if self._pending is not None:
            recvs, handle = self._pending
            self.ctx.exchange_finish(handle)
            send_owned, _ = self._exchange_plan()
            for peer, buf in recvs:  # sorted peers: ascending source rank
                send_owned[peer].scatter(buf, self.data, add=True)
        self.zero_ghost_blocks()
        self._pending = None
        self.state = OWNED

    def compress(self):
        self.compress_start()
        self.compress_finish()


def serial_matrix(pattern: BlockSparsityPattern, lane_width: int = 8, device=None,
                  columns=None) -> BlockCsrMatrix:
    return BlockCsrMatrix(pattern, serial_layout(pattern.row_blocks), None, lane_width, device,
                          columns)


def zero_out(m: BlockCsrMatrix):
    m.zero_out()


# -- small elementwise utilities (OM glue; off the hot path) --------------------


def _plan_cache(obj):
    cache = getattr(obj, "_plans", None)
    if cache is None:
        cache = {}
        obj._plans = cache
    return cache


def _glue_index(key, a: BlockCsrMatrix, refs: tuple, build):
    """Device index tensors of an element-wise glue operation, cached on the
    first operand together with (strong references to) the geometries they
    were built from, so a recycled id() can never return stale indices."""
    cache = _plan_cache(a)
    hit = cache.get(key)
    if hit is None or any(x is not y for x, y in zip(hit[1], refs)):
        arrays = build()
        hit = (tuple(torch.as_tensor(x, dtype=torch.int64, device=a.device) for x in arrays), refs)
        cache[key] = hit
    return hit[0]


def _entry_map(dst: BlockCsrMatrix, src: BlockCsrMatrix):
    """(dst offsets, src offsets) of src's owned stored entries; dst offset
    -1 where dst does not store the entry (both share the row layout)."""
    so, grow, gcol = src._valid_owned_index()
    if so.size == 0:
        return so, so
    lb, rib = dst._owned_local(grow)
    return dst.slab.offsets(lb, rib, gcol), so


def _check_glue_operands(c: BlockCsrMatrix, x: BlockCsrMatrix, what: str):
    if x.col_blocks != c.col_blocks or x.layout.blocks != c.layout.blocks:
        raise ShapeError(f"{what} operands have different blockings")
    if x.layout.rank != c.layout.rank:
        raise ShapeError(f"{what} operands belong to different ranks")


def scale_add(c: BlockCsrMatrix, a: float, x: BlockCsrMatrix | None = None, b: float = 0.0):
    """c <- a c + b x over stored blocks; x's pattern must sit inside c's
    (reference bcsr.py:532-549).  Device element-wise ops on cached indices.
    With compact storage, every stored entry of x must be stored in c."""
    c._require(OWNED)
    c.data.mul_(a)
    if x is None or b == 0.0:
        return
    _check_glue_operands(c, x, "scale_add")
    n_s = int(x.row_start[x.n_owned_blocks])
    kc = c.local_keys()[: int(c.row_start[c.n_owned_blocks])]
    kx = x.local_keys()[:n_s]
    pos = np.searchsorted(kc, kx)
    ok = (pos < kc.size) & (kc[np.minimum(pos, max(kc.size - 1, 0))] == kx) if kc.size \
        else np.zeros(kx.size, bool)
    if not ok.all():
        p = int(np.flatnonzero(~ok)[0])
        raise ShapeError(f"scale_add: block ({int(x.pos_row[p])}, {int(x.col_index[p])}) of x "
                         f"missing from c's pattern")

    def build():
        do, so = _entry_map(c, x)
        if (do < 0).any():
            raise ShapeError("scale_add: x stores entries outside c's stored columns")
        return do, so

    di, si = _glue_index(("scale_add", id(x.slab)), c, (c.slab, x.slab), build)
    c.data.index_add_(0, di, x.data[si], alpha=b)
    if c.support is not None and x.support is not c.support:
        c.support = None  # c may now hold values outside its declared support


def copy_pattern_subset(dst: BlockCsrMatrix, src: BlockCsrMatrix):
    """dst <- src where both store the entry, zero elsewhere (reference
    bcsr.py:552-563)."""
    dst.ensure_owned()
    dst.zero_out()
    _check_glue_operands(dst, src, "copy_pattern_subset")

    def build():
        do, so = _entry_map(dst, src)
        ok = do >= 0
        return do[ok], so[ok]

    di, si = _glue_index(("copy_subset", id(src.slab)), dst, (dst.slab, src.slab), build)
    dst.data[di] = src.data[si]
    if dst.support is not None and src.support is not dst.support:
        dst.support = None


def add_scaled_identity(c: BlockCsrMatrix, s: float):
    """c <- c + s I on the owned diagonal blocks (reference bcsr.py:566-577)."""
    c._require(OWNED)

    def build():
        lbs, rs, cols = [], [], []
        for lb in range(c.n_owned_blocks):
            gb = c.layout.global_block_of_local(lb)
            if c.block_pos_local(lb, gb) < 0:
                raise PatternError(f"diagonal block ({gb}, {gb}) not stored")
            n = min(int(c.local_row_sizes[lb]), int(c.col_blocks.sizes[gb]))
            k = np.arange(n, dtype=np.int64)
            lbs.append(np.full(n, lb, dtype=np.int64))
            rs.append(k)
            cols.append(int(c.col_blocks.starts[gb]) + k)
        if not lbs:
            return (np.zeros(0, dtype=np.int64),)
        off = c.slab.offsets(np.concatenate(lbs), np.concatenate(rs), np.concatenate(cols))
        if (off < 0).any():
            raise PatternError("a diagonal entry lies outside the stored columns")
        return (off,)

    (di,) = _glue_index(("identity",), c, (c.slab,), build)
    c.data[di] += s
    c.support = None


# -- K4 / K5 ----------------------------------------------------------------------


def _check_inner(a: BlockCsrMatrix, b: BlockCsrMatrix):
    if not np.array_equal(a.col_blocks.sizes, b.layout.blocks.sizes):
        raise ShapeError("inner blockings of the product operands differ")


def mmult(a: BlockCsrMatrix, b: BlockCsrMatrix, c: BlockCsrMatrix, alpha: float = 1.0,
          accumulate: bool = False, counters: OpCounters | None = None):
    """c = alpha * a @ b truncated to c's stored entries (K5 on the GPU).

    Reference bcsr.py:587-628: b must hold ghost values for the column
    blocks of a; products outside c's pattern are discarded."""
    _check_inner(a, b)
    if a.layout.blocks != c.layout.blocks or a.layout.rank != c.layout.rank:
        raise ShapeError("a and c must share row blocking and partitioning")
    if c.col_blocks != b.col_blocks:
        raise ShapeError("b and c must share column blocking")
    if b.state != GHOSTED and b.layout.ghost_groups:
        raise StateError("b must have updated ghost values before mmult")
    c.ensure_owned()
    lib = _lib.require_device()
    plan = spmm.mmult_plan(a, b, c)
    if not accumulate:
        # every owned entry of c is written by the kernel; zero_out semantics
        # for the ghost slabs and for owned rows without chunks
        _zero_range(c.data, plan.zero_begin, c.data.numel())
    _lib.check(lib.bmv_mmult_run(plan.handle.raw, _lib.dptr(a.data), _lib.dptr(b.data),
                                 _lib.dptr(c.data), float(alpha), 1 if accumulate else 0,
                                 _lib.stream_handle(c.device)), "bmv_mmult_run")
    if c.support is not None and not (a.support is c.support):
        c.support = None
    if counters is not None:
        counters.flops += plan.flops


def tmmult(a: BlockCsrMatrix, b: BlockCsrMatrix, c: BlockCsrMatrix,
           counters: OpCounters | None = None):
    """c = a^T @ b over owned rows (K4 on the GPU), then compress c
    (reference bcsr.py:631-667; PatternError if c lacks a product block)."""
    if a.layout.blocks != b.layout.blocks or a.layout.rank != b.layout.rank:
        raise ShapeError("a and b must share row blocking and partitioning")
    if not np.array_equal(c.layout.blocks.sizes, a.col_blocks.sizes):
        raise ShapeError("c's row blocking must equal a's column blocking")
    if c.col_blocks != b.col_blocks:
        raise ShapeError("c's column blocking must equal b's")
    c.ensure_owned()
    lib = _lib.require_device()
    plan = spmm.tmmult_plan(a, b, c)
    _lib.check(lib.bmv_tmmult_run(plan.handle.raw, _lib.dptr(a.data), _lib.dptr(b.data),
                                  _lib.dptr(c.data), c.data.numel(),
                                  _lib.stream_handle(c.device)), "bmv_tmmult_run")
    c.support = None
    if counters is not None:
        counters.flops += plan.flops
    c.compress()


def tr_tmmult(d: BlockCsrMatrix, g: BlockCsrMatrix, counters: OpCounters | None = None) -> float:
    """tr(d^T g) over common stored entries, reduced over ranks (reference
    bcsr.py:670-698; the line-search slope of the OM step)."""
    if d.layout.blocks != g.layout.blocks or d.layout.rank != g.layout.rank:
        raise ShapeError("operands must share row blocking and partitioning")
    if d.col_blocks != g.col_blocks:
        raise ShapeError("operands must share column blocking")
    if d.slab is g.slab or (d.pattern is g.pattern and d.columns is g.columns):
        # same geometry: one dot over the owned values (slab padding is 0)
        n = d.n_owned_values
        local = float(torch.dot(d.data[:n], g.data[:n]).item()) if n else 0.0
        if counters is not None:
            counters.flops += 2 * n
    else:
        def build():
            go, do = _entry_map(g, d)
            ok = go >= 0
            return go[ok], do[ok]

        gi, di = _glue_index(("tr_tmmult", id(d.slab)), g, (g.slab, d.slab), build)
        local = float(torch.dot(d.data[di], g.data[gi]).item()) if di.numel() else 0.0
        if counters is not None:
            counters.flops += 2 * int(di.numel())
    if d.ctx is not None:
        return float(d.ctx.allreduce_sum(local))
    return local


def tr_mult(t: BlockCsrMatrix, h: BlockCsrMatrix, counters: OpCounters | None = None) -> float:
    """tr(t h) over stored entries, reduced over ranks; h must be ghosted for
    remote rows (reference bcsr.py:701-725; the OM energy)."""
    if not np.array_equal(t.col_blocks.sizes, h.layout.blocks.sizes):
        raise ShapeError("inner blockings differ")
    if not np.array_equal(t.layout.blocks.sizes, h.col_blocks.sizes):
        raise ShapeError("outer blockings differ")
    if h.state != GHOSTED and h.layout.ghost_groups:
        raise StateError("h must have updated ghost values before tr_mult")

    def build():
        to, grow, gcol = t._valid_owned_index()  # t(alpha = grow, beta = gcol)
        if to.size == 0:
            return to, to
        cb = t.col_blocks.blocks_of(gcol)
        hl = _local_block_table(h.layout, h.layout.blocks.n_blocks)[cb]
        ok = hl >= 0
        # block (beta's block, alpha's block) must be stored in h (reference skips it otherwise)
        rib = gcol - h.layout.blocks.starts[cb]
        ho = np.full(to.size, -1, dtype=np.int64)
        ho[ok] = h.slab.offsets(hl[ok], rib[ok], grow[ok])
        keep = ho >= 0
        return to[keep], ho[keep]

    ti, hi = _glue_index(("tr_mult", id(h.slab)), t, (t.slab, h.slab), build)
    local = float(torch.dot(t.data[ti], h.data[hi]).item()) if ti.numel() else 0.0
    if counters is not None:
        counters.flops += 2 * int(ti.numel())
    if t.ctx is not None:
        return float(t.ctx.allreduce_sum(local))
    return local


# -- serialisation (the reference's byte layout) -------------------------------------


def _reference_index(m: BlockCsrMatrix):
    """(slab offsets, reference offsets) of every stored entry, and the length
    of the reference value array (padded blocks, bcsr.py:233-318)."""
    ref_sizes = m.local_row_sizes[m.pos_row] * m.col_strides[m.col_index]
    ref_off = np.concatenate([[0], np.cumsum(ref_sizes)]).astype(np.int64)
    sg = m.slab
    off, lb, r, s = sg.block_entries(np.arange(m.n_local_blocks), m.local_row_sizes)
    pos_of_slot = np.repeat(np.arange(m.col_index.size, dtype=np.int64), sg.pos_nslot)
    gs = sg.ptr[lb] + s
    pos = pos_of_slot[gs]
    cb = m.col_index[pos]
    lane = sg.cols[gs] - m.col_blocks.starts[cb]
    return off, ref_off[pos] + r * m.col_strides[cb] + lane, int(ref_off[-1])


def to_debug_json(m: BlockCsrMatrix) -> str:
    rows = [{"global_block": m.layout.global_block_of_local(lb),
             "n_rows": int(m.local_row_sizes[lb]), "ghost": lb >= m.n_owned_blocks,
             "cols": [int(c) for c in m.row_cols_local(lb)]} for lb in range(m.n_local_blocks)]
    blocks = [{"row": int(m.pos_row[p]), "col": int(m.col_index[p]),
               "values": m.block_valid(p).cpu().tolist()} for p in range(m.col_index.size)]
    return json.dumps({"lane_width": m.lane_width, "state": m.state,
                       "row_block_sizes": m.local_row_sizes.tolist(),
                       "col_block_sizes": m.col_blocks.sizes.tolist(), "rows": rows,
                       "blocks": blocks})


def value_bytes(m: BlockCsrMatrix) -> bytes:
    """Little-endian fp64 dump of the whole value array in the reference's
    layout (padded row-major blocks, owned then ghost)."""
    off, ref, n = _reference_index(m)
    out = np.zeros(n, dtype="<f8")
    out[ref] = m.data.detach().cpu().numpy()[off]
    return out.tobytes()


def load_value_bytes(m: BlockCsrMatrix, raw: bytes):
    """Inverse of value_bytes; entries the matrix does not store must be 0."""
    arr = np.frombuffer(raw, dtype="<f8")
    off, ref, n = _reference_index(m)
    if arr.size != n:
        raise ShapeError(f"value buffer holds {arr.size} reals, matrix stores {n}")
    rest = arr.copy()
    rest[ref] = 0.0
    if np.any(rest != 0.0):
        raise ShapeError("value buffer has nonzeros outside the matrix's stored entries")
    host = np.zeros(m.data.numel())
    host[off] = arr[ref]
    m.data.copy_(torch.from_numpy(host))
    m.support = None
