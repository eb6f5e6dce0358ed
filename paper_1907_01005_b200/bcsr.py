"""Block-CSR multivectors resident in GPU memory, ghost exchange, SpMM.

Drop-in for the reference `bcsrmv/bcsr.py` (same names, signatures, state
machine and errors).  What changes is where the values live and who
computes:

* `BlockCsrMatrix.data` is a torch float64 tensor on the rank's GPU with
  the reference's exact layout (`bcsr.py:233-318`): owned blocks then ghost
  blocks, each block row-major with its row stride padded to a multiple of
  the lane width, padding held at exact zeros.  Index metadata stays on the
  host (numpy) and is turned into device plans once per operand pattern.
* ghost update / compress (`bcsr.py:401-519`) pack and unpack with the
  libbmv gather/scatter kernels and move buffers with the rank context
  (NCCL point-to-point between GPUs); compress adds in ascending source
  rank order, like the reference.
* `tmmult` / `mmult` (`bcsr.py:587-667`) run the K4 / K5 kernels: by default
  the lane-compacted ones (csrc/bmv_spmm_lane.cu: FP64 tensor cores on the
  active columns of A), with BMV_DETERMINISTIC=1 the fixed-order ones
  (bmv_project.cu, bmv_postmul.cu).
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

from . import _lib, _plan
from .blocks import BlockIndices, BlockSparsityPattern
from .counters import OpCounters
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


class BlockCsrMatrix:
    """Rank-local BCSR matrix; values on the GPU in the reference layout."""

    def __init__(self, pattern: BlockSparsityPattern, layout: RankLayout, ctx=None,
                 lane_width: int = 8, device=None):
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
        sizes = self.local_row_sizes[self.pos_row] * self.col_strides[self.col_index]
        self.block_offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        self._ghost_data_begin = int(self.block_offsets[self.row_start[layout.n_owned_blocks]])
        if device is None:
            device = getattr(ctx, "device", None) or default_device()
        self.device = torch.device(device)
        self.data = torch.zeros(int(self.block_offsets[-1]), dtype=torch.float64, device=self.device)
        self.state = OWNED
        self._mid = ctx.next_matrix_id() if ctx is not None else 0
        self._pending = None
        self._xplan = None
        self.support = None  # optional entry-level column support (support.py)

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
        rows = int(self.local_row_sizes[self.pos_row[pos]])
        stride = int(self.col_strides[self.col_index[pos]])
        off = int(self.block_offsets[pos])
        return self.data[off : off + rows * stride].view(rows, stride)

    def block_valid(self, pos: int) -> torch.Tensor:
        cols = int(self.col_blocks.sizes[self.col_index[pos]])
        return self.block_values(pos)[:, :cols]

    def block_pos_local(self, lb: int, col: int) -> int:
        lo, hi = int(self.row_start[lb]), int(self.row_start[lb + 1])
        k = lo + int(np.searchsorted(self.col_index[lo:hi], col))
        if k < hi and self.col_index[k] == col:
            return k
        return -1

    def local_keys(self) -> np.ndarray:
        """Sorted keys local_block * n_col_blocks + col of the stored blocks."""
        return self.pos_row * self.col_blocks.n_blocks + self.col_index

    def _entry_index(self, positions: np.ndarray, rows_sel=None, full_rows=True) -> np.ndarray:
        """Flat element offsets of the valid entries of blocks, row-major."""
        out = []
        for pos in positions.tolist():
            cols = int(self.col_blocks.sizes[self.col_index[pos]])
            stride = int(self.col_strides[self.col_index[pos]])
            nrow = int(self.local_row_sizes[self.pos_row[pos]])
            r = np.arange(nrow) if rows_sel is None else rows_sel
            out.append((int(self.block_offsets[pos]) + r[:, None] * stride
                        + np.arange(cols)[None, :]).ravel())
        return np.concatenate(out) if out else np.zeros(0, dtype=np.int64)

    def _require(self, *states):
        if self.state not in states:
            raise StateError(f"operation requires state in {states}, matrix is {self.state}")

    def ensure_owned(self):
        if self.state == GHOSTED:
            self.release_ghosts()
        else:
            self._require(OWNED)

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
        out = BlockCsrMatrix.__new__(BlockCsrMatrix)
        out.__dict__.update(self.__dict__)
        out.data = self.data.clone()
        out._pending = None
        return out

    def _valid_owned_index(self):
        """(flat offsets, global rows, global cols) of every owned valid entry."""
        n_own = int(self.row_start[self.n_owned_blocks])
        if n_own == 0:
            z = np.zeros(0, dtype=np.int64)
            return z, z, z
        pos = np.arange(n_own)
        lb = self.pos_row[pos]
        c = self.col_index[pos]
        nrow = self.local_row_sizes[lb]
        ncol = self.col_blocks.sizes[c]
        cnt = nrow * ncol
        rep = np.repeat(pos, cnt)
        k = np.arange(int(cnt.sum())) - np.repeat(np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt)
        ncol_e = ncol[rep]
        r = k // ncol_e
        j = k - r * ncol_e
        flat = self.block_offsets[rep] + r * self.col_strides[c][rep] + j
        grow = self.layout.blocks.starts[self.layout.first_block + lb][rep] + r
        gcol = self.col_blocks.starts[c][rep] + j
        return flat, grow, gcol

    def fill_owned(self, fn):
        """Set every owned block to fn(global_rows, global_cols) (host callback)."""
        self._require(OWNED)
        host = self.data.detach().cpu().numpy().copy()
        for pos in range(int(self.row_start[self.n_owned_blocks])):
            lb = int(self.pos_row[pos])
            gb = self.layout.global_block_of_local(lb)
            r0 = int(self.layout.blocks.starts[gb])
            rows = np.arange(r0, r0 + int(self.local_row_sizes[lb]))
            c = int(self.col_index[pos])
            c0 = int(self.col_blocks.starts[c])
            cols = np.arange(c0, c0 + int(self.col_blocks.sizes[c]))
            vals = np.asarray(fn(rows, cols), dtype=np.float64)
            stride = int(self.col_strides[c])
            off = int(self.block_offsets[pos])
            blk = host[off : off + rows.size * stride].reshape(rows.size, stride)
            blk[:, : cols.size] = vals
        self.data.copy_(torch.from_numpy(host))

    def fill_owned_entries(self, fn_flat):
        """Vectorised fill: fn_flat(global_rows, global_cols) -> values per entry."""
        self._require(OWNED)
        flat, grow, gcol = self._valid_owned_index()
        if flat.size == 0:
            return
        vals = np.asarray(fn_flat(grow, gcol), dtype=np.float64)
        host = self.data.detach().cpu().numpy().copy()
        host[flat] = vals
        self.data.copy_(torch.from_numpy(host))

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
        cb, cic = self.col_blocks.global_to_block(col)
        pos = self.block_pos_local(int(lb[0]), cb)
        if pos < 0:
            return None
        return int(self.block_offsets[pos]) + int(rib[0]) * int(self.col_strides[cb]) + cic

    def get_entry(self, row: int, col: int) -> float:
        off = self._entry_offset(row, col)
        return 0.0 if off is None else float(self.data[off].item())

    def add_entry(self, row: int, col: int, value: float):
        off = self._entry_offset(row, col)
        if off is None:
            raise PatternError(f"block for entry ({row}, {col}) not stored")
        self.data[off] += value

    # -- compact support values (B200 transfer format) ---------------------------

    def _support_index(self):
        if self.support is None:
            raise StateError("no column support attached (support.attach_support)")
        key = ("support_index", id(self.support))
        cache = _plan_cache(self)
        hit = cache.get(key)
        if hit is None:
            flat, _, _ = self.support.owned_entries(self)
            hit = (_IndexList(flat, self.device), int(flat.size))
            cache[key] = hit
        return hit

    def n_support_values(self) -> int:
        return self._support_index()[1]

    def upload_support_values(self, values: torch.Tensor):
        """Owned values from the compact support order (column, then row).

        `values` (host, ideally pinned, or device) holds only the structurally
        nonzero entries -- the nnz of the multivector instead of its padded
        blocks -- so host->device traffic drops by the block fill factor.  The
        owned region is zeroed first; ghost blocks are untouched.
        """
        self._require(OWNED)
        idx, n = self._support_index()
        if values.numel() != n:
            raise ShapeError(f"{values.numel()} values for {n} support entries")
        dev = values.to(self.device, non_blocking=True) if values.device != self.device else values
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
        """Per-peer element index lists, built once per matrix."""
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
        for peer, groups in sorted(imports.items()):
            parts = []
            for g in groups:
                lb = g.block - lay.first_block
                pos = np.arange(self.row_start[lb], self.row_start[lb + 1])
                parts.append(self._entry_index(pos, rows_sel=np.asarray(g.rows_in_block)))
            idx = np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)
            send_owned[peer] = _IndexList(idx, self.device)
        for owner, gids in sorted(ghosts.items()):
            parts = []
            for gi in gids:
                lb = lay.n_owned_blocks + gi
                pos = np.arange(self.row_start[lb], self.row_start[lb + 1])
                parts.append(self._entry_index(pos))
            idx = np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)
            recv_ghost[owner] = _IndexList(idx, self.device)
        self._xplan = (send_owned, recv_ghost)
        return self._xplan

    def update_ghost_values_start(self):
        if self.state in (GHOST_XCHG, COMPRESS_XCHG):
            raise StateError(f"exchange already in flight ({self.state})")
        self._require(OWNED)
        sends = []
        if self.ctx is not None and self.layout.n_ranks > 1:
            send_owned, _ = self._exchange_plan()
            sends = [(peer, il.gather(self.data)) for peer, il in send_owned.items()]
        self._pending = sends
        self.state = GHOST_XCHG

    def update_ghost_values_finish(self):
        if self.state != GHOST_XCHG:
            raise StateError("no ghost update in flight")
        if self.ctx is not None and self.layout.n_ranks > 1:
            _, recv_ghost = self._exchange_plan()
            recvs = [(owner, torch.empty(il.size, dtype=torch.float64, device=self.device))
                     for owner, il in recv_ghost.items()]
            self.ctx.exchange(self._pending, recvs)
            for (owner, buf) in recvs:
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
        sends = []
        if self.ctx is not None and self.layout.n_ranks > 1:
            _, recv_ghost = self._exchange_plan()
            sends = [(owner, il.gather(self.data)) for owner, il in recv_ghost.items()]
        self._pending = sends
        self.state = COMPRESS_XCHG

    def compress_finish(self):
        """Owners add the partials in ascending source-rank order."""
        if self.state != COMPRESS_XCHG:
            raise StateError("no compress in flight")
        if self.ctx is not None and self.layout.n_ranks > 1:
            send_owned, _ = self._exchange_plan()
            recvs = [(peer, torch.empty(il.size, dtype=torch.float64, device=self.device))
                     for peer, il in send_owned.items()]
            self.ctx.exchange(self._pending, recvs)
            for peer, buf in recvs:  # sorted peers: ascending source rank
                send_owned[peer].scatter(buf, self.data, add=True)
        self.zero_ghost_blocks()
        self._pending = None
        self.state = OWNED

    def compress(self):
        self.compress_start()
        self.compress_finish()


def serial_matrix(pattern: BlockSparsityPattern, lane_width: int = 8, device=None) -> BlockCsrMatrix:
    return BlockCsrMatrix(pattern, serial_layout(pattern.row_blocks), None, lane_width, device)


def zero_out(m: BlockCsrMatrix):
    m.zero_out()


# -- small elementwise utilities (OM glue; off the hot path) --------------------


def _common_positions(dst: BlockCsrMatrix, src: BlockCsrMatrix):
    kd, ks = dst.local_keys(), src.local_keys()
    n_d = int(dst.row_start[dst.n_owned_blocks])
    n_s = int(src.row_start[src.n_owned_blocks])
    kd, ks = kd[:n_d], ks[:n_s]
    pos = np.searchsorted(kd, ks)
    ok = (pos < kd.size) & (kd[np.minimum(pos, max(kd.size - 1, 0))] == ks) if kd.size else np.zeros(ks.size, bool)
    return np.arange(n_s)[ok], pos[ok], np.arange(n_s)[~ok]


def _entry_offsets(m: BlockCsrMatrix, positions: np.ndarray) -> np.ndarray:
    """Flat element offsets of the valid entries of blocks `positions`,
    block by block, row-major inside a block (vectorised _entry_index)."""
    positions = np.asarray(positions, dtype=np.int64)
    if positions.size == 0:
        return np.zeros(0, dtype=np.int64)
    cb = m.col_index[positions]
    n_c = m.col_blocks.sizes[cb].astype(np.int64)
    n_r = m.local_row_sizes[m.pos_row[positions]].astype(np.int64)
    owner, t = _expand(n_r * n_c)
    r, c = t // n_c[owner], t % n_c[owner]
    return m.block_offsets[positions[owner]] + r * m.col_strides[cb[owner]] + c


def _glue_index(key, a: BlockCsrMatrix, build):
    """Device index tensors of an element-wise glue operation, cached per
    (operation, operand patterns, layouts) on the first operand."""
    cache = _plan_cache(a)
    hit = cache.get(key)
    if hit is None:
        arrays = build()
        hit = tuple(torch.as_tensor(x, dtype=torch.int64, device=a.device) for x in arrays)
        cache[key] = hit
    return hit


def _common_entries(dst: BlockCsrMatrix, src: BlockCsrMatrix):
    """(dst offsets, src offsets) of the valid entries of the owned blocks both
    store, and the src positions dst lacks."""
    s_pos, d_pos, missing = _common_positions(dst, src)
    return _entry_offsets(dst, d_pos), _entry_offsets(src, s_pos), missing


def scale_add(c: BlockCsrMatrix, a: float, x: BlockCsrMatrix | None = None, b: float = 0.0):
    """c <- a c + b x over stored blocks; x's pattern must sit inside c's
    (reference bcsr.py:532-549).  Device element-wise ops on cached indices."""
    c._require(OWNED)
    c.data.mul_(a)
    if x is None or b == 0.0:
        return
    if x.col_blocks != c.col_blocks or x.layout.blocks != c.layout.blocks:
        raise ShapeError("scale_add operands have different blockings")
    _, _, missing = _common_positions(c, x)
    if missing.size:
        p = int(missing[0])
        raise ShapeError(f"scale_add: block ({int(x.pos_row[p])}, {int(x.col_index[p])}) of x missing from c's pattern")
    di, si = _glue_index(("scale_add", id(c.pattern), id(x.pattern), id(x.layout)), c,
                         lambda: _common_entries(c, x)[:2])
    c.data.index_add_(0, di, x.data[si], alpha=b)


def copy_pattern_subset(dst: BlockCsrMatrix, src: BlockCsrMatrix):
    """dst <- src where both patterns store the block, zero elsewhere
    (reference bcsr.py:552-563)."""
    dst.ensure_owned()
    dst.zero_out()
    if src.col_blocks != dst.col_blocks or src.layout.blocks != dst.layout.blocks:
        raise ShapeError("copy_pattern_subset operands have different blockings")
    di, si = _glue_index(("copy_subset", id(dst.pattern), id(src.pattern), id(src.layout)), dst,
                         lambda: _common_entries(dst, src)[:2])
    dst.data[di] = src.data[si]


def add_scaled_identity(c: BlockCsrMatrix, s: float):
    """c <- c + s I on the owned diagonal blocks (reference bcsr.py:566-577)."""
    c._require(OWNED)

    def build():
        idx = []
        for lb in range(c.n_owned_blocks):
            gb = c.layout.global_block_of_local(lb)
            pos = c.block_pos_local(lb, gb)
            if pos < 0:
                raise PatternError(f"diagonal block ({gb}, {gb}) not stored")
            n = min(int(c.local_row_sizes[lb]), int(c.col_blocks.sizes[gb]))
            k = np.arange(n)
            idx.append(int(c.block_offsets[pos]) + k * int(c.col_strides[gb]) + k)
        return (np.concatenate(idx) if idx else np.zeros(0, dtype=np.int64),)

    (di,) = _glue_index(("identity", id(c.pattern), id(c.layout)), c, build)
    c.data[di] += s


# -- K4 / K5 ----------------------------------------------------------------------


def _check_inner(a: BlockCsrMatrix, b: BlockCsrMatrix):
    if not np.array_equal(a.col_blocks.sizes, b.layout.blocks.sizes):
        raise ShapeError("inner blockings of the product operands differ")


def _plan_cache(obj):
    cache = getattr(obj, "_plans", None)
    if cache is None:
        cache = {}
        obj._plans = cache
    return cache


def _expand(counts: np.ndarray):
    """(owner index, rank within owner) of sum(counts) expanded items."""
    counts = np.asarray(counts, dtype=np.int64)
    owner = np.repeat(np.arange(counts.size, dtype=np.int64), counts)
    start = np.concatenate([[0], np.cumsum(counts)])[:-1]
    return owner, np.arange(int(counts.sum()), dtype=np.int64) - start[owner]


def _local_block_table(layout: RankLayout, n_global: int) -> np.ndarray:
    """Local block id of every global block (-1 when neither owned nor ghost)."""
    tab = np.full(n_global, -1, dtype=np.int64)
    gl = layout.global_blocks_of_locals()
    tab[gl] = np.arange(gl.size, dtype=np.int64)
    return tab


def _group_by_output(out_pos: np.ndarray):
    """Stable grouping of work items by output block: (order, unique outputs, starts)."""
    order = np.argsort(out_pos, kind="stable")
    sp = out_pos[order]
    uniq, first = np.unique(sp, return_index=True)
    start = np.concatenate([first, [sp.size]]).astype(np.int64)
    return order, uniq, start


def _mmult_plan(a: BlockCsrMatrix, b: BlockCsrMatrix, c: BlockCsrMatrix):
    key = ("mm", id(b), id(c))
    cache = _plan_cache(a)
    hit = cache.get(key)
    if hit is not None:
        return hit[0]
    arrays, n_out, n_pairs, flops, full_cover = mmult_plan_arrays(a, b, c, _pj_parts(c.device))
    plan = _MmultPlan(arrays, n_out, n_pairs, flops)
    plan.full_cover = full_cover
    cache[key] = (plan, b, c)
    return plan


def mmult_plan_arrays(a: BlockCsrMatrix, b: BlockCsrMatrix, c: BlockCsrMatrix, n_parts: int):
    """K5 streaming plan (include/bmv.h bmv_mmult_desc): per output block of
    C the (A_ik, B_kj) products kept by C's pattern, in the reference's
    Gustavson order (bcsr.py:605-626).  Host-only; returns
    (arrays, n_out, n_pairs, flops, full_cover)."""
    n_own_pos = int(a.row_start[a.n_owned_blocks])
    pos_a = np.arange(n_own_pos, dtype=np.int64)
    k = a.col_index[pos_a]
    kb = _local_block_table(b.layout, b.layout.blocks.n_blocks)[k]
    if (kb < 0).any():
        raise PatternError(f"rank {b.layout.rank} holds no ghost of block row {int(k[kb < 0][0])}")
    if (b.local_row_sizes[kb] != a.col_blocks.sizes[k]).any():
        bad = int(k[b.local_row_sizes[kb] != a.col_blocks.sizes[k]][0])
        raise ShapeError(f"row block {bad} of b is incomplete (split ghost group)")
    nb = b.row_start[kb + 1] - b.row_start[kb]
    owner, r = _expand(nb)
    pa = pos_a[owner]
    pb = b.row_start[kb[owner]] + r
    i = a.pos_row[pa]
    ckey = i * c.col_blocks.n_blocks + b.col_index[pb]
    ckeys = c.local_keys()
    cp = np.searchsorted(ckeys, ckey)
    ok = (cp < ckeys.size) & (ckeys[np.minimum(cp, max(ckeys.size - 1, 0))] == ckey) \
        if ckeys.size else np.zeros(ckey.size, dtype=bool)
    pa, pb, cp = pa[ok], pb[ok], cp[ok]
    order, outs, start = _group_by_output(cp)
    pa, pb = pa[order], pb[order]
    n_out = int(outs.size)
    # ---- streaming plan (csrc/bmv_postmul.cu) ------------------------------
    # stage = [header][tasks][pairs][B blocks][A blocks]; a task = up to 8 row
    # tiles x one 8-column tile of an output block
    n_rows = a.n_owned_blocks
    a_row_lo = a.block_offsets[a.row_start[:n_rows]]
    a_row_hi = a.block_offsets[a.row_start[1 : n_rows + 1]]
    row_dbl = a_row_hi - a_row_lo
    per = np.repeat(np.arange(n_out), np.diff(start))
    out_row = c.pos_row[outs] if n_out else np.zeros(0, np.int64)
    out_rows = c.local_row_sizes[out_row].astype(np.int64)
    out_cols = c.col_blocks.sizes[c.col_index[outs]].astype(np.int64)
    c_str = c.col_strides[c.col_index[outs]].astype(np.int64)
    tm = (out_rows + 8 * _PM_ROW_TILES - 1) // (8 * _PM_ROW_TILES)
    tn = (out_cols + 7) // 8
    if n_out and (int(tn.max()) > 16 or int(c_str.max()) >= 1 << 16):
        raise ShapeError("mmult output blocks wider than 128 columns are not supported")
    np_o = np.diff(start).astype(np.int64)
    pair_row = out_row[per] if pa.size else np.zeros(0, np.int64)
    b_size = (b.block_offsets[pb + 1] - b.block_offsets[pb]).astype(np.int64)
    b_bytes = 8 * b_size + (8 * b_size) % 16
    nbk = int(b.pos_row.size) + 1
    rk, r_first = np.unique(pair_row * nbk + pb, return_index=True)
    row_cbytes = np.bincount(rk // nbk, weights=b_bytes[r_first], minlength=n_rows).astype(np.int64)
    row_tasks = np.bincount(out_row, weights=tm * tn, minlength=n_rows).astype(np.int64)
    row_pairs = np.bincount(pair_row, minlength=n_rows).astype(np.int64)
    row_bytes = 8 * row_dbl + 16 * (row_tasks + row_pairs) + row_cbytes
    # parts balanced by A + Y doubles; sub-chunks of consecutive rows
    y_dbl = np.bincount(out_row, weights=out_rows * c_str, minlength=n_rows).astype(np.int64)
    w = row_dbl + y_dbl
    n_parts = max(1, min(int(n_parts), n_rows))
    total = max(int(w.sum()), 1)
    before = np.concatenate([[0], np.cumsum(w)[:-1]]) if n_rows else np.zeros(0, np.int64)
    r_part = np.minimum(before * n_parts // total, n_parts - 1)
    r_sub = np.empty(n_rows, dtype=np.int64)
    sid, acc = -1, 0
    bl, pl = row_bytes.tolist(), r_part.tolist()
    for j in range(n_rows):
        if sid < 0 or pl[j] != pl[j - 1] or acc + bl[j] > _PM_STAGE_BYTES - 32:
            sid += 1
            acc = 0
        acc += bl[j]
        r_sub[j] = sid
    n_sub = sid + 1
    first_r = np.searchsorted(r_sub, np.arange(n_sub + 1)).astype(np.int64)
    sub_a = np.stack([a_row_lo[first_r[:-1]], a_row_hi[first_r[1:] - 1]], 1) if n_sub \
        else np.zeros((0, 2), np.int64)
    part_sub_start = np.searchsorted(r_part[first_r[:-1]], np.arange(n_parts + 1)).astype(np.int64)
    o_lo = np.searchsorted(out_row, first_r[:-1])       # outputs are in row order
    o_hi = np.searchsorted(out_row, first_r[1:])
    o_sub = r_sub[out_row]
    to, tq = _expand(tm * tn)
    t_mi, t_ni = tq // tn[to], tq % tn[to]               # t_mi counts 64-row task rows
    t_sub = o_sub[to]
    n_tasks_sub = np.bincount(t_sub, minlength=n_sub).astype(np.int64)
    n_pairs_sub = (start[o_hi] - start[o_lo]).astype(np.int64)
    if n_sub and int(max(np_o.max(initial=0), n_pairs_sub.max())) >= 1 << 16:
        raise ShapeError("mmult sub-chunk holds more than 65535 products")
    meta_bytes = 16 * (1 + n_tasks_sub + n_pairs_sub)
    # distinct B blocks per sub-chunk, staged after the metadata
    p_sub = o_sub[per] if pa.size else np.zeros(0, np.int64)
    sk, s_first, p_cb = np.unique(p_sub * nbk + pb, return_index=True, return_inverse=True)
    cb_sub, cb_pb, cb_bytes = sk // nbk, sk % nbk, b_bytes[s_first]
    n_cb_sub = np.bincount(cb_sub, minlength=n_sub).astype(np.int64)
    cb_first = np.concatenate([[0], np.cumsum(n_cb_sub)]).astype(np.int64)
    cb_cum = np.concatenate([[0], np.cumsum(cb_bytes)]).astype(np.int64)
    cb_soff = meta_bytes[cb_sub] + cb_cum[:-1] - cb_cum[cb_first[cb_sub]]
    a_off = meta_bytes + cb_cum[cb_first[1:]] - cb_cum[cb_first[:-1]]
    na_sub = sub_a[:, 1] - sub_a[:, 0]
    stage_bytes = int((a_off + 8 * na_sub).max(initial=16))
    stage_bytes += (-stage_bytes) % 16
    if 2 * stage_bytes > _SMEM_OPTIN - 1024:
        raise ShapeError(f"mmult block row needs {stage_bytes} bytes of shared memory (2 stages)")
    meta_off = np.concatenate([[0], np.cumsum(meta_bytes // 4)]).astype(np.int64)
    meta = np.zeros(int(meta_off[-1]), dtype=np.int64)
    meta[meta_off[:-1]] = n_tasks_sub
    task_first = np.concatenate([[0], np.cumsum(n_tasks_sub)]).astype(np.int64)
    tpos = meta_off[t_sub] + 4 * (1 + np.arange(to.size) - task_first[t_sub])
    r0 = 8 * _PM_ROW_TILES * t_mi
    t_off = c.block_offsets[outs][to] + r0 * c_str[to] + 8 * t_ni
    if t_off.size and int(t_off.max()) >= 1 << 32:
        raise ShapeError("mmult output holds more than 2^32 values")
    meta[tpos] = t_off
    meta[tpos + 1] = (np.minimum(8 * _PM_ROW_TILES, out_rows[to] - r0)
                      | (np.minimum(8, out_cols[to] - 8 * t_ni) << 8) | (t_ni << 12) | (c_str[to] << 16))
    meta[tpos + 2] = (start[to] - start[o_lo[t_sub]]) | (np_o[to] << 16)
    meta[tpos + 3] = _PM_ROW_TILES * t_mi
    a_str = a.col_strides[a.col_index[pa]].astype(np.int64)
    inner = a.col_blocks.sizes[a.col_index[pa]].astype(np.int64)
    ppos = meta_off[p_sub] + 4 * (1 + n_tasks_sub[p_sub] + np.arange(pa.size) - start[o_lo[p_sub]])
    meta[ppos] = a_off[p_sub] // 8 + a.block_offsets[pa] - sub_a[p_sub, 0]
    meta[ppos + 1] = a_str | (inner << 16)
    meta[ppos + 2] = b.col_strides[b.col_index[pb]]
    meta[ppos + 3] = cb_soff[p_cb] // 8
    meta = (meta & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
    # copy lists: metadata, B blocks, A range (last)
    e_first = np.concatenate([[0], np.cumsum(2 + n_cb_sub)]).astype(np.int64)
    copies = np.zeros((int(e_first[-1]), 4), dtype=np.int64)
    copies[e_first[:-1], 1] = meta_bytes
    copies[e_first[:-1], 2] = 4 * meta_off[:-1]
    cpos = e_first[cb_sub] + 1 + np.arange(cb_sub.size) - cb_first[cb_sub]
    copies[cpos, 0] = cb_soff
    copies[cpos, 1] = 8 * b_size[s_first] | (2 << 28)
    copies[cpos, 2] = 8 * b.block_offsets[cb_pb]
    last = e_first[1:] - 1
    copies[last, 0] = a_off
    copies[last, 1] = 8 * na_sub | (1 << 28) | (1 << 30)
    copies[last, 2] = 8 * sub_a[:, 0]
    arrays = dict(
        n_parts=n_parts, stage_bytes=stage_bytes, n_sub=n_sub,
        part_sub_start=part_sub_start, part_entry_start=e_first[part_sub_start],
        copies=_pack_copies(copies), meta=meta,
    )
    flops = int(2 * np.sum(out_rows[per] * inner * out_cols[per]))
    n_own_c = int(c.row_start[c.n_owned_blocks])
    own_cols = c.col_index[:n_own_c]
    full_cover = bool(n_out == n_own_c and
                      np.all(c.col_blocks.sizes[own_cols] == c.col_strides[own_cols]))
    return arrays, n_out, int(pa.size), flops, full_cover


_SMEM_OPTIN = 232_448   # B200 max dynamic shared memory per block (bytes)


class _MmultPlan:
    def __init__(self, arrays, n_out, n_pairs, flops):
        self.arrays = arrays
        self.flops = flops
        self.n_out = n_out
        lib = _lib.load()
        d = _lib.MmultDesc()
        d.n_parts = int(arrays["n_parts"])
        d.stage_bytes = int(arrays["stage_bytes"])
        d.n_sub = int(arrays["n_sub"])
        d.n_entries = int(arrays["copies"].size // 4)
        d.meta_len = int(arrays["meta"].size)
        for name, ct in (("part_sub_start", _lib.C.c_int64), ("part_entry_start", _lib.C.c_int64),
                         ("copies", _lib.C.c_int32), ("meta", _lib.C.c_int32)):
            arrays[name] = np.ascontiguousarray(arrays[name])
            setattr(d, name, _lib.ptr(arrays[name], ct))
        raw = _lib.C.c_void_p()
        _lib.check(lib.bmv_mmult_create(_lib.C.byref(d), _lib.C.byref(raw)), "bmv_mmult_create")
        self.handle = _lib.Handle("bmv_mmult_destroy", raw)


# -- lane-compacted K4 / K5 (csrc/bmv_spmm_lane.cu) -------------------------------


def _deterministic() -> bool:
    """BMV_DETERMINISTIC=1 keeps the fixed-order K4 / K5 kernels (bmv_project.cu,
    bmv_postmul.cu); default: the lane-compacted kernels (S reduced with fp64
    atomics, like K1's default scatter)."""
    return os.environ.get("BMV_DETERMINISTIC", "0") == "1"


def _a_lane_masks(a: BlockCsrMatrix) -> np.ndarray:
    """uint64 mask of the lanes of every owned block of `a` that may hold
    nonzeros: its declared column support (support.py) or, without one, all
    stored columns of the block.  Host-only; cached per support."""
    key = ("lanemask", id(a.support))
    cache = _plan_cache(a)
    hit = cache.get(key)
    if hit is not None and hit[1] is a.support:
        return hit[0]
    n_pos = int(a.row_start[a.n_owned_blocks])
    widths = a.col_blocks.sizes[a.col_index[:n_pos]].astype(np.int64)
    if widths.size and int(widths.max()) > 64:
        raise ShapeError("lane masks need column blocks of at most 64 columns")
    if a.support is None:
        mask = np.where(widths >= 64, np.uint64(0xFFFFFFFFFFFFFFFF),
                        (np.uint64(1) << np.minimum(widths, 63).astype(np.uint64)) - np.uint64(1))
        mask = mask.astype(np.uint64)
    else:
        flat, _rows, cols = a.support.owned_entries(a)
        mask = np.zeros(n_pos, dtype=np.uint64)
        if flat.size:
            pos = np.searchsorted(a.block_offsets[: n_pos + 1], flat, side="right") - 1
            cb = a.col_blocks.blocks_of(cols)
            lane = (cols - a.col_blocks.starts[cb]).astype(np.uint64)
            np.bitwise_or.at(mask, pos, np.uint64(1) << lane)
    cache[key] = (mask, a.support)
    return mask


def _lane_plan_or_none(build, a, b, c):
    """The lane plan, or None when the shapes exceed it (ShapeError from the
    planner: > 64 columns per block, > 32 active columns per row for K5, a
    block row larger than a stage); PatternError propagates."""
    key = ("lane_fail", build.__name__, id(b), id(c), id(a.support))
    cache = _plan_cache(a)
    if key in cache:
        return None
    try:
        return build(a, b, c)
    except ShapeError as exc:
        cache[key] = True
        import warnings

        warnings.warn(f"{build.__name__}: {exc}; using the fixed-order kernel", RuntimeWarning,
                      stacklevel=3)
        return None


def lane_plan_host(kind: int, desc, n_parts: int = 4) -> dict:
    """The stage stream of a lane plan as numpy arrays (bmv_lane_plan_host;
    no device).  Used by the tests' CPU emulation of the lane kernels."""
    lib = _lib.load()
    h = _lib.LaneHost()
    _lib.check(lib.bmv_lane_plan_host(int(kind), _lib.C.cast(_lib.C.byref(desc), _lib.C.c_void_p),
                                      int(n_parts), _lib.C.byref(h)), "bmv_lane_plan_host")
    try:
        def arr(p, n):
            return np.ctypeslib.as_array(p, shape=(int(n),)).copy() if n else np.zeros(0, np.int64)
        out = dict(stage_bytes=int(h.stage_bytes), n_parts=int(h.n_parts),
                   meta=arr(h.meta, h.meta_len).astype(np.int32),
                   copies=arr(h.copies, 4 * h.n_entries).astype(np.int32).reshape(-1, 4),
                   part_sub_start=arr(h.part_sub_start, h.n_parts + 1 if h.n_parts else 0),
                   part_entry_start=arr(h.part_entry_start, h.n_parts + 1 if h.n_parts else 0))
    finally:
        lib.bmv_lane_host_free(_lib.C.byref(h))
    return out


class _LanePlan:
    def __init__(self, kind: str, desc, keep):
        lib = _lib.load()
        raw = _lib.C.c_void_p()
        fn = lib.bmv_tmmult_lane_create if kind == "tm" else lib.bmv_mmult_lane_create
        _lib.check(fn(_lib.C.byref(desc), _lib.C.byref(raw)), f"bmv_{kind}mult_lane_create")
        self.handle = _lib.Handle("bmv_lane_plan_destroy", raw)
        self._keep = keep


def _tm_pairs(a: BlockCsrMatrix, b: BlockCsrMatrix, c: BlockCsrMatrix):
    """(row, pa, pb, c position) of every owned block pair, row-major over
    (pa, pb) inside a row; PatternError if c lacks a product block."""
    n_rows = a.n_owned_blocks
    na = a.row_start[1 : n_rows + 1] - a.row_start[:n_rows]
    nb = b.row_start[1 : n_rows + 1] - b.row_start[:n_rows]
    row, t = _expand(na * nb)
    nbr = nb[row]
    pa = a.row_start[row] + t // np.maximum(nbr, 1)
    pb = b.row_start[row] + t % np.maximum(nbr, 1)
    k = a.col_index[pa]
    ck = _local_block_table(c.layout, c.layout.blocks.n_blocks)[k]
    if (ck < 0).any():
        raise PatternError(f"rank {c.layout.rank} holds no ghost of block row {int(k[ck < 0][0])}")
    ell = b.col_index[pb]
    ckey = ck * c.col_blocks.n_blocks + ell
    ckeys = c.local_keys()
    cp = np.searchsorted(ckeys, ckey)
    ok = (cp < ckeys.size) & (ckeys[np.minimum(cp, max(ckeys.size - 1, 0))] == ckey) \
        if ckeys.size else np.zeros(ckey.size, dtype=bool)
    if not ok.all():
        j = int(np.flatnonzero(~ok)[0])
        raise PatternError(f"tmmult destination misses block ({int(k[j])}, {int(ell[j])})")
    if (c.local_row_sizes[c.pos_row[cp]] != a.col_blocks.sizes[k]).any():
        raise ShapeError("tmmult destination row block is incomplete (split ghost group)")
    return row, pa, pb, cp


def _tmmult_lane_plan(a: BlockCsrMatrix, b: BlockCsrMatrix, c: BlockCsrMatrix):
    key = ("tml", id(b), id(c), id(a.support))
    cache = _plan_cache(a)
    hit = cache.get(key)
    if hit is not None:
        return hit[0]
    d, arr = tmmult_lane_desc(a, b, c)
    plan = _LanePlan("tm", d, arr)
    cache[key] = (plan, b, c, a.support)
    return plan


def tmmult_lane_desc(a: BlockCsrMatrix, b: BlockCsrMatrix, c: BlockCsrMatrix):
    """(bmv_tmmult_lane_desc, arrays it points into): host-only."""
    n_rows = a.n_owned_blocks
    _row, _pa, _pb, cp = _tm_pairs(a, b, c)
    n_pa = int(a.row_start[n_rows])
    n_pb = int(b.row_start[n_rows])
    arr = dict(
        row_rows=a.local_row_sizes[:n_rows].astype(np.int32),
        a_row_start=a.row_start[: n_rows + 1].astype(np.int64),
        a_off=a.block_offsets[:n_pa].astype(np.int64),
        a_stride=a.col_strides[a.col_index[:n_pa]].astype(np.int32),
        a_mask=_a_lane_masks(a),
        b_row_start=b.row_start[: n_rows + 1].astype(np.int64),
        b_off=b.block_offsets[:n_pb].astype(np.int64),
        b_stride=b.col_strides[b.col_index[:n_pb]].astype(np.int32),
        b_width=b.col_blocks.sizes[b.col_index[:n_pb]].astype(np.int32),
        c_off=c.block_offsets[cp].astype(np.int64),
        c_stride=c.col_strides[c.col_index[cp]].astype(np.int32),
        c_rows=c.local_row_sizes[c.pos_row[cp]].astype(np.int32),
    )
    arr = {k: np.ascontiguousarray(v) for k, v in arr.items()}
    d = _lib.TmmultLaneDesc()
    d.n_rows = n_rows
    for name, ct in (("row_rows", _lib.C.c_int32), ("a_row_start", _lib.C.c_int64),
                     ("a_off", _lib.C.c_int64), ("a_stride", _lib.C.c_int32),
                     ("a_mask", _lib.C.c_uint64), ("b_row_start", _lib.C.c_int64),
                     ("b_off", _lib.C.c_int64), ("b_stride", _lib.C.c_int32),
                     ("b_width", _lib.C.c_int32), ("c_off", _lib.C.c_int64),
                     ("c_stride", _lib.C.c_int32), ("c_rows", _lib.C.c_int32)):
        setattr(d, name, _lib.ptr(arr[name], ct))
    return d, arr


def _mmult_lane_plan(a: BlockCsrMatrix, b: BlockCsrMatrix, c: BlockCsrMatrix):
    key = ("mml", id(b), id(c), id(a.support))
    cache = _plan_cache(a)
    hit = cache.get(key)
    if hit is not None:
        return hit[0]
    d, arr = mmult_lane_desc(a, b, c)
    plan = _LanePlan("mm", d, arr)
    cache[key] = (plan, b, c, a.support)
    return plan


def mmult_lane_desc(a: BlockCsrMatrix, b: BlockCsrMatrix, c: BlockCsrMatrix):
    """(bmv_mmult_lane_desc, arrays it points into): host-only."""
    n_rows = a.n_owned_blocks
    n_pa = int(a.row_start[n_rows])
    n_pc = int(c.row_start[n_rows])
    # b's local block row of every a position's column block
    k = a.col_index[:n_pa]
    kb = _local_block_table(b.layout, b.layout.blocks.n_blocks)[k]
    if (kb < 0).any():
        raise PatternError(f"rank {b.layout.rank} holds no ghost of block row {int(k[kb < 0][0])}")
    if (b.local_row_sizes[kb] != a.col_blocks.sizes[k]).any():
        bad = int(k[b.local_row_sizes[kb] != a.col_blocks.sizes[k]][0])
        raise ShapeError(f"row block {bad} of b is incomplete (split ghost group)")
    na = a.row_start[1 : n_rows + 1] - a.row_start[:n_rows]
    nc = c.row_start[1 : n_rows + 1] - c.row_start[:n_rows]
    row, t = _expand(na * nc)
    ncr = nc[row]
    pa = a.row_start[row] + t // np.maximum(ncr, 1)
    pc = c.row_start[row] + t % np.maximum(ncr, 1)
    bkey = kb[pa] * b.col_blocks.n_blocks + c.col_index[pc]
    bkeys = b.local_keys()
    bp = np.searchsorted(bkeys, bkey)
    ok = (bp < bkeys.size) & (bkeys[np.minimum(bp, max(bkeys.size - 1, 0))] == bkey) \
        if bkeys.size else np.zeros(bkey.size, dtype=bool)
    b_off = np.where(ok, b.block_offsets[np.minimum(bp, max(b.block_offsets.size - 2, 0))], -1)
    pair_start = np.concatenate([[0], np.cumsum(na * nc)])[:-1].astype(np.int64)
    arr = dict(
        row_rows=a.local_row_sizes[:n_rows].astype(np.int32),
        a_row_start=a.row_start[: n_rows + 1].astype(np.int64),
        a_off=a.block_offsets[:n_pa].astype(np.int64),
        a_stride=a.col_strides[a.col_index[:n_pa]].astype(np.int32),
        a_mask=_a_lane_masks(a),
        c_row_start=c.row_start[: n_rows + 1].astype(np.int64),
        c_off=c.block_offsets[:n_pc].astype(np.int64),
        c_stride=c.col_strides[c.col_index[:n_pc]].astype(np.int32),
        c_width=c.col_blocks.sizes[c.col_index[:n_pc]].astype(np.int32),
        b_pair_start=pair_start,
        b_off=b_off.astype(np.int64),
        b_stride=b.col_strides[c.col_index[pc]].astype(np.int32),
    )
    arr = {kk: np.ascontiguousarray(v) for kk, v in arr.items()}
    d = _lib.MmultLaneDesc()
    d.n_rows = n_rows
    for name, ct in (("row_rows", _lib.C.c_int32), ("a_row_start", _lib.C.c_int64),
                     ("a_off", _lib.C.c_int64), ("a_stride", _lib.C.c_int32),
                     ("a_mask", _lib.C.c_uint64), ("c_row_start", _lib.C.c_int64),
                     ("c_off", _lib.C.c_int64), ("c_stride", _lib.C.c_int32),
                     ("c_width", _lib.C.c_int32), ("b_pair_start", _lib.C.c_int64),
                     ("b_off", _lib.C.c_int64), ("b_stride", _lib.C.c_int32)):
        setattr(d, name, _lib.ptr(arr[name], ct))
    return d, arr


def mmult(a: BlockCsrMatrix, b: BlockCsrMatrix, c: BlockCsrMatrix, alpha: float = 1.0,
          accumulate: bool = False, counters: OpCounters | None = None):
    """c = alpha * a @ b truncated to c's pattern (K5 on the GPU)."""
    _check_inner(a, b)
    if a.layout.blocks != c.layout.blocks or a.layout.rank != c.layout.rank:
        raise ShapeError("a and c must share row blocking and partitioning")
    if c.col_blocks != b.col_blocks:
        raise ShapeError("b and c must share column blocking")
    if b.state != GHOSTED and b.layout.ghost_groups:
        raise StateError("b must have updated ghost values before mmult")
    c.ensure_owned()
    lib = _lib.require_device()
    if not _deterministic():
        lp = _lane_plan_or_none(_mmult_lane_plan, a, b, c)
        if lp is not None:
            # every owned block of c is written (alpha A B, + old if accumulate);
            # ghost blocks are zeroed like zero_out
            if not accumulate:
                _zero_range(c.data, c._ghost_data_begin, c.data.numel())
            _lib.check(lib.bmv_mmult_lane_run(lp.handle.raw, _lib.dptr(a.data), _lib.dptr(b.data),
                                              _lib.dptr(c.data), float(alpha),
                                              1 if accumulate else 0, 0,
                                              _lib.stream_handle(c.device)), "bmv_mmult_lane_run")
            if counters is not None:
                counters.flops += _mmult_plan(a, b, c).flops
            return
    plan = _mmult_plan(a, b, c)
    zero_len = 0 if accumulate else c.data.numel()
    if not accumulate and plan.full_cover:
        # every owned value is overwritten by the kernel (all owned blocks have
        # products, no padded lanes): only the ghost blocks need zero_out
        _zero_range(c.data, c._ghost_data_begin, c.data.numel())
        zero_len = 0
    _lib.check(lib.bmv_mmult_run(plan.handle.raw, _lib.dptr(a.data), _lib.dptr(b.data),
                                 _lib.dptr(c.data), float(alpha), 1 if accumulate else 0,
                                 zero_len, _lib.stream_handle(c.device)), "bmv_mmult_run")
    if counters is not None:
        counters.flops += plan.flops


def _tmmult_plan(a: BlockCsrMatrix, b: BlockCsrMatrix, c: BlockCsrMatrix):
    key = ("tm", id(b), id(c))
    cache = _plan_cache(a)
    hit = cache.get(key)
    if hit is not None:
        return hit[0]
    arrays, flops = tmmult_plan_arrays(a, b, c, _pj_parts(c.device))
    plan = _TmmultPlan(arrays, flops)
    cache[key] = (plan, b, c)
    return plan


def tmmult_plan_arrays(a: BlockCsrMatrix, b: BlockCsrMatrix, c: BlockCsrMatrix, n_parts: int):
    """K4 streaming plan (include/bmv.h bmv_tmmult_desc): the (A_ik, B_il)
    block products of the owned rows i, in the reference loop order
    (bcsr.py:646-666) inside each output tile; PatternError if C lacks a
    block.  Host-only; returns (arrays, flops)."""
    n_rows = a.n_owned_blocks
    na = a.row_start[1 : n_rows + 1] - a.row_start[:n_rows]
    nb = b.row_start[1 : n_rows + 1] - b.row_start[:n_rows]
    row, t = _expand(na * nb)
    nbr = nb[row]
    pa = a.row_start[row] + t // np.maximum(nbr, 1)
    pb = b.row_start[row] + t % np.maximum(nbr, 1)
    k = a.col_index[pa]
    ck = _local_block_table(c.layout, c.layout.blocks.n_blocks)[k]
    if (ck < 0).any():
        raise PatternError(f"rank {c.layout.rank} holds no ghost of block row {int(k[ck < 0][0])}")
    ell = b.col_index[pb]
    ckey = ck * c.col_blocks.n_blocks + ell
    ckeys = c.local_keys()
    cp = np.searchsorted(ckeys, ckey)
    ok = (cp < ckeys.size) & (ckeys[np.minimum(cp, max(ckeys.size - 1, 0))] == ckey) \
        if ckeys.size else np.zeros(ckey.size, dtype=bool)
    if not ok.all():
        j = int(np.flatnonzero(~ok)[0])
        raise PatternError(f"tmmult destination misses block ({int(k[j])}, {int(ell[j])})")
    if (c.local_row_sizes[c.pos_row[cp]] != a.col_blocks.sizes[k]).any():
        raise ShapeError("tmmult destination row block is incomplete (split ghost group)")
    # ---- streaming plan (csrc/bmv_project.cu) ------------------------------
    a_row_lo = a.block_offsets[a.row_start[:n_rows]]
    a_row_hi = a.block_offsets[a.row_start[1 : n_rows + 1]]
    b_row_lo = b.block_offsets[b.row_start[:n_rows]]
    b_row_hi = b.block_offsets[b.row_start[1 : n_rows + 1]]
    # output tiles: 8x8 pieces of the C blocks (blocks wider than 8 split)
    mr = a.col_blocks.sizes[k].astype(np.int64)
    mc = b.col_blocks.sizes[ell].astype(np.int64)
    tm, tn = (mr + 7) // 8, (mc + 7) // 8
    if n_rows and (int(tm.max(initial=1)) > 16 or int(tn.max(initial=1)) > 16):
        raise ShapeError("tmmult column blocks wider than 128 are not supported")
    tri, q = _expand(tm * tn)
    mt, nt = q // tn[tri], q % tn[tri]
    t_row, t_pa, t_pb, t_cp = row[tri], pa[tri], pb[tri], cp[tri]
    t_key = t_cp * 256 + mt * 16 + nt
    t_rows = a.local_row_sizes[t_row].astype(np.int64)

    # units: whole block rows, or (A group x B group) tiles of a row that
    # exceeds the stage or the tile budget of an item
    cap = _PJ_STAGE
    a_blk = np.diff(a.block_offsets[: int(a.row_start[n_rows]) + 1])
    b_blk = np.diff(b.block_offsets[: int(b.row_start[n_rows]) + 1])
    if a_blk.size or b_blk.size:
        cap = max(cap, 2 * int(max(a_blk.max(initial=0), b_blk.max(initial=0))) + 2)
    cap += cap & 1
    a_tiles = (a.col_blocks.sizes[a.col_index[: int(a.row_start[n_rows])]] + 7) // 8
    b_tiles = (b.col_blocks.sizes[b.col_index[: int(b.row_start[n_rows])]] + 7) // 8
    cs = np.concatenate([[0], np.cumsum(a_tiles)])
    ta_row = cs[a.row_start[1 : n_rows + 1]] - cs[a.row_start[:n_rows]]
    cs = np.concatenate([[0], np.cumsum(b_tiles)])
    tb_row = cs[b.row_start[1 : n_rows + 1]] - cs[b.row_start[:n_rows]]
    a_dbl = a_row_hi - a_row_lo
    b_dbl = b_row_hi - b_row_lo
    unit_dbl_row = a_dbl + (a_dbl & 1) + b_dbl
    big = (unit_dbl_row > cap) | (ta_row * tb_row > _PJ_UNITS)

    def groups(blk, tiles, p0, p1, budget, tmax):
        starts, acc, tacc = [p0], 0, 0
        for pos in range(p0, p1):
            sz, tt = int(blk[pos]), int(tiles[pos])
            if pos > starts[-1] and (acc + sz > budget or tacc + tt > tmax):
                starts.append(pos)
                acc = tacc = 0
            acc += sz
            tacc += tt
        return starts

    u_row = np.arange(n_rows, dtype=np.int64)
    u_a0, u_a1 = a.row_start[:n_rows].copy(), a.row_start[1 : n_rows + 1].copy()
    u_b0, u_b1 = b.row_start[:n_rows].copy(), b.row_start[1 : n_rows + 1].copy()
    u_full = np.ones(n_rows, dtype=bool)
    ag_start = [u_a0.copy()]
    bg_start = [u_b0.copy()]
    row_nbg = np.ones(n_rows, dtype=np.int64)
    extra = []
    for i in np.flatnonzero(big).tolist():
        pa0, pa1, pb0, pb1 = int(u_a0[i]), int(u_a1[i]), int(u_b0[i]), int(u_b1[i])
        half = cap // 2 - 2
        if a_dbl[i] <= half and ta_row[i] <= 4:
            gs_a = [pa0]
            gs_b = groups(b_blk, b_tiles, pb0, pb1, cap - 2 - int(a_dbl[i]), _PJ_UNITS // max(int(ta_row[i]), 1))
        elif b_dbl[i] <= half and tb_row[i] <= 4:
            gs_b = [pb0]
            gs_a = groups(a_blk, a_tiles, pa0, pa1, cap - 2 - int(b_dbl[i]), _PJ_UNITS // max(int(tb_row[i]), 1))
        else:
            gs_a = groups(a_blk, a_tiles, pa0, pa1, half, 4)
            gs_b = groups(b_blk, b_tiles, pb0, pb1, half, 8)
        row_nbg[i] = len(gs_b)
        extra.append((i, gs_a, gs_b, pa1, pb1))
    if extra:
        # replace the big rows' single units by their tiles (row-major, A outer)
        keep = ~big
        rows_l, a0_l, a1_l, b0_l, b1_l = [u_row[keep]], [u_a0[keep]], [u_a1[keep]], [u_b0[keep]], [u_b1[keep]]
        full_l = [u_full[keep]]
        for i, gs_a, gs_b, pa1, pb1 in extra:
            ea, eb = gs_a[1:] + [pa1], gs_b[1:] + [pb1]
            for x0, x1 in zip(gs_a, ea):
                for y0, y1 in zip(gs_b, eb):
                    rows_l.append([i]), a0_l.append([x0]), a1_l.append([x1])
                    b0_l.append([y0]), b1_l.append([y1]), full_l.append([False])
            ag_start.append(np.asarray(gs_a[1:], dtype=np.int64))
            bg_start.append(np.asarray(gs_b[1:], dtype=np.int64))
        u_row = np.concatenate([np.asarray(v, dtype=np.int64) for v in rows_l])
        u_a0 = np.concatenate([np.asarray(v, dtype=np.int64) for v in a0_l])
        u_a1 = np.concatenate([np.asarray(v, dtype=np.int64) for v in a1_l])
        u_b0 = np.concatenate([np.asarray(v, dtype=np.int64) for v in b0_l])
        u_b1 = np.concatenate([np.asarray(v, dtype=np.int64) for v in b1_l])
        u_full = np.concatenate([np.asarray(v, dtype=bool) for v in full_l])
        o = np.lexsort((u_b0, u_a0, u_row))
        u_row, u_a0, u_a1, u_b0, u_b1, u_full = u_row[o], u_a0[o], u_a1[o], u_b0[o], u_b1[o], u_full[o]
    ag_start = np.unique(np.concatenate(ag_start))
    bg_start = np.unique(np.concatenate(bg_start))
    u_base = np.searchsorted(u_row, np.arange(n_rows + 1)).astype(np.int64)
    ua = a.block_offsets[u_a1] - a.block_offsets[u_a0]
    ub = b.block_offsets[u_b1] - b.block_offsets[u_b0]
    u_dbl = ua + (ua & 1) + ub
    u_tiles = np.zeros(u_row.size, dtype=np.int64)
    # parts: balanced by staged doubles, one per SM
    n_parts = max(1, min(int(n_parts), int(u_row.size)))
    total = max(int(u_dbl.sum()), 1)
    before = np.concatenate([[0], np.cumsum(u_dbl)[:-1]]) if u_row.size else np.zeros(0, np.int64)
    u_part = np.minimum(before * n_parts // total, n_parts - 1)
    # triple tile -> unit
    ag = np.searchsorted(ag_start, t_pa, side="right") - 1
    bg = np.searchsorted(bg_start, t_pb, side="right") - 1
    row_ag0 = np.searchsorted(ag_start, a.row_start[:n_rows])
    row_bg0 = np.searchsorted(bg_start, b.row_start[:n_rows])
    t_unit = u_base[t_row] + (ag - row_ag0[t_row]) * row_nbg[t_row] + (bg - row_bg0[t_row])
    np.add.at(u_tiles, t_unit, 1)  # upper bound of distinct tiles per unit
    # sub-chunks: consecutive whole-row units of one part within the stage
    u_sub = np.empty(u_row.size, dtype=np.int64)
    sid, acc, tacc = -1, 0, 0
    dl, tl, fl, pl = u_dbl.tolist(), u_tiles.tolist(), u_full.tolist(), u_part.tolist()
    for j in range(u_row.size):
        if (sid < 0 or not fl[j] or not fl[j - 1] or pl[j] != pl[j - 1]
                or acc + dl[j] > cap or tacc + tl[j] > _PJ_UNITS):
            sid += 1
            acc = tacc = 0
        acc += dl[j]
        tacc += tl[j]
        u_sub[j] = sid
    n_sub = sid + 1
    first_u = np.searchsorted(u_sub, np.arange(n_sub + 1)).astype(np.int64)
    last_u = first_u[1:] - 1
    sub_a = np.stack([a.block_offsets[u_a0[first_u[:-1]]], a.block_offsets[u_a1[last_u]]], 1)
    sub_b = np.stack([b.block_offsets[u_b0[first_u[:-1]]], b.block_offsets[u_b1[last_u]]], 1)
    sub_part = u_part[first_u[:-1]]
    part_sub_start = np.searchsorted(sub_part, np.arange(n_parts + 1)).astype(np.int64)
    t_sub = u_sub[t_unit]
    # items: runs of sub-chunks of one part touching <= _PJ_TILES output tiles
    o = np.argsort(t_sub, kind="stable")
    s_sorted, k_sorted = t_sub[o], t_key[o]
    sub_t0 = np.searchsorted(s_sorted, np.arange(n_sub + 1))
    sub_item = np.empty(n_sub, dtype=np.int64)
    n_items = 0
    for p in range(n_parts):
        cur, end = int(part_sub_start[p]), int(part_sub_start[p + 1])
        while cur < end:
            lo, hi = sub_t0[cur], sub_t0[end]
            _, first = np.unique(k_sorted[lo:hi], return_index=True)
            fs = np.sort(s_sorted[lo:hi][first])
            stop = int(fs[_PJ_TILES]) if fs.size > _PJ_TILES else end
            if stop <= cur:
                raise ShapeError("tmmult sub-chunk touches more output tiles than an item holds")
            sub_item[cur:stop] = n_items
            n_items += 1
            cur = stop
    t_item = sub_item[t_sub]
    # owner warp + register slot of every (item, tile): round robin
    kmax = int(t_key.max(initial=0)) + 1
    ik = t_item * kmax + t_key
    uik, inv = np.unique(ik, return_inverse=True)
    it_item = uik // kmax
    it_rank = np.arange(uik.size) - np.searchsorted(it_item, it_item)
    it_warp, it_slot = it_rank % _PJ_WARPS, it_rank // _PJ_WARPS
    item_slots = np.zeros((n_items, _PJ_WARPS), dtype=np.int64)
    np.add.at(item_slots, (it_item, it_warp), 1)
    # units: the output tiles of one sub-chunk; computing warp by a snake
    # over the units in decreasing work (balanced per sub-chunk)
    sk = t_sub * kmax + t_key
    usk, uinv = np.unique(sk, return_inverse=True)
    u_sub = usk // kmax
    u_work = np.bincount(uinv, weights=t_rows, minlength=usk.size)
    o = np.lexsort((-u_work, u_sub))
    u_rank = np.empty(usk.size, dtype=np.int64)
    u_rank[o] = np.arange(usk.size) - np.searchsorted(u_sub[o], u_sub[o])
    if u_rank.size and int(u_rank.max()) >= _PJ_UNITS:
        raise ShapeError("tmmult sub-chunk touches more output tiles than a stage holds")
    cyc = u_rank % (2 * _PJ_WARPS)
    u_comp = np.where(cyc < _PJ_WARPS, cyc, 2 * _PJ_WARPS - 1 - cyc)
    u_it = np.searchsorted(uik, sub_item[u_sub] * kmax + usk % kmax)
    u_owner, u_slot = it_warp[u_it], it_slot[u_it]
    t_warp, t_unit = u_comp[uinv], u_rank[uinv]
    # triple tiles sorted by (sub, computing warp, unit), reference order inside
    o = np.lexsort((np.arange(t_key.size), t_unit, t_warp, t_sub))
    t_sub, t_warp, t_unit = t_sub[o], t_warp[o], t_unit[o]
    t_pa, t_pb, t_rows, mt, nt = t_pa[o], t_pb[o], t_rows[o], mt[o], nt[o]
    t_mr, t_mc = mr[tri][o], mc[tri][o]
    sub_tri_start = np.searchsorted(t_sub * _PJ_WARPS + t_warp,
                                    np.arange(n_sub * _PJ_WARPS + 1)).astype(np.int64)
    # per sub-chunk: stage = [header][triple tiles][A][B]; metadata = header + tiles
    n_tri_sub = np.bincount(t_sub, minlength=n_sub).astype(np.int64)
    na_sub = sub_a[:, 1] - sub_a[:, 0]
    nb_sub = sub_b[:, 1] - sub_b[:, 0]
    a_off = _PJ_HDR + 16 * n_tri_sub                       # bytes
    b_off = a_off + 8 * (na_sub + (na_sub & 1))
    stage_end = b_off + 8 * nb_sub
    stage_bytes = int(max(int(stage_end.max(initial=0)), _PJ_HDR))
    stage_bytes += (-stage_bytes) % 16
    t_first = sub_tri_start[t_sub * _PJ_WARPS]
    a_soff = a_off[t_sub] // 8 + a.block_offsets[t_pa] - sub_a[t_sub, 0] + 8 * mt
    b_soff = b_off[t_sub] // 8 + b.block_offsets[t_pb] - sub_b[t_sub, 0] + 8 * nt
    acols = np.minimum(8, t_mr - 8 * mt)
    bcols = np.minimum(8, t_mc - 8 * nt)
    a_str = a.col_strides[a.col_index[t_pa]].astype(np.int64)
    b_str = b.col_strides[b.col_index[t_pb]].astype(np.int64)
    if t_rows.size and (int(t_rows.max()) >= 1 << 16 or int(max(a_str.max(), b_str.max())) >= 1 << 16):
        raise ShapeError("tmmult block rows / strides exceed 65535")
    meta_len_sub = _PJ_HDR // 4 + 4 * n_tri_sub          # int32 values
    meta_off = np.concatenate([[0], np.cumsum(meta_len_sub)]).astype(np.int64)
    meta = np.zeros(int(meta_off[-1]), dtype=np.int64)
    hdr = np.zeros((n_sub, _PJ_HDR // 4), dtype=np.int64)
    sts = sub_tri_start[:-1].reshape(n_sub, _PJ_WARPS) if n_sub else np.zeros((0, _PJ_WARPS), np.int64)
    hdr[:, :_PJ_WARPS] = sts - sts[:, :1]
    hdr[:, _PJ_WARPS] = n_tri_sub
    hdr[:, 17] = sub_item
    hdr[:, 18] = np.concatenate([sub_item[1:] != sub_item[:-1], [True]]) if n_sub else 0
    hdr[:, 19] = np.bincount(u_sub, minlength=n_sub)
    hdr[:, 20:20 + _PJ_WARPS] = item_slots[sub_item] if n_sub else 0
    hdr[u_sub, 36 + u_rank] = u_owner | (u_slot << 8)
    meta[(meta_off[:-1, None] + np.arange(_PJ_HDR // 4)[None, :]).ravel()] = hdr.ravel()
    rowpos = meta_off[t_sub] + _PJ_HDR // 4 + 4 * (np.arange(t_sub.size) - t_first)
    meta[rowpos] = a_soff
    meta[rowpos + 1] = b_soff
    meta[rowpos + 2] = t_rows | (t_unit << 16) | (acols << 24) | (bcols << 28)
    meta[rowpos + 3] = a_str | (b_str << 16)
    meta = (meta & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
    # copy lists: metadata, A range, B range
    copies = np.zeros((n_sub, 3, 4), dtype=np.int64)
    copies[:, 0, 1], copies[:, 0, 2] = 4 * meta_len_sub, 4 * meta_off[:-1]
    copies[:, 1, 0], copies[:, 1, 1], copies[:, 1, 2] = a_off, 8 * na_sub | (1 << 28), 8 * sub_a[:, 0]
    copies[:, 2, 0], copies[:, 2, 1], copies[:, 2, 2] = b_off, 8 * nb_sub | (2 << 28) | (1 << 30), \
        8 * sub_b[:, 0]
    copies = _pack_copies(copies.reshape(-1, 4))
    part_entry_start = 3 * part_sub_start
    # output tiles and their partial sources (item order)
    tiles, tinv = np.unique(uik % kmax, return_inverse=True)
    src_order = np.lexsort((it_item, tinv))
    tile_src = ((it_item * _PJ_WARPS + it_warp) * _PJ_SLOTS + it_slot)[src_order]
    tile_src_start = np.searchsorted(tinv[src_order], np.arange(tiles.size + 1)).astype(np.int64)
    tcp, tmt, tnt = tiles // 256, (tiles // 16) % 16, tiles % 16
    c_str = c.col_strides[c.col_index[tcp]].astype(np.int64)
    tile_off = c.block_offsets[tcp] + 8 * tmt * c_str + 8 * tnt
    tr = np.minimum(8, c.local_row_sizes[c.pos_row[tcp]] - 8 * tmt)
    tc = np.minimum(8, c.col_blocks.sizes[c.col_index[tcp]] - 8 * tnt)
    arrays = dict(
        n_parts=n_parts, stage_bytes=stage_bytes, n_sub=n_sub, n_items=n_items,
        part_sub_start=part_sub_start, part_entry_start=part_entry_start,
        copies=copies, meta=meta,
        tile_off=tile_off.astype(np.int64),
        tile_shape=np.ascontiguousarray(np.stack([tr, tc, c_str], 1), dtype=np.int32).ravel(),
        tile_src_start=tile_src_start,
        tile_src=tile_src.astype(np.int64),
    )
    kk = a.col_blocks.sizes[k].astype(np.int64)
    ll = b.col_blocks.sizes[ell].astype(np.int64)
    flops = int(np.sum(2 * kk * a.local_row_sizes[row].astype(np.int64) * ll))
    return arrays, flops


_PJ_WARPS = 16       # consumer warps per CTA (bmv_project.cu kPjWarps)
_PJ_SLOTS = 8        # accumulator tiles per warp (kPjSlots)
_PJ_TILES = _PJ_WARPS * _PJ_SLOTS
_PJ_UNITS = 32       # output tiles per K4 sub-chunk (kPjUnits)
_PJ_HDR = 272        # bytes of the K4 stage header (kPjHeader)
# A + B doubles per K4 stage: 48 KB stages (header + triple tiles included)
# -> 4 stages + 32 KB of unit results per SM
_PJ_STAGE = (49152 - _PJ_HDR - 16 * 4 * _PJ_UNITS) // 8
_PM_STAGE_BYTES = 40960   # K5 stage target (5 stages per SM)
_PM_ROW_TILES = 8         # 8-row tiles per K5 task (kPmRowTiles)


def _pack_copies(entries: np.ndarray) -> np.ndarray:
    """int64 (n, 4) {dst, bytes | src << 28 | last << 30, src byte offset, 0}
    -> the C-ABI copy entries (n x 4 int32, source offset split lo / hi)."""
    out = np.empty((entries.shape[0], 4), dtype=np.int64)
    out[:, 0] = entries[:, 0]
    out[:, 1] = entries[:, 1]
    out[:, 2] = entries[:, 2] & 0xFFFFFFFF
    out[:, 3] = entries[:, 2] >> 32
    if entries.size and (int(entries[:, 0].max()) >= 1 << 31 or
                         int((entries[:, 1] & ((1 << 28) - 1)).max()) >= 1 << 28):
        raise ShapeError("stage copy out of range")
    return np.ascontiguousarray((out & 0xFFFFFFFF).astype(np.uint32).view(np.int32)).ravel()


def _pj_parts(device) -> int:
    """Persistent CTAs of the K4 stream kernel: one per SM."""
    if device is not None and torch.device(device).type == "cuda" and torch.cuda.is_available():
        return int(torch.cuda.get_device_properties(torch.device(device)).multi_processor_count)
    return 148


class _TmmultPlan:
    def __init__(self, arrays, flops):
        self.arrays = arrays
        self.flops = flops
        lib = _lib.load()
        d = _lib.TmmultDesc()
        d.n_parts = int(arrays["n_parts"])
        d.n_warps, d.slots_per_warp = _PJ_WARPS, _PJ_SLOTS
        d.stage_bytes = int(arrays["stage_bytes"])
        d.n_sub, d.n_items = int(arrays["n_sub"]), int(arrays["n_items"])
        d.n_entries = int(arrays["copies"].size // 4)
        d.meta_len = int(arrays["meta"].size)
        d.n_out_tiles = int(arrays["tile_off"].size)
        d.n_src = int(arrays["tile_src"].size)
        for name, ct in (("part_sub_start", _lib.C.c_int64), ("part_entry_start", _lib.C.c_int64),
                         ("copies", _lib.C.c_int32), ("meta", _lib.C.c_int32),
                         ("tile_off", _lib.C.c_int64), ("tile_shape", _lib.C.c_int32),
                         ("tile_src_start", _lib.C.c_int64), ("tile_src", _lib.C.c_int64)):
            arrays[name] = np.ascontiguousarray(arrays[name])
            setattr(d, name, _lib.ptr(arrays[name], ct))
        raw = _lib.C.c_void_p()
        _lib.check(lib.bmv_tmmult_create(_lib.C.byref(d), _lib.C.byref(raw)), "bmv_tmmult_create")
        self.handle = _lib.Handle("bmv_tmmult_destroy", raw)


def tmmult(a: BlockCsrMatrix, b: BlockCsrMatrix, c: BlockCsrMatrix,
           counters: OpCounters | None = None):
    """c = a^T @ b over owned rows (K4 on the GPU), then compress c."""
    if a.layout.blocks != b.layout.blocks or a.layout.rank != b.layout.rank:
        raise ShapeError("a and b must share row blocking and partitioning")
    if not np.array_equal(c.layout.blocks.sizes, a.col_blocks.sizes):
        raise ShapeError("c's row blocking must equal a's column blocking")
    if c.col_blocks != b.col_blocks:
        raise ShapeError("c's column blocking must equal b's")
    c.ensure_owned()
    lib = _lib.require_device()
    if not _deterministic():
        lp = _lane_plan_or_none(_tmmult_lane_plan, a, b, c)
        if lp is not None:
            _lib.check(lib.bmv_tmmult_lane_run(lp.handle.raw, _lib.dptr(a.data), _lib.dptr(b.data),
                                               _lib.dptr(c.data), c.data.numel(),
                                               _lib.stream_handle(c.device)), "bmv_tmmult_lane_run")
            if counters is not None:
                counters.flops += _tmmult_plan(a, b, c).flops
            c.compress()
            return
    plan = _tmmult_plan(a, b, c)
    _lib.check(lib.bmv_tmmult_run(plan.handle.raw, _lib.dptr(a.data), _lib.dptr(b.data),
                                  _lib.dptr(c.data), c.data.numel(),
                                  _lib.stream_handle(c.device)), "bmv_tmmult_run")
    if counters is not None:
        counters.flops += plan.flops
    c.compress()


def tr_tmmult(d: BlockCsrMatrix, g: BlockCsrMatrix, counters: OpCounters | None = None) -> float:
    """tr(d^T g) over common stored blocks, reduced over ranks (reference
    bcsr.py:670-698; the line-search slope of the OM step)."""
    if d.layout.blocks != g.layout.blocks or d.layout.rank != g.layout.rank:
        raise ShapeError("operands must share row blocking and partitioning")
    if d.col_blocks != g.col_blocks:
        raise ShapeError("operands must share column blocking")
    if d.pattern is g.pattern and d.lane_width == g.lane_width:
        # same blocks at the same offsets: one dot over the owned values (the
        # padded lanes are exact zeros, the layout invariant)
        n = d.n_owned_values
        local = float(torch.dot(d.data[:n], g.data[:n]).item()) if n else 0.0
        if counters is not None:
            counters.flops += 2 * n
    else:
        gi, di = _glue_index(("tr_tmmult", id(g.pattern), id(d.pattern), id(d.layout)), g,
                             lambda: _common_entries(g, d)[:2])
        local = float(torch.dot(d.data[di], g.data[gi]).item()) if di.numel() else 0.0
        if counters is not None:
            counters.flops += 2 * int(di.numel())
    if d.ctx is not None:
        return float(d.ctx.allreduce_sum(local))
    return local


def tr_mult(t: BlockCsrMatrix, h: BlockCsrMatrix, counters: OpCounters | None = None) -> float:
    """tr(t h) over stored blocks, reduced over ranks; h must be ghosted for
    remote rows (reference bcsr.py:701-725; the OM energy)."""
    if not np.array_equal(t.col_blocks.sizes, h.layout.blocks.sizes):
        raise ShapeError("inner blockings differ")
    if not np.array_equal(t.layout.blocks.sizes, h.col_blocks.sizes):
        raise ShapeError("outer blockings differ")
    if h.state != GHOSTED and h.layout.ghost_groups:
        raise StateError("h must have updated ghost values before tr_mult")

    def build():
        ti, hi = [], []
        for lb in range(t.n_owned_blocks):
            k = t.layout.global_block_of_local(lb)
            for pos in range(int(t.row_start[lb]), int(t.row_start[lb + 1])):
                ell = int(t.col_index[pos])
                hl = h.layout.local_block_of_global(ell)
                if hl < 0:
                    continue
                hpos = h.block_pos_local(hl, k)
                if hpos < 0:
                    continue
                nr, nc = int(t.local_row_sizes[lb]), int(t.col_blocks.sizes[ell])
                r, c = np.meshgrid(np.arange(nr), np.arange(nc), indexing="ij")
                ti.append(int(t.block_offsets[pos]) + r.ravel() * int(t.col_strides[ell]) + c.ravel())
                hi.append(int(h.block_offsets[hpos]) + c.ravel() * int(h.col_strides[k]) + r.ravel())
        z = np.zeros(0, dtype=np.int64)
        return (np.concatenate(ti) if ti else z, np.concatenate(hi) if hi else z)

    ti, hi = _glue_index(("tr_mult", id(t.pattern), id(h.pattern), id(t.layout), id(h.layout)), t,
                         build)
    local = float(torch.dot(t.data[ti], h.data[hi]).item()) if ti.numel() else 0.0
    if counters is not None:
        counters.flops += 2 * int(ti.numel())
    if t.ctx is not None:
        return float(t.ctx.allreduce_sum(local))
    return local


# -- serialisation --------------------------------------------------------------------


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
    """Little-endian fp64 dump of the whole value array (reference format)."""
    return m.data.detach().cpu().numpy().astype("<f8").tobytes()


def load_value_bytes(m: BlockCsrMatrix, raw: bytes):
    arr = np.frombuffer(raw, dtype="<f8")
    if arr.size != m.data.numel():
        raise ShapeError(f"value buffer holds {arr.size} reals, matrix stores {m.data.numel()}")
    m.data.copy_(torch.from_numpy(arr.astype(np.float64)))
