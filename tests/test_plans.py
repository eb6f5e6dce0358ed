"""K4 / K5 chunk plans on CPU: emulate the kernels over the native host plan
(tests/_plan_emul.py) and compare with dense products of the same data.

Covers narrow and wide column blocks, lane widths, compact (support) and
full storage, few / many parts, small stages (chunks split down to single
rows) and long block rows split into row ranges.
"""

import numpy as np
import pytest
import torch

from _helpers import Small
from _plan_emul import emulate_mmult, emulate_tmmult
from paper_1907_01005_b200 import spmm
from paper_1907_01005_b200.comm import serial_context
from paper_1907_01005_b200.problem import hashed_entries

CENTERS = np.asarray([[1.0, 1.0, 1.0], [3.0, 3.0, 2.0], [2.0, 1.5, 3.0], [0.5, 3.2, 0.7]])


def _setup(block_size, lane_width, compact, level=1, degree=2):
    s = Small((4, 4, 4), (1.0, 1.0, 1.0), level, degree, CENTERS, 1.6, block_size, 3)
    ctx = serial_context("cpu")
    rl, op, x, hx = s.operands(ctx, "cpu", lane_width)
    s.fill(x, 5, attach=compact)
    if compact:
        hx.relayout(op.image_columns(s.support))
    hx.fill_owned_entries(lambda r, c: hashed_entries(9, r, c))
    sm, cm, xc = s.projection_operands(ctx, "cpu", rl, lane_width)
    return x, hx, sm, cm, xc


def _shape(monkeypatch, stage, rows):
    monkeypatch.setattr(spmm, "chunk_bytes", lambda kind, variant=0: (stage, stage - 1024))
    monkeypatch.setattr(spmm, "K4_MAX_ROWS", rows)


def _plan(kind, a, b, c, n_parts):
    from paper_1907_01005_b200 import _plan as NP

    n = a.n_owned_blocks
    if kind == 4:
        return NP.chunk_plan(4, a.local_row_sizes[:n], spmm._Owned(a), spmm._Owned(b),
                             a.col_blocks.starts, spmm._local_table(c.layout, c.layout.blocks.n_blocks),
                             c.slab, spmm.K4_MAX_ROWS, spmm.MAX_BLOCK_ROWS, spmm.chunk_bytes(4)[1],
                             spmm.chunk_bytes(4)[0], n_parts)
    return NP.chunk_plan(5, a.local_row_sizes[:n], spmm._Owned(a), spmm._Owned(c),
                         a.col_blocks.starts, spmm._local_table(b.layout, b.layout.blocks.n_blocks),
                         b.slab, spmm.K5_MAX_ROWS, spmm.MAX_BLOCK_ROWS, spmm.chunk_bytes(5)[1],
                         spmm.chunk_bytes(5)[0], n_parts)


@pytest.mark.parametrize("block_size,lane_width", [(3, 8), (8, 8), (12, 8), (3, 4)])
@pytest.mark.parametrize("compact", [False, True])
@pytest.mark.parametrize("n_parts", [1, 7, 148])
@pytest.mark.parametrize("stage,rows", [(14208, 64), (2048, 8)])
def test_tmmult_chunk_emulation(monkeypatch, block_size, lane_width, compact, n_parts, stage, rows):
    _shape(monkeypatch, stage, rows)
    x, hx, sm, _, _ = _setup(block_size, lane_width, compact)
    arr = _plan(4, x, hx, sm, n_parts)
    got = emulate_tmmult(arr, x.data.numpy(), hx.data.numpy(), sm.data.numel())
    sm.data.copy_(torch.from_numpy(got))
    want = x.to_dense_owned().T @ hx.to_dense_owned()
    assert np.allclose(sm.to_dense_owned(), want, rtol=1e-13, atol=1e-13 * np.abs(want).max())


@pytest.mark.parametrize("block_size,lane_width", [(3, 8), (8, 8), (12, 8), (3, 4)])
@pytest.mark.parametrize("compact", [False, True])
@pytest.mark.parametrize("n_parts", [1, 7])
@pytest.mark.parametrize("accumulate", [False, True])
def test_mmult_chunk_emulation(block_size, lane_width, compact, n_parts, accumulate):
    x, _, _, cm, xc = _setup(block_size, lane_width, compact)
    if compact:
        xc.relayout(x.columns)
    xc.fill_owned_entries(lambda r, c: hashed_entries(3, r, c))
    before = xc.to_dense_owned()
    arr = _plan(5, x, cm, xc, n_parts)
    got = emulate_mmult(arr, x.data.numpy(), cm.data.numpy(), xc.data.numpy(), -0.5, accumulate)
    xc.data.copy_(torch.from_numpy(got))
    stored = np.zeros_like(before, dtype=bool)
    _, grow, gcol = xc._valid_owned_index()
    stored[grow, gcol] = True
    want = np.where(stored, -0.5 * (x.to_dense_owned() @ cm.to_dense_owned()), 0.0)
    if accumulate:
        want = want + before
    assert np.allclose(xc.to_dense_owned(), want, rtol=1e-13, atol=1e-13 * np.abs(want).max())


def test_long_block_rows_split_into_row_ranges(monkeypatch):
    """Coarse level 0 at degree 4: block rows of up to 125 rows > 64 (split)."""
    monkeypatch.setattr(spmm, "K4_MAX_ROWS", 64)
    x, hx, sm, _, _ = _setup(3, 8, True, level=0, degree=4)
    assert int(x.local_row_sizes.max()) > spmm.K4_MAX_ROWS
    arr = _plan(4, x, hx, sm, 7)
    got = emulate_tmmult(arr, x.data.numpy(), hx.data.numpy(), sm.data.numel())
    sm.data.copy_(torch.from_numpy(got))
    want = x.to_dense_owned().T @ hx.to_dense_owned()
    assert np.allclose(sm.to_dense_owned(), want, rtol=1e-13, atol=1e-13 * np.abs(want).max())


@pytest.mark.parametrize("stage", [9472, 7168, 4096])
def test_wide_rows_split_when_meta_and_rows_exceed_a_buffer(monkeypatch, stage):
    """Six wide supports, full storage (48 columns per row): the greedy row
    pieces plus their meta exceed a buffer and are halved again (a piece
    once lost its second half there)."""
    centers = np.asarray([[1.0, 1.0, 1.0], [3.0, 3.0, 2.0], [2.0, 1.5, 3.0], [0.5, 3.2, 0.7],
                          [2.5, 2.5, 0.5], [1.5, 3.5, 2.5]])
    monkeypatch.setattr(spmm, "chunk_bytes", lambda kind, variant=0: (stage, stage - 1536))
    s = Small((4, 4, 4), (1.0, 1.0, 1.0), 1, 2, centers, 3.5, 8, 8)
    ctx = serial_context("cpu")
    rl, _, x, hx = s.operands(ctx, "cpu")
    s.fill(x, 5, attach=False)
    hx.fill_owned_entries(lambda r, c: hashed_entries(9, r, c))
    sm, cm, xc = s.projection_operands(ctx, "cpu", rl)
    arr = _plan(4, x, hx, sm, 5)
    n = x.n_owned_blocks
    rows_planned = sum(int(arr["meta"][int(m0) + 1]) for m0 in arr["chunk_meta"][:-1])
    assert rows_planned == int(x.local_row_sizes[:n].sum())
    got = emulate_tmmult(arr, x.data.numpy(), hx.data.numpy(), sm.data.numel())
    sm.data.copy_(torch.from_numpy(got))
    want = x.to_dense_owned().T @ hx.to_dense_owned()
    assert np.allclose(sm.to_dense_owned(), want, rtol=1e-13, atol=1e-13 * np.abs(want).max())
    arr = _plan(5, x, cm, xc, 5)
    got = emulate_mmult(arr, x.data.numpy(), cm.data.numpy(), xc.data.numpy(), 0.75, False)
    xc.data.copy_(torch.from_numpy(got))
    stored = np.zeros(xc.to_dense_owned().shape, dtype=bool)
    _, grow, gcol = xc._valid_owned_index()
    stored[grow, gcol] = True
    want = np.where(stored, 0.75 * (x.to_dense_owned() @ cm.to_dense_owned()), 0.0)
    assert np.allclose(xc.to_dense_owned(), want, rtol=1e-13, atol=1e-13 * np.abs(want).max())
