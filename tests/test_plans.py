"""K4 / K5 streaming plans on CPU: emulate the kernels over the host plan
(tests/_plan_emul.py) and compare with dense products of the same data.

Covers wide column blocks (tiles split 2 x 2), narrow lane widths (strides
< 8, guarded fragment loads), many / few parts and rows split into
A-group x B-group tiles (small stage).
"""

import numpy as np
import pytest

from _helpers import Small
from _plan_emul import emulate_mmult, emulate_tmmult
from paper_1907_01005_b200 import bcsr as B
from paper_1907_01005_b200.comm import serial_context
from paper_1907_01005_b200.problem import hashed_entries

CENTERS = np.asarray([[1.0, 1.0, 1.0], [3.0, 3.0, 2.0], [2.0, 1.5, 3.0], [0.5, 3.2, 0.7]])


def _setup(block_size, lane_width):
    s = Small((4, 4, 4), (1.0, 1.0, 1.0), 1, 2, CENTERS, 1.6, block_size, 3)
    ctx = serial_context("cpu")
    rl, _, x, hx = s.operands(ctx, "cpu", lane_width)
    s.fill(x, 5, attach=False)
    hx.fill_owned_entries(lambda r, c: hashed_entries(9, r, c))
    sm, cm, xc = s.projection_operands(ctx, "cpu", rl, lane_width)
    return x, hx, sm, cm, xc


@pytest.mark.parametrize("block_size,lane_width", [(3, 8), (8, 8), (12, 8), (3, 4), (5, 2)])
@pytest.mark.parametrize("n_parts", [1, 7, 148])
@pytest.mark.parametrize("stage", [4864, 96])
def test_tmmult_plan_emulation(monkeypatch, block_size, lane_width, n_parts, stage):
    monkeypatch.setattr(B, "_PJ_STAGE", stage)
    x, hx, sm, _, _ = _setup(block_size, lane_width)
    arr, flops = B.tmmult_plan_arrays(x, hx, sm, n_parts)
    got = emulate_tmmult(arr, x.data.numpy(), hx.data.numpy(), sm.data.numel())
    sm.data.copy_(__import__("torch").from_numpy(got))
    want = x.to_dense_owned().T @ hx.to_dense_owned()
    assert np.allclose(sm.to_dense_owned(), want, rtol=1e-13, atol=1e-13 * np.abs(want).max())
    assert flops > 0


@pytest.mark.parametrize("block_size,lane_width", [(3, 8), (8, 8), (12, 8), (3, 4), (5, 2)])
@pytest.mark.parametrize("n_parts", [1, 7, 148])
@pytest.mark.parametrize("accumulate", [False, True])
def test_mmult_plan_emulation(block_size, lane_width, n_parts, accumulate):
    import torch

    x, _, _, cm, xc = _setup(block_size, lane_width)
    xc.fill_owned_entries(lambda r, c: hashed_entries(3, r, c))
    before = xc.to_dense_owned()
    arr, n_out, n_pairs, flops, _ = B.mmult_plan_arrays(x, cm, xc, n_parts)
    got = emulate_mmult(arr, x.data.numpy(), cm.data.numpy(), xc.data.numpy(), -0.5, accumulate)
    xc.data.copy_(torch.from_numpy(got))
    mask = xc.pattern.entry_mask()
    want = np.where(mask, -0.5 * (x.to_dense_owned() @ cm.to_dense_owned()), 0.0)
    if accumulate:
        want = want + before
    assert np.allclose(xc.to_dense_owned(), want, rtol=1e-13, atol=1e-13 * np.abs(want).max())
    assert n_pairs > 0 and flops > 0 and n_out > 0


# -- lane-compacted K4 / K5 (csrc/bmv_spmm_lane.cu): planner in the library,
#    kernels emulated on CPU over the host stage stream ----------------------


@pytest.fixture(params=["auto", "1", "1:run3"])
def interleave(request, monkeypatch):
    """Lane plans: the planner's chunk assignment, or chunks interleaved over
    the CTAs with one accumulator item per chunk (short block rows), or runs of
    3 consecutive chunks per CTA turn sharing one K4 item."""
    monkeypatch.delenv("BMV_LANE_RUN", raising=False)
    if request.param == "auto":
        monkeypatch.delenv("BMV_LANE_INTERLEAVE", raising=False)
    else:
        monkeypatch.setenv("BMV_LANE_INTERLEAVE", "1")
        monkeypatch.setenv("BMV_LANE_RUN", "3" if request.param.endswith("run3") else "1")
    return request.param


@pytest.mark.parametrize("block_size,lane_width", [(3, 8), (8, 8), (12, 8), (3, 4), (5, 2)])
@pytest.mark.parametrize("attach", [False, True])
@pytest.mark.parametrize("n_parts", [1, 7])
def test_tmmult_lane_plan_emulation(block_size, lane_width, attach, n_parts, interleave):
    from _plan_emul import emulate_tmmult_lane

    s = Small((4, 4, 4), (1.0, 1.0, 1.0), 1, 2, CENTERS, 1.6, block_size, 3)
    ctx = serial_context("cpu")
    rl, _, x, hx = s.operands(ctx, "cpu", lane_width)
    s.fill(x, 5, attach=attach)
    hx.fill_owned_entries(lambda r, c: hashed_entries(9, r, c))
    sm, _, _ = s.projection_operands(ctx, "cpu", rl, lane_width)
    d, keep = B.tmmult_lane_desc(x, hx, sm)
    arr = B.lane_plan_host(4, d, n_parts)
    got = emulate_tmmult_lane(arr, x.data.numpy(), hx.data.numpy(), sm.data.numel())
    import torch

    sm.data.copy_(torch.from_numpy(got))
    want = x.to_dense_owned().T @ hx.to_dense_owned()
    assert np.allclose(sm.to_dense_owned(), want, rtol=1e-13, atol=1e-13 * np.abs(want).max())


@pytest.mark.parametrize("block_size,lane_width", [(3, 8), (8, 8), (12, 8), (3, 4), (5, 2)])
@pytest.mark.parametrize("attach", [False, True])
@pytest.mark.parametrize("accumulate", [False, True])
def test_mmult_lane_plan_emulation(block_size, lane_width, attach, accumulate, interleave):
    import torch

    from _plan_emul import emulate_mmult_lane

    s = Small((4, 4, 4), (1.0, 1.0, 1.0), 1, 2, CENTERS, 1.6, block_size, 3)
    ctx = serial_context("cpu")
    rl, _, x, hx = s.operands(ctx, "cpu", lane_width)
    s.fill(x, 5, attach=attach)
    _, cm, xc = s.projection_operands(ctx, "cpu", rl, lane_width)
    xc.fill_owned_entries(lambda r, c: hashed_entries(3, r, c))
    before = xc.to_dense_owned()
    d, keep = B.mmult_lane_desc(x, cm, xc)
    arr = B.lane_plan_host(5, d, 3)
    got = emulate_mmult_lane(arr, x.data.numpy(), cm.data.numpy(), xc.data.numpy(), -0.5,
                             accumulate)
    xc.data.copy_(torch.from_numpy(got))
    want = np.where(xc.pattern.entry_mask(), -0.5 * (x.to_dense_owned() @ cm.to_dense_owned()), 0.0)
    if accumulate:
        want = want + before
    assert np.allclose(xc.to_dense_owned(), want, rtol=1e-13, atol=1e-13 * np.abs(want).max())


@pytest.mark.parametrize("attach", [False, True])
def test_mmult_lane_many_columns_per_row(attach):
    """Rows with more than 32 active columns: K5 passes over k-step groups and
    adds to the values it wrote (k5_lane_kernel), emulated."""
    import torch

    from _plan_emul import emulate_mmult_lane

    centers = np.asarray([[1.0, 1.0, 1.0], [3.0, 3.0, 2.0], [2.0, 1.5, 3.0], [0.5, 3.2, 0.7],
                          [2.5, 2.5, 0.5], [1.5, 3.5, 2.5]])
    s = Small((4, 4, 4), (1.0, 1.0, 1.0), 1, 2, centers, 3.5, 8, 8)  # 48 columns, wide supports
    ctx = serial_context("cpu")
    rl, _, x, hx = s.operands(ctx, "cpu")
    s.fill(x, 5, attach=attach)
    _, cm, xc = s.projection_operands(ctx, "cpu", rl)
    d, keep = B.mmult_lane_desc(x, cm, xc)
    arr = B.lane_plan_host(5, d, 3)
    ks_max = 0
    meta = arr["meta"]
    cps = arr["copies"].astype(np.int64) & 0xFFFFFFFF
    for e in cps:
        if ((e[1] >> 28) & 3) == 0:
            off = int(e[2] | (e[3] << 32)) // 4
            n_t, toff = int(meta[off]), int(meta[off + 1])
            for t in range(n_t):
                r0 = off + int(meta[off + toff + t])
                ks_max = max(ks_max, int(meta[r0 + 3]) >> 16)
    assert ks_max > 8  # exercises several k-step groups
    got = emulate_mmult_lane(arr, x.data.numpy(), cm.data.numpy(), xc.data.numpy(), 0.75, False)
    xc.data.copy_(torch.from_numpy(got))
    want = np.where(xc.pattern.entry_mask(), 0.75 * (x.to_dense_owned() @ cm.to_dense_owned()), 0.0)
    assert np.allclose(xc.to_dense_owned(), want, rtol=1e-13, atol=1e-13 * np.abs(want).max())
