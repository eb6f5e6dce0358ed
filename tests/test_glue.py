"""Element-wise glue of the OM composition (reference bcsr.py:526-577,
670-725): scale_add, copy_pattern_subset, add_scaled_identity, tr_tmmult,
tr_mult on cached index maps, against dense numpy on host matrices."""

import numpy as np
import torch

from _helpers import Small
from paper_1907_01005_b200 import bcsr as B
from paper_1907_01005_b200.comm import serial_context
from paper_1907_01005_b200.problem import hashed_entries

CENTERS = np.asarray([[1.0, 1.0, 1.0], [3.0, 3.0, 2.0], [2.0, 1.5, 3.0], [0.5, 3.2, 0.7]])


def _mats():
    s = Small((4, 4, 4), (1.0, 1.0, 1.0), 1, 2, CENTERS, 1.6, 3, 3)
    ctx = serial_context("cpu")
    rl, _, x, hx = s.operands(ctx, "cpu")
    s.fill(x, 5, attach=False)
    hx.fill_owned_entries(lambda r, c: hashed_entries(9, r, c))
    sm, cm, _ = s.projection_operands(ctx, "cpu", rl)
    return x, hx, sm, cm


def test_scale_add_and_copy_subset():
    x, hx, _, _ = _mats()
    xd, hd = x.to_dense_owned(), hx.to_dense_owned()
    B.scale_add(hx, 0.5, x, -2.0)  # x's pattern sits inside the grown one
    assert np.allclose(hx.to_dense_owned(), 0.5 * hd - 2.0 * xd, rtol=0, atol=1e-14)
    y = B.BlockCsrMatrix(x.pattern, x.layout, x.ctx, x.lane_width, "cpu")
    B.copy_pattern_subset(y, hx)
    assert np.array_equal(y.to_dense_owned(),
                          np.where(x.pattern.entry_mask(), hx.to_dense_owned(), 0.0))


def test_identity_and_traces():
    x, hx, sm, cm = _mats()
    cd = cm.to_dense_owned()
    B.add_scaled_identity(cm, 2.0)
    assert np.allclose(cm.to_dense_owned(), cd + 2.0 * np.eye(cd.shape[0]), atol=1e-15)
    xd, hd = x.to_dense_owned(), hx.to_dense_owned()
    got = B.tr_tmmult(x, hx)
    want = float(np.sum(xd * np.where(x.pattern.entry_mask(), hd, 0.0)))
    assert abs(got - want) <= 1e-12 * max(1.0, abs(want))
    sm.data.copy_(torch.from_numpy(np.random.default_rng(3).standard_normal(sm.data.numel())))
    t, h = sm.to_dense_owned(), cm.to_dense_owned()
    mask_t = sm.pattern.entry_mask()
    got = B.tr_mult(sm, cm)
    want = float(np.sum(np.where(mask_t, t, 0.0) * h.T))
    assert abs(got - want) <= 1e-12 * max(1.0, abs(want))
