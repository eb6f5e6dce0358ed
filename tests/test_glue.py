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


CENTERS6 = np.asarray([[1.0, 1.0, 1.0], [3.0, 3.0, 2.0], [2.0, 1.5, 3.0], [0.5, 3.2, 0.7],
                      [4.5, 4.5, 4.5], [5.0, 1.0, 3.0]])


def _compact():
    """Coarse level 0, one vector per centre: supports cover 38 % of the
    stored block columns, so compact and full storage differ."""
    s = Small((6, 6, 6), (1.0, 1.0, 1.0), 0, 2, CENTERS6, 1.6, 3, 1)
    ctx = serial_context("cpu")
    rl, op, x, hx = s.operands(ctx, "cpu")
    s.fill(x, 5, attach=True)
    return s, op, x, hx


def test_copy_keeps_storage_and_writes_clear_the_support_declaration():
    """A copy stores the same columns (its structural zeros are part of the
    storage); a write whose source is not declared with the same support
    drops the declaration, so K1 falls back to every stored column instead of
    silently skipping pairs (copy() + scale_add)."""
    import pytest

    from paper_1907_01005_b200.errors import ShapeError

    s, op, x, hx = _compact()
    x2 = x.copy()
    assert x2.support is x.support and x2.slab is x.slab
    assert np.array_equal(x2.to_dense_owned(), x.to_dense_owned())
    B.scale_add(x2, 1.0, x, -0.5)  # same support: declaration kept
    assert x2.support is x.support
    assert np.allclose(x2.to_dense_owned(), 0.5 * x.to_dense_owned(), atol=1e-15)
    d = x.copy()
    d.fill_owned_entries(lambda r, c: hashed_entries(11, r, c))  # values off the support
    assert d.support is None and d.slab is x.slab
    B.scale_add(x2, 1.0, d, 1.0)
    assert x2.support is None  # no longer a valid declaration
    full = B.BlockCsrMatrix(x.pattern, x.layout, x.ctx, x.lane_width, "cpu")
    full.fill_owned_entries(lambda r, c: hashed_entries(12, r, c))
    with pytest.raises(ShapeError):
        B.scale_add(x2, 1.0, full, 1.0)  # stores entries x2 has no room for


def test_attach_support_relayouts_and_checks():
    import pytest

    from paper_1907_01005_b200.errors import ConsistencyError
    from paper_1907_01005_b200.support import attach_support

    s, op, x, hx = _compact()
    full = B.BlockCsrMatrix(x.pattern, x.layout, x.ctx, x.lane_width, "cpu")
    s.fill(full, 5, attach=False)
    assert full.support is None and full.data.numel() > x.data.numel()
    attach_support(full, s.support, check=True)
    assert full.data.numel() == x.data.numel()
    assert np.array_equal(full.to_dense_owned(), x.to_dense_owned())
    bad = B.BlockCsrMatrix(x.pattern, x.layout, x.ctx, x.lane_width, "cpu")
    bad.fill_owned_entries(lambda r, c: hashed_entries(3, r, c))
    with pytest.raises(ConsistencyError):
        attach_support(bad, s.support, check=True)


def test_image_columns_cover_the_operator_reach():
    """H X stored with op.image_columns(support) holds every column some cell
    couples to its rows, and no more than the full grown pattern."""
    s, op, x, hx = _compact()
    img = B.BlockCsrMatrix(hx.pattern, hx.layout, hx.ctx, hx.lane_width, "cpu",
                           columns=op.image_columns(x.columns))
    act = op.active_pairs(s.support)
    assert img.data.numel() < hx.data.numel()
    # every (cell, column) pair reaches every block row of the cell
    p_cell = np.repeat(np.arange(act.shape[0]), np.diff(act.indptr))
    g0, g1 = op.cell_gstart[p_cell], op.cell_gstart[p_cell + 1]
    for c, a, b in zip(act.indices, g0, g1):
        lbs = op.grp_block[a:b]
        assert (img.slab.slots(lbs, np.full(lbs.size, c)) >= 0).all()


def test_unknown_variant_rejected():
    import pytest

    from paper_1907_01005_b200.errors import ShapeError
    from paper_1907_01005_b200.matfree import hamiltonian_operator

    s, op, x, hx = _compact()
    with pytest.raises(ShapeError):
        op.apply(hamiltonian_operator(None), x, hx, variant="stencil")


def test_base_element_matrix_matches_oracle():
    """Kinetic part of the gemm variant's element matrix against the oracle's
    direct quadrature (reference element_matrices, matfree.py:375-397)."""
    from oracle import numpy_oracle as O

    s, op, x, hx = _compact()
    got = op._base_element_matrix("hamiltonian")
    want = O.element_matrix(op.shape.degree, op.mesh.spacing, "h", None)
    assert np.allclose(got, want, rtol=1e-13, atol=1e-13 * np.abs(want).max())
