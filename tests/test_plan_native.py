"""The native plan builder (libbmvplan.so, include/bmv_plan.h) against the numpy
restatements it replaces: bit-identical arrays on the smoke, random and full-size
layouts (CPU only; matrices live on the CPU)."""

import numpy as np
import pytest

from paper_1907_01005_b200 import _plan
from paper_1907_01005_b200 import problem as P
from paper_1907_01005_b200.bcsr import BlockCsrMatrix
from paper_1907_01005_b200.comm import run_ranks, serial_context
from paper_1907_01005_b200.matfree import _first_occurrence_groups_numpy, make_dof_layout


def test_library_exports():
    lib = _plan.load()
    assert lib.bmvp_version() == 1
    for name in ("bmvp_hash_fill", "bmvp_owned_entries_count", "bmvp_owned_entries_fill",
                 "bmvp_first_groups_count", "bmvp_first_groups_fill"):
        assert hasattr(lib, name)


def test_hash_fill_matches_numpy():
    rng = np.random.default_rng(3)
    rows = rng.integers(0, 1 << 40, 100_003)
    cols = rng.integers(0, 4096, rows.size)
    cmap = rng.permutation(4096)
    for seed in (0, 1, 7, -5, (1 << 63) + 11):
        want = 2.0 * P.hashed_entries(seed, rows, cmap[cols])
        got = _plan.hash_fill(seed, rows, cols, cmap, None, 2.0)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    flat = rng.permutation(rows.size)
    out = np.zeros(rows.size)
    _plan.hash_fill(1, rows, cols, None, flat, 1.0, out)
    want = np.zeros(rows.size)
    want[flat] = P.hashed_entries(1, rows, cols)
    assert np.array_equal(out, want)


def _groups_equal(lb):
    a = _plan.first_occurrence_groups(lb)
    b = _first_occurrence_groups_numpy(lb)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_first_groups_random():
    rng = np.random.default_rng(5)
    for n3 in (8, 27, 125):
        _groups_equal(rng.integers(0, 9, (300, n3)))
        _groups_equal(np.zeros((4, n3), dtype=np.int64))


def _owned_check(ctx, prob):
    if True:
        layout = make_dof_layout(ctx, prob.mesh, prob.partition, prob.numbering)
        m = BlockCsrMatrix(prob.pattern, layout, ctx, prob.cfg.lane_width, "cpu")
        a = _plan.owned_entries(prob.column_support, m)
        b = prob.column_support._owned_entries_numpy(m)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
        c, _, _ = prob.column_support.owned_entries(m)
        assert np.array_equal(c, b[0])
        # the same offsets in the layout the CellOperator builds
        op_groups = P.CellOperator(prob.mesh, prob.partition, prob.numbering, layout)
        _groups_equal(op_groups._lb)


@pytest.mark.parametrize("name", ["smoke", "q2"])
def test_owned_entries_and_groups_configs(name):
    _owned_check(serial_context("cpu"), P.build_problem(name))


@pytest.mark.parametrize("n_ranks", [2, 4])
def test_owned_entries_and_groups_ranks(n_ranks):
    prob = P.build_problem("smoke", n_ranks)
    run_ranks(n_ranks, lambda ctx: _owned_check(ctx, prob), device="cpu")


def test_fill_multivector_native_equals_numpy(monkeypatch):
    prob = P.build_problem("smoke")
    st = P.make_rank_setup(serial_context("cpu"), prob, device="cpu")
    got = st.x.data.numpy().copy()
    monkeypatch.setenv("BMV_PLAN_NATIVE", "0")
    prob2 = P.build_problem("smoke")
    st2 = P.make_rank_setup(serial_context("cpu"), prob2, device="cpu")
    assert np.array_equal(got, st2.x.data.numpy())
    assert np.array_equal(st.op.cell_slots, st2.op.cell_slots)


def test_blocks_of_matches_searchsorted():
    rng = np.random.default_rng(9)
    starts = np.concatenate([[5], 5 + np.cumsum(rng.integers(1, 70, 5000))])
    idx = rng.integers(starts[0], starts[-1], 300_001)
    b, off = _plan.blocks_of(starts, idx)
    want = np.searchsorted(starts, idx, side="right") - 1
    assert np.array_equal(b, want) and np.array_equal(off, idx - starts[want])
    from paper_1907_01005_b200.errors import DomainError

    with pytest.raises(DomainError):
        _plan.blocks_of(starts, np.asarray([starts[-1]]))


@pytest.mark.parametrize("name", ["smoke", "q2"])
def test_support_overlap_equals_node_set_intersection(name):
    """Cell-adjacency form of support_overlap == pairwise intersection of the DoF supports."""
    prob = P.build_problem(name)
    ov = prob.support_overlap().toarray()
    lay = prob.loc_layout
    nc, v = lay.centers.shape[0], lay.vectors_per_center
    new = lay.new_col_of_old.reshape(nc, v)
    want = np.zeros_like(ov)
    for a in range(nc):
        for b in range(nc):
            if a == b or np.intersect1d(prob.supports[a], prob.supports[b]).size:
                want[np.ix_(new[a], new[b])] = True
    assert np.array_equal(ov, want)


@pytest.mark.parametrize("name", ["smoke", "q2", "q4"])
def test_grow_pattern_native_equals_sparse_product(name):
    from paper_1907_01005_b200.localization import (_grow_sparsity_numpy,
                                                    grow_sparsity_for_operator)

    prob = P.build_problem(name)
    a = grow_sparsity_for_operator(prob.pattern, prob.mesh, prob.numbering)
    b = _grow_sparsity_numpy(prob.pattern, prob.mesh, prob.numbering)
    assert np.array_equal(a.row_start, b.row_start) and np.array_equal(a.col_index, b.col_index)


def test_grow_pattern_random_patterns():
    from paper_1907_01005_b200.localization import (_grow_sparsity_numpy,
                                                    grow_sparsity_for_operator)
    from paper_1907_01005_b200.blocks import BlockSparsityPattern

    prob = P.build_problem("smoke", 2)
    rng = np.random.default_rng(11)
    nrb = prob.pattern.row_blocks.n_blocks
    for n_cb_frac in (0.05, 0.3):
        from paper_1907_01005_b200.blocks import BlockIndices

        cb = BlockIndices(np.full(130, 1))  # > 64 column blocks: several bitset words
        mask = rng.random((nrb, 130)) < n_cb_frac
        row_start = np.concatenate([[0], np.cumsum(mask.sum(1))])
        pat = BlockSparsityPattern.from_csr(prob.pattern.row_blocks, cb, row_start,
                                            np.nonzero(mask)[1])
        a = grow_sparsity_for_operator(pat, prob.mesh, prob.numbering)
        b = _grow_sparsity_numpy(pat, prob.mesh, prob.numbering)
        assert np.array_equal(a.row_start, b.row_start) and np.array_equal(a.col_index, b.col_index)


def test_first_touch_matches_minimum_at():
    rng = np.random.default_rng(2)
    touches = rng.integers(0, 5000, 200_000)
    first = np.full(5003, touches.size, dtype=np.int64)
    np.minimum.at(first, touches, np.arange(touches.size))
    assert np.array_equal(_plan.first_touch(5003, touches), first)


@pytest.mark.parametrize("n_ranks", [1, 3])
def test_enumerate_dofs_native_equals_numpy(monkeypatch, n_ranks):
    from paper_1907_01005_b200.mesh import build_mesh, enumerate_dofs, partition_and_order_cells

    mesh = build_mesh((6, 5, 7), (1 / 6, 1 / 5, 1 / 7), 0)
    part = partition_and_order_cells(mesh, n_ranks)
    a = enumerate_dofs(mesh, part, 3)
    monkeypatch.setenv("BMV_PLAN_NATIVE", "0")
    b = enumerate_dofs(mesh, part, 3)
    assert np.array_equal(a.new_index_of_node, b.new_index_of_node)
    assert a.owned_ranges == b.owned_ranges


@pytest.mark.gpu
@pytest.mark.parametrize("name,n_ranks", [("smoke", 1), ("q2", 1), ("smoke", 2)])
def test_fill_multivector_device_scatter_equals_host_image(name, n_ranks):
    """The device path (compact values + upload_support_values) writes the same X as the
    host image path, ghosts included, bit for bit."""
    import torch

    prob = P.build_problem(name, n_ranks)
    dev = torch.device("cuda", 0)

    def prog(ctx):
        layout = make_dof_layout(ctx, prob.mesh, prob.partition, prob.numbering)
        a = P.fill_multivector(BlockCsrMatrix(prob.pattern, layout, ctx, 8, dev), prob, 1)
        b = P.fill_multivector(BlockCsrMatrix(prob.pattern, layout, ctx, 8, "cpu"), prob, 1)
        torch.cuda.synchronize()
        return bool(torch.equal(a.data.cpu(), b.data))

    assert all(run_ranks(n_ranks, prog, device=dev))


@pytest.mark.parametrize("name", ["smoke", "q2"])
def test_native_pairs_images_and_k1_tables_equal_numpy(monkeypatch, name):
    """bmvp_cell_pairs / bmvp_block_image / bmvp_k1_plan against the sparse-product
    restatements (active pairs, ImageColumns, K1 group tables)."""
    from paper_1907_01005_b200 import problem as P
    from paper_1907_01005_b200.comm import serial_context
    from paper_1907_01005_b200.matfree import CellOperator, ImageColumns, _CellPlan
    from paper_1907_01005_b200.slabs import FULL

    prob = P.build_problem(name)
    st = P.make_rank_setup(serial_context("cpu"), prob, device="cpu", projection=False)
    op = st.op
    gb = st.layout.global_blocks_of_locals()
    sup = prob.column_support
    nat = {}
    for native in ("1", "0"):
        monkeypatch.setenv("BMV_PLAN_NATIVE", native)
        fresh = CellOperator(prob.mesh, prob.partition, prob.numbering, st.layout)
        act = fresh.active_pairs(sup)
        img = ImageColumns(fresh, sup).columns_for(prob.grown, gb)
        img_full = ImageColumns(fresh, FULL).columns_for(prob.grown, gb)
        plan = _CellPlan(fresh, st.x, st.hx, upload=False)
        nat[native] = (act, img, img_full, plan.arrays)
    a1, a0 = nat["1"][0], nat["0"][0]
    assert np.array_equal(a1.indptr, a0.indptr) and np.array_equal(a1.indices, a0.indices)
    for k in (1, 2):
        assert np.array_equal(nat["1"][k][0], nat["0"][k][0])
        assert np.array_equal(nat["1"][k][1], nat["0"][k][1])
    for key in ("pair_cell", "pair_gtab", "pair_ngp", "gtab", "codes"):
        assert np.array_equal(nat["1"][3][key], nat["0"][3][key]), key


def test_images_at_two_ranks_agree_with_the_owner(monkeypatch):
    """ImageColumns is defined per GLOBAL block row: a ghost copy on rank 1
    stores exactly the owner's columns (whole slab rows travel in exchanges)."""
    from paper_1907_01005_b200 import problem as P
    from paper_1907_01005_b200.comm import run_ranks

    prob = P.build_problem("smoke", 2)

    def program(ctx):
        st = P.make_rank_setup(ctx, prob, device="cpu", projection=False)
        gb = st.layout.global_blocks_of_locals()
        sg = st.hx.slab
        return {int(b): sg.cols[sg.ptr[i]:sg.ptr[i + 1]].tolist() for i, b in enumerate(gb)}

    r0, r1 = run_ranks(2, program)
    shared = set(r0) & set(r1)
    assert shared  # the ranks share ghost block rows
    for b in shared:
        assert r0[b] == r1[b], b
