"""Host-side drop-in API (CPU storage, no kernels): layouts, ghost exchange
protocol, state machine, cell DoF map, accessor, errors.  Scenarios follow
the reference's own tests (file:line cited per test)."""

import numpy as np
import pytest
import torch

from paper_1907_01005_b200.bcsr import (
    GHOSTED,
    OWNED,
    BlockCsrMatrix,
    build_rank_layout,
    group_rows_by_block,
    load_value_bytes,
    serial_layout,
    serial_matrix,
    value_bytes,
)
from paper_1907_01005_b200.blocks import BlockIndices, BlockSparsityPattern
from paper_1907_01005_b200.comm import run_ranks
from paper_1907_01005_b200.errors import (
    ConfigurationError,
    DeviceError,
    PatternError,
    ProtocolError,
    RankFailure,
    StateError,
)
from paper_1907_01005_b200.hilbert import hilbert_index, hilbert_keys
from paper_1907_01005_b200.matfree import (
    CellOperator,
    RowsBlockAccessor,
    build_cell_dof_map_from_rows,
    hamiltonian_operator,
    make_dof_layout,
)
from paper_1907_01005_b200.mesh import build_mesh, enumerate_dofs, partition_and_order_cells

CPU = "cpu"


def test_ghost_grouping_documented_scenario():
    # paper Fig. 5a, reference tests/test_bcsr.py:44-51: groups of sizes 3, 2, 3, 1
    blocks = BlockIndices([4, 4, 4, 4])
    rows = [1, 2, 3, 4, 6, 8, 9, 11, 13]
    groups = group_rows_by_block(rows, blocks)
    assert [len(r) for _, r in groups] == [3, 2, 3, 1]
    assert [b for b, _ in groups] == [0, 1, 2, 3]
    assert group_rows_by_block([], blocks) == []


def test_padding_alignment_and_entries():
    # reference tests/test_bcsr.py:82-107
    pat = BlockSparsityPattern(BlockIndices([3, 2]), BlockIndices([3, 5]), [[0, 1], [1]])
    m = serial_matrix(pat, lane_width=4, device=CPU)
    assert m.col_strides.tolist() == [4, 8]
    m.fill_owned(lambda r, c: np.ones((r.size, c.size)))
    for pos in range(m.col_index.size):
        blk = m.block_values(pos)
        cols = int(m.col_blocks.sizes[m.col_index[pos]])
        assert torch.all(blk[:, cols:] == 0)
    m.add_entry(4, 6, 2.5)
    assert m.get_entry(4, 6) == 3.5
    assert m.get_entry(0, 5) == 1.0  # block (0, 1) stored
    assert m.get_entry(3, 0) == 0.0  # block (1, 0) absent
    with pytest.raises(PatternError):
        m.add_entry(3, 0, 1.0)  # block (1, 0) not stored


def test_state_machine():
    # reference tests/test_bcsr.py:109-128
    pat = BlockSparsityPattern(BlockIndices([2]), BlockIndices([2]), [[0]])
    m = serial_matrix(pat, device=CPU)
    m.update_ghost_values()
    assert m.state == GHOSTED
    with pytest.raises(StateError):
        m.zero_out()
    with pytest.raises(StateError):
        m.compress()
    m.release_ghosts()
    assert m.state == OWNED
    m.update_ghost_values_start()
    with pytest.raises(StateError):
        m.update_ghost_values_start()
    m.update_ghost_values_finish()
    with pytest.raises(StateError):
        m.update_ghost_values_finish()


def test_serialization_roundtrip():
    pat = BlockSparsityPattern(BlockIndices([2, 3]), BlockIndices([2, 1]), [[0, 1], [1]])
    m = serial_matrix(pat, device=CPU)
    m.fill_owned(lambda r, c: (r[:, None] * 10.0 + c[None, :]))
    raw = value_bytes(m)
    m2 = serial_matrix(pat, device=CPU)
    load_value_bytes(m2, raw)
    assert np.array_equal(m.to_dense_owned(), m2.to_dense_owned())


def two_rank_blocks():
    return BlockIndices([3, 3, 3, 3]), np.asarray([0, 2, 4])


def test_update_ghost_values_bit_equal():
    # reference tests/test_bcsr.py:157-174
    blocks, starts = two_rank_blocks()
    pat = BlockSparsityPattern(blocks, BlockIndices([2, 2]), [[0, 1], [0], [1], [0, 1]])

    def program(ctx):
        ghost = [6, 8] if ctx.rank == 0 else [2]
        lay = build_rank_layout(ctx, blocks, starts, ghost)
        m = BlockCsrMatrix(pat, lay, ctx, 4, device=CPU)
        m.fill_owned(lambda r, c: (10.0 * r[:, None] + c[None, :]).astype(float))
        m.update_ghost_values()
        if ctx.rank == 0:
            return m.get_entry(6, 3), m.get_entry(8, 2)
        return m.get_entry(2, 0), m.get_entry(2, 1)

    r0, r1 = run_ranks(2, program)
    assert r0 == (63.0, 82.0)
    assert r1 == (20.0, 21.0)


def test_compress_additive_and_ghosts_zeroed():
    # reference tests/test_bcsr.py:177-195
    blocks, starts = two_rank_blocks()
    pat = BlockSparsityPattern(blocks, BlockIndices([1]), [[0], [0], [0], [0]])

    def program(ctx):
        lay = build_rank_layout(ctx, blocks, starts, [7] if ctx.rank == 0 else [])
        m = BlockCsrMatrix(pat, lay, ctx, 4, device=CPU)
        m.add_entry(7, 0, 1.0)
        m.compress()
        if ctx.rank == 1:
            return m.get_entry(7, 0)
        return float(m.data[m._ghost_data_begin:].sum())

    ghost_left, owner = run_ranks(2, program)
    assert owner == 2.0 and ghost_left == 0.0


def test_compress_matches_single_rank_sum():
    # reference tests/test_bcsr.py:215-248
    rng = np.random.default_rng(3)
    blocks = BlockIndices([2, 3, 2, 3])
    starts = np.asarray([0, 1, 2, 3, 4])
    cb = BlockIndices([2, 1])
    pat = BlockSparsityPattern(blocks, cb, [[0, 1], [0], [0, 1], [1]])
    contrib = {r: rng.random((blocks.total, cb.total)) for r in range(4)}
    mask = pat.entry_mask()

    def program(ctx):
        ghosts = [i for b in range(4) if b != ctx.rank
                  for i in range(blocks.block_start(b), blocks.block_start(b) + blocks.block_size(b))]
        lay = build_rank_layout(ctx, blocks, starts, ghosts)
        m = BlockCsrMatrix(pat, lay, ctx, 4, device=CPU)
        for row in range(blocks.total):
            for col in range(cb.total):
                if mask[row, col]:
                    m.add_entry(row, col, contrib[ctx.rank][row, col])
        m.compress()
        return m.to_dense_owned()

    got = np.sum(run_ranks(4, program), axis=0)
    want = np.sum([contrib[r] for r in range(4)], axis=0) * mask
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-12


def test_inconsistent_ghost_request_is_protocol_error():
    # reference tests/test_bcsr.py:251-268
    blocks = BlockIndices([2, 2])
    starts = np.asarray([0, 1, 2])

    def program(ctx):
        if ctx.rank == 0:
            ctx.isend(1, ("ghost_req", 1), (np.asarray([0]), [np.asarray([0, 1])]))
            ctx.irecv(1, ("ghost_req", 1)).wait()
            ctx.irecv(1, ("ghost_ack", 1)).wait()
            return "sent"
        return build_rank_layout(ctx, blocks, starts, [])

    with pytest.raises(RankFailure) as info:
        run_ranks(2, program, deadlock_timeout=2.0)
    assert any(isinstance(e, ProtocolError) for e in info.value.failures.values())


def fig_blocking():
    return BlockIndices([4, 1, 2, 2, 1, 1, 1, 1, 3])


def test_cell_dof_map_documented_arrays():
    # paper Fig. 4b, reference tests/test_matfree.py:78-95
    rb = fig_blocking()
    s = rb.block_start
    rows = [s(8) + 0, s(8) + 1, s(0) + 1, s(2) + 0, s(0) + 3, s(3) + 0, s(8) + 2, s(2) + 1, s(3) + 1]
    pat = BlockSparsityPattern(rb, BlockIndices([2]), [[0]] * 9)
    m = serial_matrix(pat, device=CPU)
    cmap = build_cell_dof_map_from_rows([rows], m.layout.map_rows)
    assert cmap.dof_indices.tolist() == [[0, 0], [1, 1], [2, 6], [1, 2], [3, 4], [0, 3],
                                         [1, 7], [0, 5], [1, 8]]
    assert cmap.block_indices.tolist() == [[8, 3], [0, 2], [2, 2], [3, 2]]
    assert cmap.cell_offsets.tolist() == [[0, 0], [9, 4]]


def test_accessor_merge_and_pattern_error():
    # reference tests/test_matfree.py:116-135,194-202
    rb = fig_blocking()
    cb = BlockIndices([2, 2, 2])
    rows_cols = [[1, 2], [], [0], [2], [], [], [], [], [0, 1]]
    pat = BlockSparsityPattern(rb, cb, rows_cols)
    m = serial_matrix(pat, device=CPU)
    s = rb.block_start
    cell = [s(8), s(0), s(2), s(3)]
    cmap = build_cell_dof_map_from_rows([cell], m.layout.map_rows)
    acc = RowsBlockAccessor(m, cmap)
    assert acc.emitted_columns(0) == [0, 1, 2]
    acc.reinit(0)
    act = acc.active_groups()
    assert len(act) == 2  # blocks 8 and 2 hold column 0
    small = serial_matrix(BlockSparsityPattern(rb, cb, [[1], [], [0], [], [], [], [], [], [0]]),
                          device=CPU)
    w = RowsBlockAccessor(small, cmap)
    w.reinit(0)
    with pytest.raises(PatternError):
        w.advance_to(2)


def test_hilbert_2d_orientation_and_bijection():
    # reference hilbert.py:1-12: d=2, levels=1 visits (0,0),(0,1),(1,1),(1,0)
    pts = [(0, 0), (0, 1), (1, 1), (1, 0)]
    assert [hilbert_index(p, 1).index for p in pts] == [0, 1, 2, 3]
    for d, lv in ((2, 4), (3, 3)):
        g = np.stack(np.meshgrid(*[np.arange(1 << lv)] * d, indexing="ij"), -1).reshape(-1, d)
        k = hilbert_keys(g, lv)
        assert np.array_equal(np.sort(k), np.arange(g.shape[0], dtype=np.uint64))
        # consecutive keys are lattice neighbours
        order = g[np.argsort(k)]
        assert np.all(np.abs(np.diff(order, axis=0)).sum(1) == 1)


def test_configuration_errors():
    with pytest.raises(ConfigurationError):
        build_mesh((3, 4, 4), (1.0, 1.0, 1.0), 1)
    mesh = build_mesh((2, 2, 2), (1.0, 1.0, 1.0), 0)
    with pytest.raises(ConfigurationError):
        partition_and_order_cells(mesh, 9)
    part = partition_and_order_cells(mesh, 1)
    with pytest.raises(ConfigurationError):
        enumerate_dofs(mesh, part, 5)


def test_compute_refuses_cpu_storage():
    """No CPU fallback: the operator path fails loudly on CPU data."""
    mesh = build_mesh((2, 2, 2), (1.0, 1.0, 1.0), 0)
    part = partition_and_order_cells(mesh, 1)
    num = enumerate_dofs(mesh, part, 1)
    ctx = run_ranks  # noqa: F841
    from paper_1907_01005_b200.comm import serial_context

    c = serial_context(CPU)
    lay = make_dof_layout(c, mesh, part, num)
    op = CellOperator(mesh, part, num, lay)
    pat = BlockSparsityPattern(num.row_blocks, BlockIndices([1]), [[0]] * num.row_blocks.n_blocks)
    x = BlockCsrMatrix(pat, lay, c, 8, device=CPU)
    y = BlockCsrMatrix(pat, lay, c, 8, device=CPU)
    with pytest.raises(DeviceError):
        op.apply(hamiltonian_operator(None), x, y)


def test_compact_support_values_roundtrip():
    """upload/download_support_values (the compact transfer format) round-trip."""
    from paper_1907_01005_b200 import problem as P
    from paper_1907_01005_b200.comm import serial_context

    prob = P.build_problem("smoke")
    st = P.make_rank_setup(serial_context(CPU), prob, device=CPU)
    vals = st.x.download_support_values().clone()
    assert vals.numel() == st.x.n_support_values() == 5320  # nnzX of the smoke config
    dense = st.x.to_dense_owned()
    st.x.data.fill_(3.0)
    st.x.upload_support_values(vals)
    assert np.array_equal(st.x.to_dense_owned(), dense)
