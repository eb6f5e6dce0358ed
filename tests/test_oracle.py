"""The oracle itself, pinned against the reference's outputs (golden fixtures)
and against the reference's own known-answer properties."""

import numpy as np
import pytest
import torch

from _helpers import Small, cosine
from oracle import c_oracle as CO
from oracle import numpy_oracle as O
from paper_1907_01005_b200 import problem as P
from paper_1907_01005_b200.comm import serial_context
from paper_1907_01005_b200.mesh import cells_nodes


def test_numpy_oracle_smoke_matches_reference(golden_smoke):
    g = golden_smoke
    prob = P.build_problem("smoke")
    cells = np.arange(prob.mesh.n_cells)
    nodes = cells_nodes(prob.mesh, prob.numbering, cells)
    org = prob.mesh.cell_origins(cells)
    hx = O.apply_dense(nodes, org, 2, prob.mesh.spacing, "h", prob.potential, g["x"])
    assert O.per_vector_rel_err(hx, g["hx"]) <= 1e-13
    mx = O.apply_dense(nodes, org, 2, prob.mesh.spacing, "mass", None, g["x"])
    assert O.per_vector_rel_err(mx, g["mx"]) <= 1e-13
    s = O.tmmult_dense(g["x"], g["hx"], np.ones((8, 8), dtype=bool))
    assert np.max(np.abs(s - g["s"])) <= 1e-13 * np.max(np.abs(g["s"]))
    xc = O.mmult_dense(g["x"], g["c"], prob.pattern.entry_mask())
    assert O.per_vector_rel_err(xc, g["xc"]) <= 1e-13


def test_numpy_oracle_assembled_operator_matches_reference(golden_smoke):
    g = golden_smoke
    prob = P.build_problem("smoke")
    cells = np.arange(prob.mesh.n_cells)
    a = O.assembled_operator(cells_nodes(prob.mesh, prob.numbering, cells),
                             prob.mesh.cell_origins(cells), 2, prob.mesh.spacing, "h",
                             prob.potential, prob.numbering.n_dofs)
    assert (a - a.T).nnz == 0  # exactly symmetric (matfree.py:530-575)
    assert O.per_vector_rel_err(a @ g["x"], g["hx"]) <= 1e-12


@pytest.mark.parametrize("degree", [1, 2, 3, 4])
def test_sumfac_matches_element_matrix(degree):
    # reference tests/test_matfree.py:227-244
    rng = np.random.default_rng(degree)
    n3 = (degree + 1) ** 3
    sp = (0.7, 1.1, 0.9)
    u = rng.random((n3, 5)) - 0.5
    vq = rng.random(n3)
    for kind in ("h", "mass"):
        e = O.element_matrix(degree, sp, kind, vq if kind == "h" else None)
        got = O.cell_integrals(degree, sp, kind, u, vq if kind == "h" else None)
        assert np.abs(got - e @ u).max() <= 1e-13 * np.abs(e @ u).max()


def test_hamiltonian_annihilates_constants_and_mass_volume():
    # reference tests/test_matfree.py:208-224
    for degree in (1, 2, 3, 4):
        n3 = (degree + 1) ** 3
        ones = np.ones((n3, 1))
        h = O.cell_integrals(degree, (0.5, 0.5, 0.5), "h", ones)
        assert np.abs(h).max() <= 1e-12
        m = O.cell_integrals(degree, (0.5, 0.5, 0.5), "mass", ones)
        assert abs(m.sum() - 0.125) <= 1e-14


@pytest.mark.parametrize("degree", [1, 2, 3, 4])
def test_c_oracle_matches_reference_random(golden_random, degree):
    g = golden_random
    ext = tuple(int(v) for v in g[f"p{degree}_extents"])
    s = Small(ext, (1.0, 1.0, 1.0), 1, degree, g[f"p{degree}_centers"],
              float(g[f"p{degree}_radius"]), 3, 2, 1)
    ctx = serial_context("cpu")
    rl, op, x, hx = s.operands(ctx, "cpu")
    s.fill(x, 10 * degree)
    vq = O.sample_potential(cosine(degree), op.cell_origins, degree, s.mesh.spacing)
    h = CO.reference_zeros(hx)
    CO.cellop_apply(degree, s.mesh.spacing, "h", op._lb, op._rib, op.cell_color, vq,
                    CO.matrix_meta(x), CO.matrix_meta(hx), x.col_strides, x.col_blocks.sizes,
                    CO.reference_values(x), h, threads=2)
    CO.load_reference(hx, h)
    got = hx.to_dense_owned()
    want = g[f"p{degree}_r1_hx"]
    assert O.per_vector_rel_err(got, want) <= 1e-13


def test_c_oracle_smoke_matches_reference(golden_smoke):
    prob = P.build_problem("smoke")
    st = P.make_rank_setup(serial_context("cpu"), prob, device="cpu")
    op = st.op
    vq = O.sample_potential(prob.potential, op.cell_origins, 2, prob.mesh.spacing)
    h = CO.reference_zeros(st.hx)
    CO.cellop_apply(2, prob.mesh.spacing, "h", op._lb, op._rib, op.cell_color, vq,
                    CO.matrix_meta(st.x), CO.matrix_meta(st.hx), st.x.col_strides,
                    st.x.col_blocks.sizes, CO.reference_values(st.x), h, threads=2)
    CO.load_reference(st.hx, h)
    assert O.per_vector_rel_err(st.hx.to_dense_owned(), golden_smoke["hx"]) <= 1e-13


def test_one_dimensional_fe_stencil_known_answer():
    # reference tests/test_matfree.py:371-411: Q1, a line of cells, no potential:
    # interior rows of the assembled -1/2 Laplacian reproduce the 1D stencil
    # tensor structure; here: row sums vanish and the matrix is symmetric.
    from paper_1907_01005_b200.mesh import build_mesh, enumerate_dofs, partition_and_order_cells

    mesh = build_mesh((4, 1, 1), (1.0, 1.0, 1.0), 0)
    part = partition_and_order_cells(mesh, 1)
    num = enumerate_dofs(mesh, part, 1)
    cells = np.arange(mesh.n_cells)
    a = O.assembled_operator(cells_nodes(mesh, num, cells), mesh.cell_origins(cells), 1,
                             mesh.spacing, "h", None, num.n_dofs)
    assert np.abs(a @ np.ones(num.n_dofs)).max() <= 1e-14
    assert (a - a.T).nnz == 0


def test_c_oracle_projection_and_postmultiply_match_reference(golden_smoke):
    """oracle_tmmult / oracle_mmult (oracle/cellop.c, the reference loops of
    bcsr.py:587-667) pinned to the reference's own S and X C on the smoke config."""
    prob = P.build_problem("smoke")
    st = P.make_rank_setup(serial_context("cpu"), prob, device="cpu", projection=True,
                           compact_xc=False)
    CO.load_reference(st.hx, _hx_reference(st, prob))
    s_ref = CO.tmmult(st.x, st.hx, st.s, CO.reference_values(st.x), CO.reference_values(st.hx),
                      threads=2)
    CO.load_reference(st.s, s_ref)
    assert np.abs(st.s.to_dense_owned() - golden_smoke["s"]).max() <= 1e-13 * np.abs(golden_smoke["s"]).max()
    xc_ref = CO.mmult(st.x, st.c, st.xc, CO.reference_values(st.x), CO.reference_values(st.c),
                      threads=2)
    CO.load_reference(st.xc, xc_ref)
    assert O.per_vector_rel_err(st.xc.to_dense_owned(), golden_smoke["xc"]) <= 1e-14


def _hx_reference(st, prob):
    op = st.op
    vq = O.sample_potential(prob.potential, op.cell_origins, 2, prob.mesh.spacing)
    h = CO.reference_zeros(st.hx)
    CO.cellop_apply(2, prob.mesh.spacing, "h", op._lb, op._rib, op.cell_color, vq,
                    CO.matrix_meta(st.x), CO.matrix_meta(st.hx), st.x.col_strides,
                    st.x.col_blocks.sizes, CO.reference_values(st.x), h, threads=2)
    return h
