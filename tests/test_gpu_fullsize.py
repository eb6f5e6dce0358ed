"""Full-size parity of the BASELINE configs against the C restatement of the
reference loops (oracle/cellop.c on the reference BCSR layout):

* H X at proj and weak G = 1 (cell loop, 18 contractions, all lanes), with
  V sampled by the numpy oracle (not by the device);
* S = X^T (H Y) at proj (BASELINE configs[3]: Y a second seeded multivector
  on X's pattern, H Y on the grown pattern) and S = X^T (H X) at weak G = 1
  against oracle_tmmult;
* Y = X C at proj and weak G = 1 against oracle_mmult (block-level
  truncation; compact X C compared on its stored entries).

Errors: H X and X C <= 1e-12 relative per vector; S entries <= 1e-11
relative to max(|S_ab|, ||x_a|| ||(HY)_b||).  Compared on the
stored entries (dense forms would not fit in memory)."""

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

from oracle import c_oracle as CO
from oracle import numpy_oracle as O
from paper_1907_01005_b200 import problem as P
from paper_1907_01005_b200.bcsr import BlockCsrMatrix, mmult, tmmult
from paper_1907_01005_b200.comm import serial_context

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def col_sq(m, data: torch.Tensor) -> np.ndarray:
    """Per-column sum of squares of a value array in m's storage (owned entries)."""
    flat, _, gcol = m._valid_owned_index()
    v = data[torch.as_tensor(flat, device=data.device)]
    out = torch.zeros(m.col_blocks.total, dtype=torch.float64, device=data.device)
    out.index_add_(0, torch.as_tensor(gcol, device=data.device), v * v)
    return out.cpu().numpy()


def per_vector_err(m, got: torch.Tensor, want: torch.Tensor) -> float:
    diff = col_sq(m, got - want)
    ref = col_sq(m, want)
    ok = ref > 0
    return float(np.sqrt(np.max(diff[ok] / ref[ok]))) if ok.any() else 0.0


_VQ: dict = {}


@pytest.fixture(scope="module", params=["proj", "weak1"])
def big(request):
    """One problem + rank setup per config for the whole module (pytest groups the
    tests by this parameter, so each config is built once and V is sampled once)."""
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_1907_01005_b200 import _lib

    _lib.require_device()
    dev = torch.device("cuda", 0)
    name = request.param
    prob = P.build_problem(name)
    st = P.make_rank_setup(serial_context(dev), prob, projection=True, device=dev,
                           with_y=name == "proj")
    yield name, prob, st
    del st, prob
    _VQ.clear()
    torch.cuda.empty_cache()


def oracle_potential(prob, op):
    """V at the quadrature points of every cell by the numpy oracle (cell chunks)."""
    key = prob.cfg.name
    if key not in _VQ:
        deg = prob.cfg.degree
        # the oracle's per-point sum over the centres, cell chunks spread over the host
        # threads (numpy releases the GIL inside the ufuncs)
        starts = range(0, len(op.cells), 2048)
        with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as pool:
            parts = list(pool.map(
                lambda c0: O.sample_potential(prob.potential, op.cell_origins[c0 : c0 + 2048],
                                              deg, prob.mesh.spacing), starts))
        _VQ.clear()
        _VQ[key] = np.concatenate(parts)
    return _VQ[key]


def oracle_apply(st, prob, x):
    """H x with the C oracle; V sampled by the numpy oracle at the quadrature points."""
    op = st.op
    deg = prob.cfg.degree
    vq = oracle_potential(prob, op)
    want = CO.reference_zeros(st.hx)
    CO.cellop_apply(deg, prob.mesh.spacing, "h", op._lb, op._rib, op.cell_color, vq,
                    CO.matrix_meta(x), CO.matrix_meta(st.hx), x.col_strides,
                    x.col_blocks.sizes, CO.reference_values(x), want)
    return want


def like(m, ref_values):
    """A matrix with m's storage holding reference-layout values."""
    out = BlockCsrMatrix(m.pattern, m.layout, m.ctx, m.lane_width, m.device, columns=m.columns)
    CO.load_reference(out, ref_values)
    return out


def test_large_config_hx_matches_c_oracle(cuda, big):
    name, prob, st = big
    st.op.apply(prob.spec_h(), st.x, st.hx)
    torch.cuda.synchronize()
    want = like(st.hx, oracle_apply(st, prob, st.x))
    err = per_vector_err(st.hx, st.hx.data, want.data)
    assert err <= 1e-12, err


def _proj_err(st, s_got, s_want, x, z):
    """max |S - S_ref| / max(|S_ref|, ||x_a|| ||z_b||) over S's stored entries."""
    xn = np.sqrt(col_sq(x, x.data))
    zn = np.sqrt(col_sq(z, z.data))
    flat, grow, gcol = s_got._valid_owned_index()
    g = s_got.data.cpu().numpy()[flat]
    w = s_want.data.cpu().numpy()[flat]
    scale = np.maximum(np.abs(w), xn[grow] * zn[gcol])
    scale = np.where(scale > 0, scale, 1.0)
    return float(np.max(np.abs(g - w) / scale)) if flat.size else 0.0


def test_large_config_projection_and_postmultiply_match_c_oracle(cuda, big):
    name, prob, st = big
    with_y = name == "proj"
    src = st.y if with_y else st.x          # S = X^T (H Y) at proj, X^T (H X) at weak G = 1
    z = st.hy if with_y else st.hx
    st.op.apply(prob.spec_h(), src, z)
    tmmult(st.x, z, st.s)
    st.c.update_ghost_values()
    mmult(st.x, st.c, st.xc)
    torch.cuda.synchronize()
    # oracle: H src, then X^T (H src) and X C in the reference layout
    z_ref = oracle_apply(st, prob, src)
    z_want = like(z, z_ref)
    assert per_vector_err(z, z.data, z_want.data) <= 1e-12
    s_ref = CO.tmmult(st.x, z, st.s, CO.reference_values(st.x), z_ref)
    s_want = like(st.s, s_ref)
    err = _proj_err(st, st.s, s_want, st.x, z_want)
    assert err <= 1e-11, err
    xc_ref = CO.mmult(st.x, st.c, st.xc, CO.reference_values(st.x), CO.reference_values(st.c))
    full = BlockCsrMatrix(st.xc.pattern, st.xc.layout, st.xc.ctx, st.xc.lane_width, cuda)
    CO.load_reference(full, xc_ref)                  # the reference's block-truncated X C
    want = BlockCsrMatrix(st.xc.pattern, st.xc.layout, st.xc.ctx, st.xc.lane_width, cuda,
                          columns=st.xc.columns)
    flat, grow, gcol = st.xc._valid_owned_index()
    lb, rib = full._owned_local(grow)
    src_off = full.slab.offsets(lb, rib, gcol)
    assert (src_off >= 0).all()
    want.data[torch.as_tensor(flat, device=cuda)] = full.data[torch.as_tensor(src_off, device=cuda)]
    assert per_vector_err(st.xc, st.xc.data, want.data) <= 1e-12


def test_gaussian_potential_matches_oracle_at_512_centres(cuda, big):
    """The device potential (bmv_potential_gaussian, 512 centres at weak G = 1)
    against the numpy oracle's V at the quadrature points of a cell sample."""
    name, prob, st = big
    coef, stride = st.op.coefficient(prob.spec_h(), cuda)
    w3 = st.op.kernels.w3.ravel()
    rng = np.random.default_rng(3)
    cells = np.sort(rng.choice(len(st.op.cells), 4096, replace=False))
    got = coef.view(-1, stride)[torch.as_tensor(cells, device=cuda)].cpu().numpy()[:, : w3.size]
    vq = O.sample_potential(prob.potential, st.op.cell_origins[cells], prob.cfg.degree,
                            prob.mesh.spacing)
    want = vq.reshape(cells.size, -1) * w3[None, :]
    assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want))
