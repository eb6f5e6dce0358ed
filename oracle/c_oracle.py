"""ctypes wrapper of oracle/liboracle.so (TEST INFRASTRUCTURE ONLY; see __init__)."""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from . import numpy_oracle as NO

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
_lib = None


class Tables(C.Structure):
    _fields_ = [("n", C.c_int), ("W", C.c_int), ("kind", C.c_int),
                ("S", C.c_double * 25), ("D", C.c_double * 25), ("w3", C.c_double * 125),
                ("grad_scale", C.c_double * 3)]


def build():
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        _lib = C.CDLL(str(LIB))
        _lib.oracle_cellop_apply.restype = C.c_int
        _lib.oracle_tmmult.restype = C.c_int
        _lib.oracle_mmult.restype = C.c_int
        _lib.oracle_potential_gaussian.restype = C.c_int
    return _lib


def _p(a, ct):
    if a is None:
        return C.cast(None, C.POINTER(ct))
    return a.ctypes.data_as(C.POINTER(ct))


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def tables(degree, spacing, kind, lane_width):
    S, D, _, _ = NO.lagrange_tables(degree)
    n = degree + 1
    t = Tables()
    t.n, t.W, t.kind = n, lane_width, (0 if kind == "mass" else 1)
    for i in range(n * n):
        t.S[i] = S.ravel()[i]
        t.D[i] = D.ravel()[i]
    w3 = NO.weights3(degree, spacing).ravel()
    for i in range(n**3):
        t.w3[i] = w3[i]
    for k in range(3):
        t.grad_scale[k] = 0.5 / spacing[k] ** 2
    return t


def cellop_apply(degree, spacing, kind, cell_lb, cell_rib, cell_color, vq, x_meta, h_meta,
                 col_strides, col_sizes, x_data, hx_data, lane_width=8, threads=None):
    """hx_data += Op x_data over the given cells (reference Algorithm 6, all lanes)."""
    lib = load()
    t = tables(degree, spacing, kind, lane_width)
    lb, rib = _i64(cell_lb), _i64(cell_rib)
    col = None if cell_color is None else np.ascontiguousarray(cell_color, dtype=np.int32)
    vq = None if vq is None else np.ascontiguousarray(vq, dtype=np.float64)
    xr, xc, xo = (_i64(a) for a in x_meta)
    hr, hc, ho = (_i64(a) for a in h_meta)
    cs, cz = _i64(col_strides), _i64(col_sizes)
    threads = int(threads or os.cpu_count() or 1)
    rc = lib.oracle_cellop_apply(
        C.byref(t), C.c_int64(lb.shape[0]), _p(lb, C.c_int64), _p(rib, C.c_int64),
        _p(col, C.c_int32), _p(vq, C.c_double), _p(xr, C.c_int64), _p(xc, C.c_int64),
        _p(xo, C.c_int64), _p(hr, C.c_int64), _p(hc, C.c_int64), _p(ho, C.c_int64),
        _p(cs, C.c_int64), _p(cz, C.c_int64), _p(x_data, C.c_double), _p(hx_data, C.c_double),
        C.c_int(threads))
    if rc == -3:
        raise LookupError("destination pattern misses a block (PatternError)")
    if rc != 0:
        raise RuntimeError(f"oracle_cellop_apply failed ({rc})")
    return threads


def reference_offsets(m):
    """Block offsets of a BlockCsrMatrix's blocks in the reference layout
    (rows x padded stride per block, owned then ghost; reference bcsr.py:233-318)."""
    sizes = m.local_row_sizes[m.pos_row] * m.col_strides[m.col_index]
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


def matrix_meta(m):
    """(row_start, col_index, block_offsets) of a BlockCsrMatrix in the
    reference's BCSR layout -- the layout the C restatement runs on."""
    return m.row_start, m.col_index, reference_offsets(m)


def reference_values(m) -> np.ndarray:
    """Values of a BlockCsrMatrix in the reference layout (through the public
    value_bytes, which converts from the B200 slab layout)."""
    from paper_1907_01005_b200.bcsr import value_bytes

    return np.frombuffer(value_bytes(m), dtype="<f8").astype(np.float64)


def reference_zeros(m) -> np.ndarray:
    return np.zeros(int(reference_offsets(m)[-1]))


def load_reference(m, values: np.ndarray):
    """Write reference-layout values into a BlockCsrMatrix (load_value_bytes)."""
    from paper_1907_01005_b200.bcsr import load_value_bytes

    load_value_bytes(m, np.ascontiguousarray(values, dtype="<f8").tobytes())


def _ltab(layout, n_global):
    tab = np.full(n_global, -1, dtype=np.int64)
    gl = layout.global_blocks_of_locals()
    tab[gl] = np.arange(gl.size, dtype=np.int64)
    return tab


def tmmult(a, b, c, a_vals, b_vals, threads=None):
    """C = A^T B over the owned rows of a (reference tmmult loop, bcsr.py:631-667,
    before the compress), all arrays in the reference layout; returns c's values."""
    lib = load()
    n = a.n_owned_blocks
    out = reference_zeros(c)
    ar, ac, ao = (_i64(v) for v in matrix_meta(a))
    br, bc, bo = (_i64(v) for v in matrix_meta(b))
    cr, cc, co = (_i64(v) for v in matrix_meta(c))
    cl = _i64(_ltab(c.layout, c.layout.blocks.n_blocks))
    rows = _i64(a.local_row_sizes)
    av = np.ascontiguousarray(a_vals, dtype=np.float64)
    bv = np.ascontiguousarray(b_vals, dtype=np.float64)
    rc = lib.oracle_tmmult(
        C.c_int64(n), _p(ar, C.c_int64), _p(ac, C.c_int64), _p(ao, C.c_int64),
        _p(_i64(a.col_strides), C.c_int64), _p(_i64(a.col_blocks.sizes), C.c_int64),
        _p(rows, C.c_int64), _p(av, C.c_double), _p(br, C.c_int64), _p(bc, C.c_int64),
        _p(bo, C.c_int64), _p(_i64(b.col_strides), C.c_int64),
        _p(_i64(b.col_blocks.sizes), C.c_int64), _p(bv, C.c_double), _p(cl, C.c_int64),
        _p(cr, C.c_int64), _p(cc, C.c_int64), _p(co, C.c_int64),
        _p(_i64(c.col_strides), C.c_int64), _p(out, C.c_double), C.c_int64(out.size),
        C.c_int(int(threads or os.cpu_count() or 1)))
    if rc == -3:
        raise LookupError("tmmult destination misses a block (PatternError)")
    if rc != 0:
        raise RuntimeError(f"oracle_tmmult failed ({rc})")
    return out


def mmult(a, b, c, a_vals, b_vals, alpha=1.0, threads=None):
    """C = alpha A B truncated to c's block pattern (reference mmult,
    bcsr.py:587-628), reference layout; returns c's values (zero start)."""
    lib = load()
    n = a.n_owned_blocks
    out = reference_zeros(c)
    ar, ac, ao = (_i64(v) for v in matrix_meta(a))
    br, bc, bo = (_i64(v) for v in matrix_meta(b))
    cr, cc, co = (_i64(v) for v in matrix_meta(c))
    bl = _i64(_ltab(b.layout, b.layout.blocks.n_blocks))
    rows = _i64(a.local_row_sizes)
    av = np.ascontiguousarray(a_vals, dtype=np.float64)
    bv = np.ascontiguousarray(b_vals, dtype=np.float64)
    rc = lib.oracle_mmult(
        C.c_int64(n), _p(ar, C.c_int64), _p(ac, C.c_int64), _p(ao, C.c_int64),
        _p(_i64(a.col_strides), C.c_int64), _p(_i64(a.col_blocks.sizes), C.c_int64),
        _p(rows, C.c_int64), _p(av, C.c_double), _p(bl, C.c_int64), _p(br, C.c_int64),
        _p(bc, C.c_int64), _p(bo, C.c_int64), _p(_i64(b.col_strides), C.c_int64),
        _p(_i64(b.col_blocks.sizes), C.c_int64), _p(bv, C.c_double), _p(cr, C.c_int64),
        _p(cc, C.c_int64), _p(co, C.c_int64), _p(out, C.c_double), C.c_double(alpha),
        C.c_int(int(threads or os.cpu_count() or 1)))
    if rc != 0:
        raise RuntimeError(f"oracle_mmult failed ({rc})")
    return out


def potential_gaussian(pot, cell_origins, degree, spacing, threads=None) -> np.ndarray:
    """(n_cells, q^3) V of a GaussianPotential at the cell quadrature points (C, OpenMP)."""
    lib = load()
    qo = np.ascontiguousarray(NO.quad_offsets(degree, spacing), dtype=np.float64)
    org = np.ascontiguousarray(cell_origins, dtype=np.float64)
    cen = np.ascontiguousarray(pot.centers, dtype=np.float64)
    out = np.empty((org.shape[0], qo.shape[0]))
    lib.oracle_potential_gaussian(C.c_int64(org.shape[0]), C.c_int(qo.shape[0]),
                                  _p(org, C.c_double), _p(qo, C.c_double), _p(cen, C.c_double),
                                  C.c_int(cen.shape[0]), C.c_double(pot.inv_sigma2),
                                  C.c_double(pot.scale), _p(out, C.c_double),
                                  C.c_int(int(threads or os.cpu_count() or 1)))
    return out
