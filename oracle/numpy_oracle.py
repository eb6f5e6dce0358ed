"""numpy restatement of the reference hot-path arithmetic (oracle; tests only).

Each function cites the reference lines it restates.  Structures (mesh,
numbering, patterns) are taken as inputs; they are pinned separately
against golden fixtures generated from the reference itself.
"""

from __future__ import annotations

import numpy as np
from scipy import sparse


# -- tables (bcsrmv/shapes.py:14-69) ---------------------------------------------


def gauss01(nq):
    x, w = np.polynomial.legendre.leggauss(nq)
    return 0.5 * (x + 1.0), 0.5 * w


def lagrange_tables(degree, nq=None):
    """(S, D, points, weights): S[q, a] = l_a(x_q), D[q, a] = l_a'(x_q)."""
    nq = degree + 1 if nq is None else nq
    nodes = np.linspace(0.0, 1.0, degree + 1)
    x, w = gauss01(nq)
    n = nodes.size
    S = np.ones((x.size, n))
    D = np.zeros((x.size, n))
    for a in range(n):
        for b in range(n):
            if b != a:
                S[:, a] *= (x - nodes[b]) / (nodes[a] - nodes[b])
        for k in range(n):
            if k == a:
                continue
            t = np.full(x.size, 1.0 / (nodes[a] - nodes[k]))
            for b in range(n):
                if b != a and b != k:
                    t *= (x - nodes[b]) / (nodes[a] - nodes[b])
            D[:, a] += t
    return S, D, x, w


def quad_offsets(degree, spacing):
    """(q^3, 3) physical offsets of the Gauss points in a cell, x fastest (matfree.py:259-261)."""
    _, _, x, _ = lagrange_tables(degree)
    hx, hy, hz = spacing
    gz, gy, gx = np.meshgrid(x * hz, x * hy, x * hx, indexing="ij")
    return np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)


def weights3(degree, spacing):
    _, _, _, w = lagrange_tables(degree)
    det = float(np.prod(spacing))
    return (w[:, None, None] * w[None, :, None] * w[None, None, :]) * det


# -- cell integral, 18 contractions (matfree.py:243-367) --------------------------


def _con(mat, t, axis):
    return np.moveaxis(np.tensordot(mat, t, axes=(1, axis)), 0, axis)


def cell_integrals(degree, spacing, kind, u, v_q=None):
    """Reference-formulation cell action on u of shape (..., n^3, L): batched over leading axes."""
    S, D, _, _ = lagrange_tables(degree)
    n = degree + 1
    lead = u.shape[:-2]
    L = u.shape[-1]
    t = u.reshape(lead + (n, n, n, L))
    b = len(lead)
    ax = lambda k: b + k  # noqa: E731
    w3 = weights3(degree, spacing)
    wb = w3.reshape((1,) * b + (n, n, n, 1))
    tz = _con(S, t, ax(0))
    tzy = _con(S, tz, ax(1))
    uq = _con(S, tzy, ax(2))
    if kind == "mass":
        r = uq * wb
        r = _con(S.T, r, ax(2))
        r = _con(S.T, r, ax(1))
        out = _con(S.T, r, ax(0))
        return out.reshape(u.shape)
    gx = _con(D, tzy, ax(2))
    tzd = _con(D, tz, ax(1))
    gy = _con(S, tzd, ax(2))
    tdz = _con(D, t, ax(0))
    tdzy = _con(S, tdz, ax(1))
    gz = _con(S, tdzy, ax(2))
    hx, hy, hz = spacing
    gx = gx * (wb * (0.5 / hx**2))
    gy = gy * (wb * (0.5 / hy**2))
    gz = gz * (wb * (0.5 / hz**2))
    a = _con(D.T, gx, ax(2))
    if v_q is not None:
        vb = np.asarray(v_q).reshape(lead + (n, n, n, 1)) if np.ndim(v_q) > 1 else \
            np.asarray(v_q).reshape((1,) * b + (n, n, n, 1))
        a = a + _con(S.T, uq * (wb * vb), ax(2))
    by = _con(S.T, gy, ax(2))
    czl = _con(S.T, gz, ax(2))
    ab = _con(S.T, a, ax(1)) + _con(D.T, by, ax(1))
    cc = _con(S.T, czl, ax(1))
    out = _con(S.T, ab, ax(0)) + _con(D.T, cc, ax(0))
    return out.reshape(u.shape)


def element_matrix(degree, spacing, kind, v_q=None):
    """Dense element matrix by direct quadrature (matfree.py:375-397), symmetrised."""
    S, D, _, _ = lagrange_tables(degree)
    w = weights3(degree, spacing).ravel()
    n3 = np.kron(S, np.kron(S, S))
    if kind == "mass":
        m = n3.T @ (w[:, None] * n3)
    else:
        g3 = (np.kron(S, np.kron(S, D)), np.kron(S, np.kron(D, S)), np.kron(D, np.kron(S, S)))
        m = np.zeros((n3.shape[1],) * 2)
        for g, h in zip(g3, spacing):
            m += g.T @ ((w * (0.5 / h**2))[:, None] * g)
        if v_q is not None:
            m += n3.T @ ((w * v_q)[:, None] * n3)
    u = np.triu(m)
    return u + u.T - np.diag(np.diag(m))


# -- operator application on dense multivectors ----------------------------------


def sample_potential(potential, cell_origins, degree, spacing):
    """(n_cells, q^3) V at the cell quadrature points (matfree.py:35-40,491-495)."""
    qo = quad_offsets(degree, spacing)
    if potential is None:
        return None
    if not callable(potential):
        return np.full((cell_origins.shape[0], qo.shape[0]), float(potential))
    pts = (cell_origins[:, None, :] + qo[None, :, :]).reshape(-1, 3)
    return np.asarray(potential(pts), dtype=float).reshape(cell_origins.shape[0], -1)


def apply_dense(cell_nodes, cell_origins, degree, spacing, kind, potential, xd, chunk=2048):
    """Y = Op X for dense X (n_dofs x M): sum over cells of scatter(cell integral(gather))."""
    n_dofs, m = xd.shape
    out = np.zeros_like(xd)
    for c0 in range(0, cell_nodes.shape[0], chunk):
        nodes = cell_nodes[c0 : c0 + chunk]
        u = xd[nodes]  # (c, n3, M)
        vq = None
        if kind != "mass" and potential is not None:
            vq = sample_potential(potential, cell_origins[c0 : c0 + chunk], degree, spacing)
        r = cell_integrals(degree, spacing, kind, u, vq)
        rows = nodes.ravel()
        scat = sparse.csr_matrix((np.ones(rows.size), (rows, np.arange(rows.size))),
                                 shape=(n_dofs, rows.size))
        out += scat @ r.reshape(-1, m)
    return out


def assembled_operator(cell_nodes, cell_origins, degree, spacing, kind, potential, n_dofs):
    """Exactly symmetric assembled CSR (matfree.py:530-575)."""
    rows, cols, vals = [], [], []
    vqs = sample_potential(potential, cell_origins, degree, spacing) if kind != "mass" else None
    for c in range(cell_nodes.shape[0]):
        ek = element_matrix(degree, spacing, kind, None if vqs is None else vqs[c])
        gi = cell_nodes[c]
        I = np.repeat(gi, gi.size)
        J = np.tile(gi, gi.size)
        keep = I <= J
        rows.append(I[keep])
        cols.append(J[keep])
        vals.append(ek.ravel()[keep])
    up = sparse.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                           shape=(n_dofs, n_dofs)).tocsr()
    return (up + up.T - sparse.diags(up.diagonal())).tocsr()


# -- dense SpMM oracles (bcsr.py:587-667) ------------------------------------------


def tmmult_dense(a_dense, b_dense, c_mask):
    """C = A^T B restricted to C's pattern (the reference raises if a product block is absent)."""
    return np.where(c_mask, a_dense.T @ b_dense, 0.0)


def mmult_dense(a_dense, b_dense, c_mask, alpha=1.0, c_prev=None):
    """C = alpha A B truncated to C's pattern (+ previous content with accumulate)."""
    prod = np.where(c_mask, alpha * (a_dense @ b_dense), 0.0)
    return prod if c_prev is None else c_prev + prod


def per_vector_rel_err(got, want):
    """max over columns of ||got_j - want_j|| / ||want_j|| (columns with want_j != 0)."""
    num = np.linalg.norm(got - want, axis=0)
    den = np.linalg.norm(want, axis=0)
    ok = den > 0
    if not ok.any():
        return float(np.max(num)) if num.size else 0.0
    return float(max(np.max(num[ok] / den[ok]), np.max(num[~ok]) if (~ok).any() else 0.0))
