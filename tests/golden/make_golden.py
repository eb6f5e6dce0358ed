"""Generate golden fixtures from the REFERENCE package (run in the build container).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports `bcsrmv` from /root/reference/pkg/src (pure Python; read-only) and
writes small .npz fixtures plus a JSON of sha256 digests of the full-size
index maps.  The fixtures are committed; the GPU box never reads the
reference.  Everything is computed with the reference's public API, in
the configuration choices of SURVEY.md section 0.1 (L = 0, B = 8, one
vector per centre, 2 * hashed fill masked by the support, Gaussian
potential).
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from bcsrmv.bcsr import BlockCsrMatrix, mmult, tmmult  # noqa: E402
from bcsrmv.bench.problem import hashed_values  # noqa: E402
from bcsrmv.comm import run_ranks  # noqa: E402
from bcsrmv.energy import (  # noqa: E402
    column_space_ghost_blocks,
    compute_energy,
    compute_gradient,
    directional_derivative,
    make_column_layout,
    make_workspace,
    projected_pattern,
)
from bcsrmv.localization import (  # noqa: E402
    build_support_sparsity,
    column_supports,
    grow_sparsity_for_operator,
    order_and_block_columns,
)
from bcsrmv.matfree import CellOperator, hamiltonian_operator, make_dof_layout, mass_operator  # noqa: E402
from bcsrmv.mesh import build_mesh, enumerate_dofs, partition_and_order_cells  # noqa: E402

OUT = Path(__file__).resolve().parent


def gaussian(centers, sigma):
    centers = np.asarray(centers, dtype=float)
    inv = 1.0 / (sigma * sigma)

    def v(points):
        pts = np.atleast_2d(points)
        out = np.zeros(pts.shape[0])
        for c in centers:
            d = pts - c
            out += np.exp(-(d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1] + d[:, 2] * d[:, 2]) * inv)
        return -out

    return v


def cosine(seed):
    def v(points):
        return np.cos(np.atleast_2d(points) @ np.asarray([0.8, 1.4, 0.5]) + seed)

    return v


def lattice(counts, spacing, offset):
    nx, ny, nz = counts
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    return offset + spacing * np.stack([i.ravel(), j.ravel(), k.ravel()], axis=1).astype(float)


def setup(extents, spacing, level, degree, centers, radius, vpc, bs, n_ranks):
    mesh = build_mesh(extents, spacing, level)
    part = partition_and_order_cells(mesh, n_ranks)
    num = enumerate_dofs(mesh, part, degree)
    lay = order_and_block_columns(mesh, part, centers, radius, vpc, bs)
    sup = column_supports(mesh, num, lay)
    pat = build_support_sparsity(mesh, part, num, lay, sup)
    gro = grow_sparsity_for_operator(pat, mesh, num)
    return mesh, part, num, lay, sup, pat, gro


def structure_arrays(prefix, part, num, lay, sup, pat, gro, proj=None):
    d = {
        f"{prefix}ordered_cells": part.ordered_cells,
        f"{prefix}rank_group_start": part.rank_group_start,
        f"{prefix}new_index_of_node": num.new_index_of_node,
        f"{prefix}row_block_sizes": num.row_blocks.sizes,
        f"{prefix}owned_ranges": np.asarray(num.owned_ranges, dtype=np.int64),
        f"{prefix}rank_block_start": num.rank_block_start,
        f"{prefix}old_col_of_new": lay.old_col_of_new,
        f"{prefix}col_block_sizes": lay.column_blocks.sizes,
        f"{prefix}col_rank_block_start": lay.rank_block_start,
        f"{prefix}support_ptr": np.concatenate([[0], np.cumsum([s.size for s in sup])]),
        f"{prefix}support_rows": np.concatenate(sup),
        f"{prefix}pattern_row_start": pat.row_start,
        f"{prefix}pattern_col_index": pat.col_index,
        f"{prefix}grown_row_start": gro.row_start,
        f"{prefix}grown_col_index": gro.col_index,
    }
    if proj is not None:
        d[f"{prefix}proj_row_start"] = proj.row_start
        d[f"{prefix}proj_col_index"] = proj.col_index
    return d


def support_mask(num, lay, sup):
    m = np.zeros((num.n_dofs, lay.n_columns), dtype=bool)
    for new in range(lay.n_columns):
        m[sup[int(lay.old_col_of_new[new]) // lay.vectors_per_center], new] = True
    return m


def filler(lay, sup, seed, scale=2.0, zero_rows=None):
    old = lay.old_col_of_new
    v = lay.vectors_per_center

    def values(rows, cols):
        o = old[cols]
        vals = scale * hashed_values(seed, rows, o)
        for j, oc in enumerate(o):
            inside = np.isin(rows, sup[oc // v], assume_unique=True)
            vals[~inside, j] = 0.0
        if zero_rows is not None:
            vals[np.isin(rows, zero_rows)] = 0.0
        return vals

    return values


def boundary_rows(mesh, num, degree):
    sx, sy, sz = mesh.node_grid_shape(degree)
    k, j, i = np.meshgrid(np.arange(sz), np.arange(sy), np.arange(sx), indexing="ij")
    b = ((i == 0) | (i == sx - 1) | (j == 0) | (j == sy - 1) | (k == 0) | (k == sz - 1)).ravel()
    return np.sort(num.new_index_of_node[np.flatnonzero(b)])


def make_smoke():
    centers = lattice((2, 2, 2), 0.5, 0.25)
    mesh, part, num, lay, sup, pat, gro = setup((8, 8, 8), (1 / 8,) * 3, 0, 2, centers, 0.3, 1, 8, 1)
    proj = projected_pattern(pat, gro)
    pot = gaussian(centers, 0.2)
    smask = support_mask(num, lay, sup)
    ov = (smask.T.astype(np.int64) @ smask.astype(np.int64)) > 0
    bnd = boundary_rows(mesh, num, 2)
    out = structure_arrays("", part, num, lay, sup, pat, gro, proj)
    old = lay.old_col_of_new

    def program(ctx, zero_rows):
        rl = make_dof_layout(ctx, mesh, part, num)
        op = CellOperator(mesh, part, num, rl)
        x = BlockCsrMatrix(pat, rl, ctx, 8)
        x.fill_owned(filler(lay, sup, 1, zero_rows=zero_rows))
        hx = BlockCsrMatrix(gro, rl, ctx, 8)
        op.apply(hamiltonian_operator(pot), x, hx)
        res = {"x": x.to_dense_owned(), "hx": hx.to_dense_owned()}
        if zero_rows is not None:
            return res
        ghosts = column_space_ghost_blocks(gro, proj, rl, lay.rank_block_start, ctx.rank)
        cl = make_column_layout(ctx, lay.column_blocks, lay.rank_block_start, ghosts)
        s = BlockCsrMatrix(proj, cl, ctx, 8)
        tmmult(x, hx, s)
        c = BlockCsrMatrix(proj, cl, ctx, 8)
        c.fill_owned(lambda r, cc: np.where(ov[np.ix_(r, cc)], 2.0 * hashed_values(7, old[r], old[cc]), 0.0))
        c.update_ghost_values()
        xc = BlockCsrMatrix(pat, rl, ctx, 8)
        mmult(x, c, xc)
        hm = BlockCsrMatrix(gro, rl, ctx, 8)
        op.apply(mass_operator(), x, hm)
        res.update(s=s.to_dense_owned(), c=c.to_dense_owned(), xc=xc.to_dense_owned(),
                   mx=hm.to_dense_owned())
        return res

    r = run_ranks(1, program, None)[0]
    rd = run_ranks(1, program, bnd)[0]
    hx_d = rd["hx"].copy()
    hx_d[bnd] = 0.0
    out.update({"x": r["x"], "hx": r["hx"], "s": r["s"], "c": r["c"], "xc": r["xc"], "mx": r["mx"],
                "x_dirichlet": rd["x"], "hx_dirichlet": hx_d, "boundary_rows": bnd,
                "centers": centers, "overlap": ov})
    np.savez_compressed(OUT / "smoke.npz", **out)
    print("smoke.npz", {k: v.shape for k, v in out.items() if k in ("x", "hx", "s")})


def make_energy():
    """The OM energy / gradient composition (reference energy.py:129-174) on the
    smoke config at 1 and 2 ranks: E, G, mbar, hbar and the slope tr(G^T G)."""
    centers = lattice((2, 2, 2), 0.5, 0.25)
    out = {}
    for n_ranks in (1, 2):
        mesh, part, num, lay, sup, pat, gro = setup((8, 8, 8), (1 / 8,) * 3, 0, 2, centers, 0.3, 1,
                                                    8, n_ranks)
        pot = gaussian(centers, 0.2)

        def program(ctx):
            rl = make_dof_layout(ctx, mesh, part, num)
            op = CellOperator(mesh, part, num, rl)
            x = BlockCsrMatrix(pat, rl, ctx, 8)
            x.fill_owned(filler(lay, sup, 1, scale=0.25))
            ws = make_workspace(ctx, op, x, lay)
            e = compute_energy(op, mass_operator(), hamiltonian_operator(pot), x, ws)
            g = compute_gradient(ws)
            slope = directional_derivative(g, g)
            return (e, slope, g.to_dense_owned(), ws.mbar.to_dense_owned(),
                    ws.hbar.to_dense_owned(), ws.phi_m.to_dense_owned())

        parts = run_ranks(n_ranks, program)
        out[f"r{n_ranks}_energy"] = np.asarray(parts[0][0])
        out[f"r{n_ranks}_slope"] = np.asarray(parts[0][1])
        for k, name in ((2, "g"), (3, "mbar"), (4, "hbar"), (5, "phi_m")):
            out[f"r{n_ranks}_{name}"] = np.sum([p[k] for p in parts], axis=0)
    np.savez_compressed(OUT / "energy.npz", **out)
    print("energy.npz", {k: (v.shape if v.ndim else float(v)) for k, v in out.items()})


def make_random():
    """Acceptance-style small problems (test_acceptance.py:68-127): p=1..4, ranks 1/2/4."""
    meshes = {1: (8, 8, 8), 2: (6, 6, 6), 3: (4, 4, 4), 4: (4, 4, 4)}
    rng = np.random.default_rng(2024)
    out = {}
    for degree, extents in meshes.items():
        centers = rng.random((int(rng.integers(2, 4)), 3)) * np.asarray(extents, dtype=float)
        radius = float(rng.uniform(1.0, 1.8))
        out[f"p{degree}_centers"] = centers
        out[f"p{degree}_radius"] = np.asarray(radius)
        out[f"p{degree}_extents"] = np.asarray(extents)
        for n_ranks in (1, 2, 4):
            mesh, part, num, lay, sup, pat, gro = setup(extents, (1.0, 1.0, 1.0), 1, degree,
                                                        centers, radius, 2, 3, n_ranks)
            out.update(structure_arrays(f"p{degree}_r{n_ranks}_", part, num, lay, sup, pat, gro))
            for kind, spec in (("h", hamiltonian_operator(cosine(degree))), ("m", mass_operator())):

                def program(ctx):
                    rl = make_dof_layout(ctx, mesh, part, num)
                    op = CellOperator(mesh, part, num, rl)
                    x = BlockCsrMatrix(pat, rl, ctx, 8)
                    x.fill_owned(filler(lay, sup, 10 * degree, scale=1.0))
                    hx = BlockCsrMatrix(gro, rl, ctx, 8)
                    op.apply(spec, x, hx)
                    return x.to_dense_owned(), hx.to_dense_owned()

                parts = run_ranks(n_ranks, program)
                out[f"p{degree}_r{n_ranks}_x"] = np.sum([p[0] for p in parts], axis=0)
                out[f"p{degree}_r{n_ranks}_{kind}x"] = np.sum([p[1] for p in parts], axis=0)
    np.savez_compressed(OUT / "random.npz", **out)
    print("random.npz", len(out), "arrays")


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes()).hexdigest()


def make_digests(only=None):
    cfgs = {
        "q2": ((32, 32, 32), (1 / 32,) * 3, 2, lattice((4, 4, 4), 0.25, 0.125), 0.25, 1),
        "q4": ((32, 32, 32), (1 / 32,) * 3, 4, lattice((4, 4, 4), 0.25, 0.125), 0.25, 1),
        "proj": ((64, 64, 64), (1 / 64,) * 3, 2, lattice((8, 8, 8), 1 / 8, 1 / 16), 1.5 / 8, 1),
        "weak1": ((64, 64, 64), (1 / 64,) * 3, 4, lattice((8, 8, 8), 8 / 64, 4 / 64), 8 / 64, 1),
        "weak2": ((64, 64, 128), (1 / 64,) * 3, 4, lattice((8, 8, 16), 8 / 64, 4 / 64), 8 / 64, 2),
        "weak4": ((64, 64, 256), (1 / 64,) * 3, 4, lattice((8, 8, 32), 8 / 64, 4 / 64), 8 / 64, 4),
        "weak8": ((64, 64, 512), (1 / 64,) * 3, 4, lattice((8, 8, 64), 8 / 64, 4 / 64), 8 / 64, 8),
    }
    path = OUT / "digests.json"
    res = json.loads(path.read_text()) if (only and path.exists()) else {}
    for name, (ext, sp, deg, centers, radius, nr) in cfgs.items():
        if only and name not in only:
            continue
        t0 = time.time()
        mesh, part, num, lay, sup, pat, gro = setup(ext, sp, 0, deg, centers, radius, 1, 8, nr)
        arrays = structure_arrays("", part, num, lay, sup, pat, gro)
        if name in ("q2", "proj"):
            proj = projected_pattern(pat, gro)
            arrays["proj_row_start"] = proj.row_start
            arrays["proj_col_index"] = proj.col_index
        res[name] = {k: digest(v) for k, v in arrays.items()}
        res[name]["_sizes"] = {"n_dofs": int(num.n_dofs), "pattern_blocks": int(pat.col_index.size),
                               "grown_blocks": int(gro.col_index.size),
                               "support_nnz": int(sum(s.size for s in sup))}
        print(name, "%.1fs" % (time.time() - t0), res[name]["_sizes"], flush=True)
        path.write_text(json.dumps(res, indent=1, sort_keys=True))


if __name__ == "__main__":
    which = sys.argv[1:] or ["smoke", "random", "digests", "energy"]
    if "smoke" in which:
        make_smoke()
    if "energy" in which:
        make_energy()
    if "random" in which:
        make_random()
    if "digests" in which:
        make_digests()
    extra = [w for w in which if w.startswith("weak") or w in ("q2", "q4", "proj")]
    if extra:  # e.g. `python make_golden.py weak4 weak8`: add those digests to digests.json
        make_digests(extra)
