"""CPU emulation of the K4 / K5 chunk kernels (csrc/bmv_spmm.cu) over their
host plans (spmm.py / bmv_plan.cpp bmvp_chunk_plan), TEST INFRASTRUCTURE:
every part's chunks are staged exactly as the producer warp does (meta words
+ the A and B element ranges) and the consumer arithmetic is replayed from
the staged bytes only, asserting every read stays inside the stage."""

from __future__ import annotations

import numpy as np

H_NSEG, H_NROWS, H_UA, H_UB, H_NK, H_AOFF, H_BOFF, H_SEG, H_CMA, H_CMB, H_RB, H_KK, H_ST = range(13)


def _segments(meta, nseg):
    """(rows, A offset, K_A, B / Y offset, K_B) per segment."""
    w = int(meta[H_SEG])
    rec = meta[w : w + 8 * nseg].astype(np.int64).reshape(nseg, 8)
    assert np.all(rec[:, 5:] == 0)
    return rec[:, :5]


def _stage(arr, j, a, b):
    m0, m1 = int(arr["chunk_meta"][j]), int(arr["chunk_meta"][j + 1])
    meta = arr["meta"][m0:m1]
    a0, a1 = (int(v) for v in arr["chunk_a"][2 * j : 2 * j + 2])
    av = a[a0:a1]
    assert meta[H_AOFF] == 4 * (m1 - m0)
    total = 4 * (m1 - m0) + 8 * (a1 - a0)
    bv = None
    if arr["chunk_b"] is not None:
        b0, b1 = (int(v) for v in arr["chunk_b"][2 * j : 2 * j + 2])
        bv = b[b0:b1]
        assert meta[H_BOFF] == meta[H_AOFF] + 8 * (a1 - a0)
        total += 8 * (b1 - b0)
    assert total <= arr["stage_bytes"], (total, arr["stage_bytes"])
    return meta, av, bv


def _colmap(meta, word, nbr, u):
    raw = meta[word : word + (nbr * u + 1) // 2].astype(np.int32).view(np.int16)
    return raw[: nbr * u].reshape(nbr, u).astype(np.int64)


def _check_parts(arr):
    ps = arr["part_chunk_start"]
    assert ps[0] == 0 and ps[-1] == arr["n_chunks"] and np.all(np.diff(ps) >= 0)


def emulate_tmmult(arr, a, b, c_len):
    """c = A^T B as K4 computes it (c zeroed first)."""
    _check_parts(arr)
    c = np.zeros(c_len)
    for j in range(arr["n_chunks"]):
        meta, av, bv = _stage(arr, j, a, b)
        nseg, nrows, ua, ub = (int(meta[k]) for k in (H_NSEG, H_NROWS, H_UA, H_UB))
        segs = _segments(meta, nseg)
        assert int(segs[:, 0].sum()) == nrows
        cma = _colmap(meta, int(meta[H_CMA]), nseg, ua)
        cmb = _colmap(meta, int(meta[H_CMB]), nseg, ub)
        prod = np.zeros((ua, ub))
        for s, (n, ao, ka, bo, kb) in enumerate(segs):
            sa, sb = cma[s], cmb[s]
            assert sa.max(initial=-1) < ka and sb.max(initial=-1) < kb
            assert ao + n * ka <= av.size and bo + n * kb <= bv.size
            A = np.zeros((n, ua))
            B = np.zeros((n, ub))
            A[:, sa >= 0] = av[ao : ao + n * ka].reshape(n, ka)[:, sa[sa >= 0]]
            B[:, sb >= 0] = bv[bo : bo + n * kb].reshape(n, kb)[:, sb[sb >= 0]]
            prod += A.T @ B
        rb = meta[meta[H_RB] : meta[H_RB] + ua].astype(np.int64)
        kk = meta[meta[H_KK] : meta[H_KK] + ua].astype(np.int64)
        nk = int(meta[H_NK])
        st = meta[meta[H_ST] : meta[H_ST] + nk * ub].astype(np.int64).reshape(nk, ub)
        for aa in range(ua):
            sl = st[kk[aa]]
            ok = sl >= 0
            np.add.at(c, rb[aa] + sl[ok], prod[aa, ok])
            assert np.all(prod[aa, ~ok] == 0.0), "product entry without an S slot"
    return c


def emulate_mmult(arr, a, cmat, y, alpha, accumulate):
    """y = alpha A C (+ y) on the stored entries of the plan's rows."""
    _check_parts(arr)
    y = y.copy()
    for j in range(arr["n_chunks"]):
        meta, av, _ = _stage(arr, j, a, None)
        nseg, nrows, ua, ub = (int(meta[k]) for k in (H_NSEG, H_NROWS, H_UA, H_UB))
        segs = _segments(meta, nseg)
        assert int(segs[:, 0].sum()) == nrows
        cma = _colmap(meta, int(meta[H_CMA]), nseg, ua)
        cmy = _colmap(meta, int(meta[H_CMB]), nseg, ub)
        cb = meta[meta[H_RB] : meta[H_RB] + ua].astype(np.int64)
        ck = meta[meta[H_KK] : meta[H_KK] + ua].astype(np.int64)
        nk = int(meta[H_NK])
        ct = meta[meta[H_ST] : meta[H_ST] + nk * ub].astype(np.int64).reshape(nk, ub)
        C = np.zeros((ua, ub))
        for aa in range(ua):
            sl = ct[ck[aa]]
            C[aa, sl >= 0] = cmat[cb[aa] + sl[sl >= 0]]
        for s, (n, ao, ka, yo, ky) in enumerate(segs):
            sa, sy = cma[s], cmy[s]
            assert sa.max(initial=-1) < ka and sy.max(initial=-1) < ky
            assert ao + n * ka <= av.size
            A = np.zeros((n, ua))
            A[:, sa >= 0] = av[ao : ao + n * ka].reshape(n, ka)[:, sa[sa >= 0]]
            D = alpha * (A @ C)
            ok = sy >= 0
            assert np.count_nonzero(ok) == ky, "a stored Y column outside the union"
            idx = yo + np.arange(n)[:, None] * ky + sy[ok][None, :]
            y[idx] = D[:, ok] + (y[idx] if accumulate else 0.0)
    return y
