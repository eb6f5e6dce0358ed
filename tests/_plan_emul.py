"""CPU emulation of the K4 / K5 streaming kernels over their host plans.

Executes what csrc/bmv_tma.cuh (producer: copy lists -> stage bytes),
csrc/bmv_project.cu and csrc/bmv_postmul.cu (consumers: header, work
descriptors, warp slots, partial layout, reduction order) do with a plan,
in numpy, reading everything back from the emulated stage and asserting
every read stays inside what was staged, so plan bugs surface on CPU.
Tests only.
"""

from __future__ import annotations

import numpy as np

PJ_WARPS, PJ_SLOTS, PJ_HDR = 16, 8, 272
PM_WARPS = 16


def _subs(arr):
    """Yield (sub index, staged bytes, staged mask) per sub-chunk, part by part."""
    cps = arr["copies"].reshape(-1, 4).astype(np.int64) & 0xFFFFFFFF
    pss, pes = arr["part_sub_start"], arr["part_entry_start"]
    for p in range(int(arr["n_parts"])):
        e = int(pes[p])
        for s in range(int(pss[p]), int(pss[p + 1])):
            first = e
            ents = []
            while True:
                assert e < pes[p + 1], "malformed copy list"
                ents.append(cps[e])
                e += 1
                if (ents[-1][1] >> 30) & 1:
                    break
            yield s, ents
        assert e == pes[p + 1], "stray copy entries"


def _stage(ents, srcs, stage_bytes):
    buf = np.zeros(stage_bytes, dtype=np.uint8)
    mask = np.zeros(stage_bytes, dtype=bool)
    for x, y, lo, hi in ents:
        n, sel = int(y & ((1 << 28) - 1)), int((y >> 28) & 3)
        src = int(lo) | (int(hi) << 32)
        assert x + n <= stage_bytes, "copy past the stage"
        assert not mask[x:x + n].any(), "copies overlap"
        buf[x:x + n] = srcs[sel][src:src + n]
        mask[x:x + n] = True
    return buf, mask


def _dbl(buf, mask, off, n):
    """n doubles at double offset off, all staged."""
    assert off >= 0 and mask[8 * off: 8 * (off + n)].all(), "read outside the staged bytes"
    return buf[8 * off: 8 * (off + n)].view(np.float64)


def emulate_tmmult(arr, a_data, b_data, c_len):
    srcs = [arr["meta"].view(np.uint8), a_data.view(np.uint8), b_data.view(np.uint8)]
    sb = int(arr["stage_bytes"])
    partial = np.zeros((int(arr["n_items"]) * PJ_WARPS * PJ_SLOTS, 8, 8))
    slots = np.zeros((PJ_WARPS, PJ_SLOTS, 8, 8))
    for s, ents in _subs(arr):
        buf, mask = _stage(ents, srcs, sb)
        hdr = buf[:PJ_HDR].view(np.int32)
        n_tri, n_units = int(hdr[PJ_WARPS]), int(hdr[19])
        tri = buf[PJ_HDR:PJ_HDR + 16 * n_tri].view(np.int32).reshape(-1, 4).astype(np.int64) & 0xFFFFFFFF
        res = np.full((32, 8, 8), np.nan)
        done = np.zeros(32, dtype=bool)
        for w in range(PJ_WARPS):
            t, t1 = int(hdr[w]), int(hdr[w + 1])
            while t < t1:
                unit = (tri[t][2] >> 16) & 0xFF
                assert unit < n_units and not done[unit], "unit computed twice"
                acc = np.zeros((8, 8))
                while t < t1 and ((tri[t][2] >> 16) & 0xFF) == unit:
                    x, y, z, ww = tri[t]
                    rows, ac, bc = z & 0xFFFF, (z >> 24) & 15, (z >> 28) & 15
                    a_s, b_s = ww & 0xFFFF, ww >> 16
                    am = np.stack([_dbl(buf, mask, x + r * a_s, ac) for r in range(rows)])
                    bm = np.stack([_dbl(buf, mask, y + r * b_s, bc) for r in range(rows)])
                    acc[:ac, :bc] += am.T @ bm
                    t += 1
                res[unit] = acc
                done[unit] = True
        assert done[:n_units].all(), "unit never computed"
        for u in range(n_units):
            ow = int(hdr[36 + u])
            slots[ow & 0xFF, ow >> 8] += res[u]
        if hdr[18]:
            it = int(hdr[17])
            for w in range(PJ_WARPS):
                for k in range(hdr[20 + w]):
                    partial[(it * PJ_WARPS + w) * PJ_SLOTS + k] = slots[w, k]
                slots[w] = 0.0
    assert not slots.any(), "slot left unflushed"
    c = np.zeros(c_len)
    shp = arr["tile_shape"].reshape(-1, 3)
    for t in range(arr["tile_off"].size):
        acc = np.zeros((8, 8))
        for j in range(arr["tile_src_start"][t], arr["tile_src_start"][t + 1]):
            acc += partial[arr["tile_src"][j]]
        r, cc, st = shp[t]
        for i in range(r):
            o = arr["tile_off"][t] + i * st
            c[o:o + cc] = acc[i, :cc]
    return c


def emulate_mmult(arr, a_data, b_data, c_data, alpha=1.0, accumulate=False):
    c = c_data.copy() if accumulate else np.zeros_like(c_data)
    written = np.zeros(c.size, dtype=bool)
    srcs = [arr["meta"].view(np.uint8), a_data.view(np.uint8), b_data.view(np.uint8)]
    sb = int(arr["stage_bytes"])
    for s, ents in _subs(arr):
        buf, mask = _stage(ents, srcs, sb)
        nt = int(buf[:16].view(np.int32)[0])
        meta = buf[16:].view(np.int32)
        tasks = meta[:4 * nt].reshape(-1, 4).astype(np.int64) & 0xFFFFFFFF
        for k in range(nt):
            off, y, z, mi0 = tasks[k]
            rows, cv, ni, ys = y & 0x7F, (y >> 8) & 15, (y >> 12) & 15, y >> 16
            p0, npairs = z & 0xFFFF, z >> 16
            assert rows <= 64 and cv <= 8
            acc = np.zeros((rows, cv))
            for p in range(p0, p0 + npairs):
                q = meta[4 * (nt + p): 4 * (nt + p) + 4].astype(np.int64)
                a_s, inner, bs = q[1] & 0xFFFF, q[1] >> 16, q[2]
                am = np.stack([_dbl(buf, mask, q[0] + (8 * mi0 + r) * a_s, inner) for r in range(rows)])
                bm = np.stack([_dbl(buf, mask, q[3] + kk * bs + 8 * ni, cv) for kk in range(inner)])
                acc += am @ bm
            for i in range(rows):
                o = off + i * ys
                assert not written[o:o + cv].any(), "output written twice"
                written[o:o + cv] = True
                c[o:o + cv] = (c[o:o + cv] if accumulate else 0.0) + alpha * acc[i]
    return c
