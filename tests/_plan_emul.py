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


# -- lane-compacted kernels (csrc/bmv_spmm_lane.cu) -----------------------------


def _i32(buf, byte_off, n):
    return buf[byte_off:byte_off + 4 * n].view(np.int32)


def emulate_tmmult_lane(arr, a_data, b_data, c_len):
    """k4_lane_kernel over a lane plan: tiles -> shared accumulator -> flush."""
    srcs = [arr["meta"].view(np.uint8), a_data.view(np.uint8), b_data.view(np.uint8)]
    sb = arr["stage_bytes"]
    out = np.zeros(c_len)
    acc = np.zeros(64 * 64)
    pss = arr["part_sub_start"]
    for s_idx, ents in _subs(arr):
        if s_idx in pss:  # a new CTA: its accumulator starts empty
            assert not acc.any(), "accumulator of the previous part not flushed"
        buf, mask = _stage(ents, srcs, sb)
        hdr = _i32(buf, 0, 4)
        n_tiles, n_flush, rec_off, fl_off = (int(v) for v in hdr)
        dbl = buf[: sb - sb % 8].view(np.float64)
        dmask = mask[: sb - sb % 8].reshape(-1, 8).all(axis=1)
        for t in range(n_tiles):
            r = _i32(buf, 4 * (rec_off + 20 * t), 20)
            rows, bs = int(r[17]) & 0xFFFF, int(r[17]) >> 16
            nb = int(r[18])
            B = np.zeros((rows, 8))
            for n in range(nb):
                idx = int(r[16]) + n + bs * np.arange(rows)
                assert dmask[idx].all(), "B read outside the staged data"
                B[:, n] = dbl[idx]
            for m in range(8):
                ac = int(r[m])
                if ac < 0 or int(r[8 + m]) < 0:
                    continue
                ao, as_ = ac & 0xFFFF, (ac >> 16) & 0x7FFF
                idx = ao + as_ * np.arange(rows)
                assert dmask[idx].all(), "A read outside the staged data"
                acc[int(r[8 + m]): int(r[8 + m]) + nb] += dbl[idx] @ B[:, :nb]
        for f in range(n_flush):
            x, y, z, w = (int(v) for v in _i32(buf, 4 * fl_off + 16 * f, 4))
            rr, cc = z & 0xFF, (z >> 8) & 0xFF
            tile = acc[w * 64: w * 64 + 64].reshape(8, 8)
            for row in range(rr):
                out[x + row * y: x + row * y + cc] += tile[row, :cc]
            acc[w * 64: w * 64 + 64] = 0.0
    assert not acc.any(), "accumulator not flushed"
    return out


def emulate_mmult_lane(arr, a_data, b_data, c_data, alpha=1.0, accumulate=False):
    """k5_lane_kernel over a lane plan (c_data: the output before the call)."""
    srcs = [arr["meta"].view(np.uint8), a_data.view(np.uint8)]
    sb = arr["stage_bytes"]
    out = c_data.copy()
    for _s, ents in _subs(arr):
        buf, mask = _stage(ents, srcs, sb)
        n_tasks, toff = (int(v) for v in _i32(buf, 0, 2))
        dbl = buf[: sb - sb % 8].view(np.float64)
        dmask = mask[: sb - sb % 8].reshape(-1, 8).all(axis=1)
        offs = _i32(buf, 4 * toff, n_tasks)
        for t in range(n_tasks):
            r0 = int(offs[t])
            head = _i32(buf, 4 * r0, 4)
            yoff = (int(head[0]) & 0xFFFFFFFF) | (int(head[1]) << 32)
            rows, ys = int(head[2]) & 0xFFFF, int(head[2]) >> 16
            ncol, nst, ks = int(head[3]) & 0xFF, (int(head[3]) >> 8) & 0xFF, int(head[3]) >> 16
            rec = _i32(buf, 4 * (r0 + 4), 8 * ks)
            D = np.zeros((rows, 8))
            for s in range(ks):
                for m in range(4):
                    ac, co = int(rec[8 * s + m]), int(rec[8 * s + 4 + m])
                    if ac < 0 or co < 0:
                        continue
                    ao, as_ = ac & 0xFFFF, (ac >> 16) & 0x7FFF
                    idx = ao + as_ * np.arange(rows)
                    assert dmask[idx].all(), "A read outside the staged data"
                    crow = np.zeros(8)
                    crow[:ncol] = b_data[co: co + ncol]
                    D += np.outer(dbl[idx], crow)
            for row in range(rows):
                p = yoff + row * ys
                v = alpha * D[row, :nst]
                out[p: p + nst] = (out[p: p + nst] + v) if accumulate else v
    return out
