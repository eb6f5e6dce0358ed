"""CPU emulation of the K4 / K5 streaming kernels over their host plans.

Executes exactly what csrc/bmv_project.cu and csrc/bmv_postmul.cu do with a
plan (stage contents, tile offsets, warp slots, partial layout, reduction
order) in numpy, and asserts every stage read stays inside the staged
range, so plan bugs surface on CPU.  Tests only.
"""

from __future__ import annotations

import numpy as np

W, SLOTS = 8, 16


def emulate_tmmult(arr, a_data, b_data, c_len):
    sa = arr["sub_a"].reshape(-1, 2)
    sb = arr["sub_b"].reshape(-1, 2)
    tri = arr["tri"].reshape(-1, 4).astype(np.int64) & 0xFFFFFFFF
    pss, sts, item = arr["part_sub_start"], arr["sub_tri_start"], arr["sub_item"]
    cap = int(arr["stage_doubles"])
    partial = np.zeros((int(arr["n_items"]) * W * SLOTS, 8, 8))
    slots = np.zeros((W, SLOTS, 8, 8))
    for p in range(int(arr["n_parts"])):
        for s in range(pss[p], pss[p + 1]):
            na, nb = sa[s, 1] - sa[s, 0], sb[s, 1] - sb[s, 0]
            boff = na + (na & 1)
            assert boff + nb <= cap
            S = np.full(cap + 64 * 16, np.nan)
            S[:na] = a_data[sa[s, 0]:sa[s, 1]]
            S[boff:boff + nb] = b_data[sb[s, 0]:sb[s, 1]]
            for w in range(W):
                for t in range(sts[s * W + w], sts[s * W + w + 1]):
                    x, y, z, ww = tri[t]
                    rows, slot, ac, bc = z & 0xFFFF, (z >> 16) & 0xFF, (z >> 24) & 15, (z >> 28) & 15
                    a_s, b_s = ww & 0xFFFF, ww >> 16
                    assert 0 <= x and x + (rows - 1) * a_s + ac <= na, "A tile outside the stage"
                    assert boff <= y and y + (rows - 1) * b_s + bc <= boff + nb, "B tile outside"
                    am = np.stack([S[x + r * a_s: x + r * a_s + ac] for r in range(rows)])
                    bm = np.stack([S[y + r * b_s: y + r * b_s + bc] for r in range(rows)])
                    slots[w, slot, :ac, :bc] += am.T @ bm
            it = item[s]
            if s + 1 == pss[p + 1] or item[s + 1] != it:
                for w in range(W):
                    for k in range(arr["item_slots"][it * W + w]):
                        partial[(it * W + w) * SLOTS + k] = slots[w, k]
                        slots[w, k] = 0.0
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
    sa = arr["sub_a"].reshape(-1, 2)
    stile = arr["sub_tile"].reshape(-1, 2)
    pair = arr["pair"].reshape(-1, 4).astype(np.int64)
    shp = arr["out_shape"].reshape(-1, 4)
    ts, ps = arr["tile_start"], arr["pair_start"]
    pss = arr["part_sub_start"]
    cap = int(arr["stage_doubles"])
    seen = 0
    for p in range(int(arr["n_parts"])):
        for s in range(pss[p], pss[p + 1]):
            na = sa[s, 1] - sa[s, 0]
            assert na <= cap
            S = np.full(cap + 4096, np.nan)
            S[:na] = a_data[sa[s, 0]:sa[s, 1]]
            o = arr["sub_out0"][s]
            for t in range(stile[s, 0], stile[s, 1]):
                while ts[o + 1] <= t:
                    o += 1
                rows, cols, ys, _ = shp[o]
                tn = (cols + 7) // 8
                mi, ni = divmod(t - ts[o], tn)
                r0, r1 = 8 * mi, min(rows, 8 * mi + 8)
                c0, c1 = 8 * ni, min(cols, 8 * ni + 8)
                acc = np.zeros((r1 - r0, c1 - c0))
                for q in range(ps[o], ps[o + 1]):
                    x, y, bs, boff = pair[q]
                    a_s, inner = y & 0xFFFF, y >> 16
                    assert 0 <= x and x + (rows - 1) * a_s + inner <= na, "A block outside the stage"
                    am = np.stack([S[x + r * a_s: x + r * a_s + inner] for r in range(r0, r1)])
                    bm = np.stack([b_data[boff + k * bs + c0: boff + k * bs + c1] for k in range(inner)])
                    acc += am @ bm
                for i in range(r0, r1):
                    off = arr["out_off"][o] + i * ys
                    c[off + c0: off + c1] = (c[off + c0: off + c1] if accumulate else 0.0) \
                        + alpha * acc[i - r0]
                seen += 1
    assert seen == ts[-1], "tiles skipped or repeated"
    return c
