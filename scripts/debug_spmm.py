"""Debug: K4 / K5 on the many-columns test shape; prints where S and X C differ."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from _helpers import Small  # noqa: E402
from paper_1907_01005_b200.bcsr import mmult, tmmult  # noqa: E402
from paper_1907_01005_b200.comm import serial_context  # noqa: E402
from paper_1907_01005_b200.problem import hashed_entries  # noqa: E402

cuda = torch.device("cuda", 0)
centers = np.asarray([[1.0, 1.0, 1.0], [3.0, 3.0, 2.0], [2.0, 1.5, 3.0], [0.5, 3.2, 0.7],
                      [2.5, 2.5, 0.5], [1.5, 3.5, 2.5]])
s = Small((4, 4, 4), (1.0, 1.0, 1.0), 1, 2, centers, 3.5, 8, 8)
ctx = serial_context(cuda)
rl, _, x, hx = s.operands(ctx, cuda)
s.fill(x, 5, attach=False)
hx.fill_owned_entries(lambda r, c: hashed_entries(9, r, c))
sm, cm, xc = s.projection_operands(ctx, cuda, rl)
tmmult(x, hx, sm)
mmult(x, cm, xc, alpha=0.75, accumulate=False)
xd, hd, cd = x.to_dense_owned(), hx.to_dense_owned(), cm.to_dense_owned()
want = xd.T @ hd
got = sm.to_dense_owned()
bad = np.abs(got - want) > 1e-9 * np.abs(want).max()
print("S bad entries", int(bad.sum()), "of", bad.size)
print("bad rows", np.flatnonzero(bad.any(axis=1)))
print("bad cols", np.flatnonzero(bad.any(axis=0)))
r, c = np.argwhere(bad)[0] if bad.any() else (0, 0)
print("first bad", r, c, got[r, c], want[r, c], got[r, c] - want[r, c])
wy = 0.75 * (xd @ cd)
gy = xc.to_dense_owned()
stored = np.zeros_like(gy, dtype=bool)
_, grow, gcol = xc._valid_owned_index()
stored[grow, gcol] = True
by = stored & (np.abs(gy - wy) > 1e-9 * np.abs(wy).max())
print("XC bad", int(by.sum()), "rows", np.flatnonzero(by.any(axis=1))[:20], "cols",
      np.flatnonzero(by.any(axis=0)))
from paper_1907_01005_b200 import spmm  # noqa: E402
plan = spmm.tmmult_plan(x, hx, sm)
a = plan.arrays
print("K4 chunks", a["n_chunks"], "stage", a["stage_bytes"])
m = a["meta"]
for j in range(min(int(a["n_chunks"]), 6)):
    m0 = int(a["chunk_meta"][j])
    print(" chunk", j, "hdr", m[m0:m0 + 16].tolist(), "meta words", int(a["chunk_meta"][j + 1]) - m0,
          "a", a["chunk_a"][2 * j:2 * j + 2].tolist(), "b", a["chunk_b"][2 * j:2 * j + 2].tolist())
