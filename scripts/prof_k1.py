"""Profiling driver: one config's hot path, K1 launched a few times (for ncu).

    python scripts/prof_k1.py q4 [reps]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1907_01005_b200 import problem as P  # noqa: E402
from paper_1907_01005_b200.bcsr import mmult, tmmult  # noqa: E402
from paper_1907_01005_b200.comm import serial_context  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "q4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda", 0)
prob = P.build_problem(name)
st = P.make_rank_setup(serial_context(dev), prob, projection=True, device=dev)
st.c.update_ghost_values()
spec = prob.spec_h()
for _ in range(reps):
    st.op.apply(spec, st.x, st.hx)
    tmmult(st.x, st.hx, st.s)
    mmult(st.x, st.c, st.xc)
torch.cuda.synchronize()
print("done", name, reps)
