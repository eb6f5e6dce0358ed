"""Time K4 (tmmult) and K5 (mmult) alone on a config (CUDA events).

    python scripts/spmm_timing.py q4 [reps]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1907_01005_b200 import problem as P  # noqa: E402
from paper_1907_01005_b200.bcsr import mmult, tmmult  # noqa: E402
from paper_1907_01005_b200.comm import serial_context  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "q4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
dev = torch.device("cuda", 0)
prob = P.build_problem(name)
st = P.make_rank_setup(serial_context(dev), prob, projection=True, device=dev)
st.c.update_ghost_values()
st.op.apply(prob.spec_h(), st.x, st.hx)
out = {"config": name}
for label, fn in (("tmmult", lambda: tmmult(st.x, st.hx, st.s)),
                  ("mmult", lambda: mmult(st.x, st.c, st.xc))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    out[label + "_ms"] = round(e0.elapsed_time(e1) / reps, 4)
out["x_stored_mb"] = round(st.x.data.numel() * 8e-6, 1)
out["hx_stored_mb"] = round(st.hx.data.numel() * 8e-6, 1)
print(json.dumps(out))
