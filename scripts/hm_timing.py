"""Fused H X + M X (apply_h_and_mass) vs two applies, through the drop-in API.

    python scripts/hm_timing.py weak1 [reps]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1907_01005_b200 import problem as P  # noqa: E402
from paper_1907_01005_b200.bcsr import BlockCsrMatrix  # noqa: E402
from paper_1907_01005_b200.comm import serial_context  # noqa: E402
from paper_1907_01005_b200.matfree import mass_operator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "q4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
dev = torch.device("cuda", 0)
prob = P.build_problem(name)
st = P.make_rank_setup(serial_context(dev), prob, projection=False, device=dev)
mx = BlockCsrMatrix(st.hx.pattern, st.hx.layout, st.hx.ctx, st.hx.lane_width, dev)
spec = prob.spec_h()
out = {"config": name}
for label, fn in (("separate_ms", lambda: (st.op.apply(spec, st.x, st.hx),
                                           st.op.apply(mass_operator(), st.x, mx))),
                  ("fused_ms", lambda: st.op.apply_h_and_mass(spec, st.x, st.hx, mx))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    out[label] = round(e0.elapsed_time(e1) / reps, 4)
print(json.dumps(out))
