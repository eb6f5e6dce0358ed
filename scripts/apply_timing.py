"""Time CellOperator.apply (zero + K1 through the drop-in API) on a config.

    python scripts/apply_timing.py weak1 [reps]
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1907_01005_b200 import problem as P  # noqa: E402
from paper_1907_01005_b200.comm import serial_context  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "q4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
dev = torch.device("cuda", 0)
prob = P.build_problem(name)
st = P.make_rank_setup(serial_context(dev), prob, projection=False, device=dev)
spec = prob.spec_h()
for _ in range(3):
    st.op.apply(spec, st.x, st.hx)
torch.cuda.synchronize()
ref = st.hx.data.clone()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    st.op.apply(spec, st.x, st.hx)
e1.record()
e1.synchronize()
diff = float((st.hx.data - ref).abs().max())
print(json.dumps({"config": name, "fused_zero": os.environ.get("BMV_K1_FUSED_ZERO", "1"),
                  "apply_ms": round(e0.elapsed_time(e1) / reps, 4), "rerun_max_diff": diff}))
