"""Time the K1 kernel alone (CUDA events) on a config; optional BMV_LIB variant.

    python scripts/k1_timing.py q4 [reps]
"""
import ctypes as C
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1907_01005_b200 import _lib  # noqa: E402
from paper_1907_01005_b200 import problem as P  # noqa: E402
from paper_1907_01005_b200.comm import serial_context  # noqa: E402
from paper_1907_01005_b200.matfree import implemented_flops_per_pair  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "q4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
dev = torch.device("cuda", 0)
prob = P.build_problem(name)
st = P.make_rank_setup(serial_context(dev), prob, projection=False, device=dev)
spec = prob.spec_h()
st.op.apply(spec, st.x, st.hx)
plan = st.op.plan_for(st.x, st.hx)
coef, stride = st.op.coefficient(spec, dev)
lib = _lib.load()
s = _lib.stream_handle(dev)


def k1():
    _lib.check(lib.bmv_cellop_apply(plan.handle.raw, 1, _lib.dptr(coef), stride,
                                    _lib.dptr(st.x.data), _lib.dptr(st.hx.data), 0, s))


for _ in range(3):
    k1()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    k1()
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / reps
f = plan.n_pairs * implemented_flops_per_pair(prob.cfg.degree + 1, "hamiltonian", True)
print(json.dumps({"config": name, "lib": os.environ.get("BMV_LIB", "default"), "k1_ms": round(ms, 4),
                  "tflops": round(f / ms / 1e9, 3), "pairs": plan.n_pairs}))
