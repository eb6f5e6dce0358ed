"""Time the OM energy + gradient step (compute_energy + compute_gradient +
directional_derivative) through the drop-in API on a config.

    python scripts/energy_timing.py weak1 [reps]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_1907_01005_b200 import problem as P  # noqa: E402
from paper_1907_01005_b200.comm import serial_context  # noqa: E402
from paper_1907_01005_b200.energy import (compute_energy, compute_gradient,  # noqa: E402
                                          directional_derivative, make_workspace)
from paper_1907_01005_b200.matfree import mass_operator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "q4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device("cuda", 0)
prob = P.build_problem(name)
ctx = serial_context(dev)
st = P.make_rank_setup(ctx, prob, projection=False, device=dev)
t0 = time.time()
ws = make_workspace(ctx, st.op, st.x, prob.loc_layout)


def step():
    e = compute_energy(st.op, mass_operator(), prob.spec_h(), st.x, ws)
    g = compute_gradient(ws)
    return e, directional_derivative(g, g)


e, s = step()
torch.cuda.synchronize()
setup = time.time() - t0
t0 = time.time()
for _ in range(reps):
    e, s = step()
torch.cuda.synchronize()
print(json.dumps({"config": name, "energy": e, "slope": s, "ms_per_step": round((time.time() - t0) / reps * 1e3, 3),
                  "first_step_incl_setup_s": round(setup, 1)}))
