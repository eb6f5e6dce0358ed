"""Per-call device times of the OM energy + gradient step (weak1)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1907_01005_b200 import bcsr as B  # noqa: E402
from paper_1907_01005_b200 import problem as P  # noqa: E402
from paper_1907_01005_b200.comm import serial_context  # noqa: E402
from paper_1907_01005_b200.energy import compute_energy, make_workspace  # noqa: E402
from paper_1907_01005_b200.matfree import mass_operator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "weak1"
dev = torch.device("cuda", 0)
prob = P.build_problem(name)
ctx = serial_context(dev)
st = P.make_rank_setup(ctx, prob, projection=False, device=dev)
ws = make_workspace(ctx, st.op, st.x, prob.loc_layout)
compute_energy(st.op, mass_operator(), prob.spec_h(), st.x, ws)
out = {}


def timed(label, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    out[label] = round(a.elapsed_time(b) / reps, 3)


timed("apply_h_and_mass", lambda: st.op.apply_h_and_mass(prob.spec_h(), st.x, ws.phi_h, ws.phi_m))
timed("tmmult_m", lambda: B.tmmult(st.x, ws.phi_m, ws.mbar))
timed("tmmult_h", lambda: B.tmmult(st.x, ws.phi_h, ws.hbar))
timed("glue_t2", lambda: (B.copy_pattern_subset(ws.t2, ws.mbar), B.scale_add(ws.t2, -1.0),
                          B.add_scaled_identity(ws.t2, 2.0)))
ws.hbar.update_ghost_values()
ws.t2.update_ghost_values()
timed("tr_mult", lambda: B.tr_mult(ws.t2, ws.hbar))
timed("mmult_phi_m_hbar", lambda: B.mmult(ws.phi_m, ws.hbar, ws.g, alpha=-2.0))
timed("mmult_phi_h_t2_acc", lambda: B.mmult(ws.phi_h, ws.t2, ws.g, alpha=2.0, accumulate=True))
timed("tr_tmmult", lambda: B.tr_tmmult(ws.g, ws.g))
print(json.dumps(out))
