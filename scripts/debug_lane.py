"""Debug: lane K4/K5 on the GPU vs the CPU emulation of the same plan vs the
deterministic kernels.  python scripts/debug_lane.py smoke"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from _plan_emul import emulate_mmult_lane, emulate_tmmult_lane  # noqa: E402
from paper_1907_01005_b200 import bcsr as B  # noqa: E402
from paper_1907_01005_b200 import problem as P  # noqa: E402
from paper_1907_01005_b200.comm import serial_context  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "smoke"
dev = torch.device("cuda", 0)
prob = P.build_problem(name)
st = P.make_rank_setup(serial_context(dev), prob, projection=True, device=dev)
st.op.apply(prob.spec_h(), st.x, st.hx)
st.c.update_ghost_values()
torch.cuda.synchronize()
os.environ["BMV_DETERMINISTIC"] = "0"
B.tmmult(st.x, st.hx, st.s)
torch.cuda.synchronize()
s_lane = st.s.data.cpu().numpy().copy()
os.environ["BMV_DETERMINISTIC"] = "1"
B.tmmult(st.x, st.hx, st.s)
torch.cuda.synchronize()
s_det = st.s.data.cpu().numpy().copy()
d, keep = B.tmmult_lane_desc(st.x, st.hx, st.s)
arr = B.lane_plan_host(4, d, torch.cuda.get_device_properties(0).multi_processor_count)
if st.x.data.numel() < 5e7:
    s_emu = emulate_tmmult_lane(arr, st.x.data.cpu().numpy(), st.hx.data.cpu().numpy(), st.s.data.numel())
    print("S emu vs det", np.abs(s_emu - s_det).max(), "scale", np.abs(s_det).max())
print("S lane vs det", np.abs(s_lane - s_det).max(), "scale", np.abs(s_det).max())
bad = np.flatnonzero(np.abs(s_lane - s_det) > 1e-9 * np.abs(s_det).max())
print("bad entries", bad.size, bad[:20], s_lane[bad[:5]], s_det[bad[:5]])
print("chunks", len(arr["copies"]), "parts", arr["n_parts"], "stage", arr["stage_bytes"])
os.environ["BMV_DETERMINISTIC"] = "0"
B.mmult(st.x, st.c, st.xc)
torch.cuda.synchronize()
y_lane = st.xc.data.cpu().numpy().copy()
os.environ["BMV_DETERMINISTIC"] = "1"
B.mmult(st.x, st.c, st.xc)
torch.cuda.synchronize()
y_det = st.xc.data.cpu().numpy().copy()
print("Y lane vs det", np.abs(y_lane - y_det).max(), "scale", np.abs(y_det).max())
