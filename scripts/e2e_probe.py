"""Where the end-to-end step time goes (weak G = 1): H2D copy alone, + scatter, + compute."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1907_01005_b200 import problem as P  # noqa: E402
from paper_1907_01005_b200.bcsr import mmult, tmmult  # noqa: E402
from paper_1907_01005_b200.comm import serial_context  # noqa: E402

dev = torch.device("cuda", 0)
prob = P.build_problem(sys.argv[1] if len(sys.argv) > 1 else "weak1")
st = P.make_rank_setup(serial_context(dev), prob, projection=True, device=dev)
st.c.update_ghost_values()
spec = prob.spec_h()
for _ in range(3):
    st.op.apply(spec, st.x, st.hx)
    tmmult(st.x, st.hx, st.s)
    mmult(st.x, st.c, st.xc)
torch.cuda.synchronize()
n_sv = st.x.n_support_values()
NB = 3
host_x = [torch.empty(n_sv, dtype=torch.float64, pin_memory=True) for _ in range(NB)]
for h in host_x:
    h.copy_(st.x.download_support_values().cpu())
host_s = torch.empty(st.s.data.numel(), dtype=torch.float64, pin_memory=True)
xs = [st.x] + [st.x.copy() for _ in range(NB - 1)]
dev_x = [torch.empty(n_sv, dtype=torch.float64, device=dev) for _ in range(NB)]
cstream = torch.cuda.Stream(device=dev)
copied = [torch.cuda.Event() for _ in range(NB)]
consumed = [torch.cuda.Event() for _ in range(NB)]
main = torch.cuda.current_stream(dev)


def issue_copy(k):
    b = k % NB
    with torch.cuda.stream(cstream):
        cstream.wait_event(consumed[b])
        dev_x[b].copy_(host_x[b], non_blocking=True)
        copied[b].record(cstream)


def run(n, upload, compute):
    for b in range(NB):
        consumed[b].record(main)
    for k in range(min(NB - 1, n)):
        issue_copy(k)
    for k in range(n):
        b = k % NB
        main.wait_event(copied[b])
        xk = xs[b]
        if upload:
            xk.upload_support_values(dev_x[b])
        consumed[b].record(main)
        if k + NB - 1 < n:
            issue_copy(k + NB - 1)
        if compute:
            st.op.apply(spec, xk, st.hx)
            tmmult(xk, st.hx, st.s)
            mmult(xk, st.c, st.xc)
            host_s.copy_(st.s.data, non_blocking=True)


for label, up, comp in (("copy only", False, False), ("copy + upload", True, False),
                        ("copy + upload + step", True, True)):
    run(3, up, comp)
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    run(10, up, comp)
    a1.record()
    a1.synchronize()
    print(f"{label}: {a0.elapsed_time(a1) / 10:.2f} ms per step", flush=True)
import time
t = time.perf_counter()
for _ in range(10):
    st.op.apply(spec, st.x, st.hx)
    tmmult(st.x, st.hx, st.s)
    mmult(st.x, st.c, st.xc)
print(f"host time to issue a step: {(time.perf_counter() - t) / 10 * 1e3:.2f} ms")
torch.cuda.synchronize()
