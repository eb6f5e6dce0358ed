"""Zeroing bandwidth: bmv_zero (our kernel) vs torch zero_ (fill kernel) vs cudaMemsetAsync."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1907_01005_b200 import _lib  # noqa: E402

n = 3_607_220_224 // 8
t = torch.empty(n, dtype=torch.float64, device="cuda")
lib = _lib.load()
cudart = C.CDLL("libcudart.so") if False else None
st = _lib.stream_handle(t.device)


def run(label, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / reps
    print(f"{label}: {ms:.3f} ms, {n * 8 / ms / 1e6:.0f} GB/s")


run("bmv_zero", lambda: _lib.check(lib.bmv_zero(_lib.dptr(t), n, st)))
run("torch.zero_", lambda: t.zero_())
