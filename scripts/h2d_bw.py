"""Pinned host -> device copy bandwidth with 1, 2 and 4 concurrent streams."""
import torch

n = 542_040_064 // 8
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    parts = torch.tensor_split(torch.arange(n), ns)
    bounds = [(int(p[0]), int(p[-1]) + 1) for p in parts]
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s, (a, b) in zip(streams, bounds):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[a:b].copy_(h[a:b], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        e1.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"streams={ns}: {n * 8 / ms / 1e6:.1f} GB/s ({ms:.2f} ms)")
