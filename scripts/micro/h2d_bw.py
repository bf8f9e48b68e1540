"""Pinned host -> device copy bandwidth with 1, 2 and 4 concurrent streams (debug aid)."""
import torch
n = 598 * 20000 * 72
h = torch.empty(n, dtype=torch.float32).pin_memory()
h.uniform_()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    parts = torch.chunk(torch.arange(n), ns)
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s, p in zip(streams, torch.chunk(h, ns)):
            pass
        off = 0
        chunks = torch.chunk(h, 8 * ns)
        for i, c in enumerate(chunks):
            s = streams[i % ns]
            s.wait_event(e0) if i < ns else None
            with torch.cuda.stream(s):
                d[off:off + c.numel()].copy_(c, non_blocking=True)
            off += c.numel()
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"streams {ns}: {ms:.2f} ms  {n * 4 / ms / 1e6:.1f} GB/s")
