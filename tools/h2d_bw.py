"""Pinned host -> device bandwidth with 1, 2 and 4 concurrent copy streams (1.89 GB total)."""
import torch
n = 18
src = [torch.empty(26_214_400, dtype=torch.float32).pin_memory() for _ in range(n)]   # 18 x 105 MB
dst = [torch.empty_like(s, device="cuda") for s in src]
for ns in (1, 2, 3, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(3):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(n):
            s = streams[i % ns]
            s.wait_event(a)
            with torch.cuda.stream(s):
                dst[i].copy_(src[i], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b)
    print(f"{ns} streams: {sum(x.numel()*4 for x in src)/ms/1e6:.1f} GB/s ({ms:.1f} ms)", flush=True)
