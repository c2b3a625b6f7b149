"""Host->device upload rate of C3's per-step gradients (8 x 102 MB pinned fp32)
with 1, 2 or 4 copy streams."""
import torch

D, M = 25_600_000, 8
host = [torch.empty(D, dtype=torch.float32, pin_memory=True) for _ in range(M)]
dev = [torch.empty(D, dtype=torch.float32, device="cuda") for _ in range(M)]
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for s in streams:
            s.wait_event(a)
        evs = []
        for w in range(M):
            s = streams[w % ns]
            with torch.cuda.stream(s):
                dev[w].copy_(host[w], non_blocking=True)
        for s in streams:
            e = torch.cuda.Event()
            e.record(s)
            torch.cuda.current_stream().wait_event(e)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
    print(f"{ns} stream(s): {ms:.2f} ms, {M * D * 4 / ms / 1e6:.1f} GB/s")
