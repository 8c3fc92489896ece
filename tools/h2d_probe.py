"""Host->device copy bandwidth from pinned memory with 1/2/4 concurrent streams (GPU)."""
import torch
n = 137_067_452
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = (n + ns - 1) // ns
    for rep in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        e1.synchronize()
        if rep == 3:
            t = e0.elapsed_time(e1) * 1e-3
            print(f"{ns} streams: {n / t / 1e9:.1f} GB/s ({t * 1e3:.3f} ms)")
