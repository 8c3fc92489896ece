"""Feature pass (K1, kp_gather_features) bandwidth on growing offsets arrays (GPU).
Algorithmic bytes = (R+1) x offset bytes; CUDA events, L2 flushed, median of 10."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2403_17017_b200 import features  # noqa: E402

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
for R in (10_000, 1 << 20, 2_000_000, 16 << 20, 64 << 20, 256 << 20):
    for dt in (torch.int32, torch.int64):
        if dt == torch.int32 and R * 8 >= 2**31:
            continue
        lens = torch.randint(0, 16, (R,), device="cuda", dtype=torch.int64)
        off = torch.zeros(R + 1, dtype=torch.int64, device="cuda")
        torch.cumsum(lens, 0, out=off[1:])
        from types import SimpleNamespace
        A = SimpleNamespace(n_rows=R, n_cols=R, row_offsets=off.to(dt))  # gather_features duck-types these
        out = features.gather_outcome(A)
        ts = []
        for _ in range(12):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            features.gather_outcome(A, out=out)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        t = statistics.median(ts[2:])
        b = (R + 1) * A.row_offsets.element_size()
        print(f"R={R:10d} {str(dt):12s} {t * 1e6:9.1f} us  {b / t / 1e9:8.1f} GB/s  {b / t / 1e9 / peak:5.3f}", flush=True)
        del A, off, lens
