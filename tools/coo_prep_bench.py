import sys, os, statistics
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from paper_2403_17017_b200 import gen, kernels
for name in ("C2", "C3", "band4"):
    m = gen.config(name, device="cuda") if name != "band4" else gen.banded(32_000_000, 4, device="cuda")
    A = m.to_device_csr(torch.float32); del m
    P = kernels.prepare(A, kernels.COO_WM, cache=False)
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); P = kernels.prepare(A, kernels.COO_WM, cache=False); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(name, "COO prep us", round(statistics.median(ts[2:]), 1), flush=True)
