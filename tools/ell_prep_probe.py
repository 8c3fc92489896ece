"""ELL,TM preparation cost on a large constant-row matrix (GPU): constant-model Seer plans
with k = 1 and k = 2 (prep = t1 - (t2 - t1)) and the preparation alone captured as a graph."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

from kbench import MATS  # noqa: E402
from paper_2403_17017_b200 import kernels, seer  # noqa: E402

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def med(fn, n=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


for name in (sys.argv[1] if len(sys.argv) > 1 else "const8big,C3").split(","):
    m, dt = MATS[name](torch.device("cuda"))
    A = m.to_device_csr(dt)
    del m
    x = torch.rand(A.n_cols, device="cuda", dtype=dt)
    y = torch.empty(A.n_rows, device="cuda", dtype=dt)
    for k in (kernels.ELL_TM, kernels.COO_WM, kernels.ADAPTIVE_CSR):
        t = {}
        for it in (1, 2):
            p = seer.SeerPlan(seer.fixed_model(k), A, x, y, it)
            t[it] = med(p.launch)
            p.close()
        print(f"{name} {kernels.KERNELS[k]}: plan k=1 {t[1]:.3f} ms, k=2 {t[2]:.3f} ms -> prep {2 * t[1] - t[2]:.3f} ms, "
              f"SpMV {t[2] - t[1]:.3f} ms", flush=True)
