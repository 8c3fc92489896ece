"""Launch-path check (GPU): the same fixed kernel's prep + k SpMVs timed as a torch-captured
CUDA graph (torch.cuda.graph + replay) and as a kp_seer_plan built from a constant model
(known path -> the kernel's body), CUDA events, L2 flushed, median of N.  Any gap is launch
machinery, not kernel time, and must not leak into Seer-vs-fixed comparisons.

    python tools/graph_launch_probe.py [C1,u1m,C2] [kernels 1,3,4,5]
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

from kbench import MATS  # noqa: E402
from paper_2403_17017_b200 import kernels, seer  # noqa: E402

mats = (sys.argv[1] if len(sys.argv) > 1 else "C1,u1m,C2").split(",")
ks = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "1,3,4,5").split(",")]
N = 30
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def med(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(N):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


for name in mats:
    m, dt = MATS[name](torch.device("cuda"))
    A = m.to_device_csr(dt)
    x = torch.rand(A.n_cols, device="cuda", dtype=dt)
    y = torch.empty(A.n_rows, device="cuda", dtype=dt)
    for k in ks:
        def body():
            P = kernels.prepare(A, k, cache=False) if k in kernels.NEEDS_PREP else None
            kernels.spmv(A, x, k, y=y, prepared=P)
        body()
        cs = torch.cuda.Stream()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cs):
            body()
        t_torch = med(g.replay)
        plan = seer.SeerPlan(seer.fixed_model(k), A, x, y, 1)
        t_plan = med(plan.launch)
        plan.close()
        print(json.dumps({"matrix": name, "kernel": kernels.KERNELS[k], "torch_graph_us": round(t_torch, 2),
                          "kp_plan_us": round(t_plan, 2)}), flush=True)
