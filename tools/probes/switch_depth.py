"""Gathered-path plan cost vs the same body as a plain graph, as a function of k (GPU).

    python tools/probes/switch_depth.py [matrix] [k,k,...]

For each k: the forced-gathered Seer plan (feature pass + tree + device SWITCH -> body of
prep + k SpMVs) against the body captured as an ordinary graph.  A difference that grows
with k is a per-node cost of kernels inside the conditional body; a constant one is the
selection + SWITCH overhead.  CUDA events, L2 flushed before each launch, median of N."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

from kbench import MATS  # noqa: E402
from paper_2403_17017_b200 import kernels, seer  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "band27"
ks = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "1,10,100").split(",")]
dev = torch.device("cuda", 0)
m, dt = MATS[name](dev)
A = m.to_device_csr(dt, device=dev)
x = (torch.rand(A.n_cols, device=dev, dtype=torch.float64) * 2 - 1).to(dt)
y = torch.empty(A.n_rows, device=dev, dtype=dt)
model = seer.SeerModel.load(os.path.join(ROOT, "paper_2403_17017_b200", "models", "seer_b200.json"))
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def med(fn, n=7):
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
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


for k in ks:
    plan = seer.SeerPlan(model, A, x, y, k, force_gathered=True)
    plan.launch()
    torch.cuda.synchronize()
    kern = int(plan.outcome().kernel)

    def body(kern=kern, k=k):
        P = kernels.prepare(A, kern, cache=False) if kern in kernels.NEEDS_PREP else None
        for _ in range(k):
            kernels.spmv(A, x, kern, y=y, prepared=P)

    body()
    cs = torch.cuda.Stream()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs):
        body()
    tp, tb = med(plan.launch), med(g.replay)
    print(f"{name} k={k:4d} {kernels.KERNELS[kern]:12s} plan {tp:10.2f} us  body graph {tb:10.2f} us  "
          f"diff {tp - tb:8.2f} us  ({(tp - tb) / k:6.2f} us per iteration)", flush=True)
    plan.close()
    del g
