"""Where the Seer step's time goes on one matrix (GPU): selection kernel alone, the
whole-pipeline graph (kp_seer_plan), the chosen kernel's prep+SpMV eager and as a plain
captured graph.  CUDA events, L2 flushed before each sample, median of N.

    python tools/plan_overhead.py [C2] [N]
"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2403_17017_b200 import gen, kernels, seer  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
dt = torch.float64 if name == "C4" else torch.float32
A = gen.config(name, device="cuda").to_device_csr(dt)
model = seer.SeerModel.load(os.path.join(ROOT, "paper_2403_17017_b200", "models", "seer_b200.json"))
x = (torch.rand(A.n_cols, device="cuda", dtype=torch.float64) * 2 - 1).to(dt)
y = torch.empty(A.n_rows, device="cuda", dtype=dt)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
k = 1
plan = seer.SeerPlan(model, A, x, y, k)
plan.launch()
torch.cuda.synchronize()
kern = int(plan.outcome().kernel)
print(f"{name}: seer -> {kernels.KERNELS[kern]} path={'gathered' if plan.outcome().path else 'known'}")
out = torch.empty(96, dtype=torch.uint8, device="cuda")


def fixed():
    P = kernels.prepare(A, kern, cache=False) if kern in kernels.NEEDS_PREP else None
    kernels.spmv(A, x, kern, y=y, prepared=P)


fixed()
s = torch.cuda.Stream()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    fixed()
torch.cuda.synchronize()


def t(fn):
    for _ in range(3):
        fn()
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


res = {
    "select kernel (known/gathered path)": t(lambda: seer.select_async(model, A, k, out=out)),
    "seer plan graph (select + switch + body)": t(plan.launch),
    "fixed kernel eager (prep + spmv)": t(fixed),
    "fixed kernel plain graph": t(g.replay),
    "spmv only": t(lambda: kernels.spmv(A, x, kern, y=y, prepared=kernels.prepare(A, kern) if kern in kernels.NEEDS_PREP else None)),
}
for kk, v in res.items():
    print(f"  {kk:45s} {v:9.2f} us")
