"""Decompose the gathered-path plan overhead on one matrix (GPU): forced-gathered plan
(K15g feature pass + tree + device SWITCH -> body) vs the body alone as a graph vs the
feature kernel alone.  CUDA events, L2 flushed, median of N."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2403_17017_b200 import features, gen, kernels, seer  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
N = 30
A = gen.config(name, device="cuda").to_device_csr(torch.float64 if name == "C4" else torch.float32)
x = torch.rand(A.n_cols, device="cuda", dtype=A.values.dtype)
y = torch.empty(A.n_rows, device="cuda", dtype=A.values.dtype)
model = seer.SeerModel.load(os.path.join(ROOT, "paper_2403_17017_b200", "models", "seer_b200.json"))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
plan = seer.SeerPlan(model, A, x, y, 1, force_gathered=True)
plan.launch()
torch.cuda.synchronize()
kern = int(plan.outcome().kernel)


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


def body():
    P = kernels.prepare(A, kern, cache=False) if kern in kernels.NEEDS_PREP else None
    kernels.spmv(A, x, kern, y=y, prepared=P)


body()
cs = torch.cuda.Stream()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=cs):
    body()
out = torch.empty(96, dtype=torch.uint8, device="cuda")
gf = torch.cuda.CUDAGraph()
with torch.cuda.graph(gf, stream=cs):
    features.gather_outcome(A, out=out)
print(f"{name}: kernel {kernels.KERNELS[kern]}")
print(f"  gathered plan (feature pass + tree + SWITCH + body): {med(plan.launch):8.2f} us")
print(f"  body alone (graph):                                   {med(g.replay):8.2f} us")
print(f"  feature kernel alone (graph):                         {med(gf.replay):8.2f} us")
print(f"  empty graph-ish reference (tiny zero_):               {med(lambda: y[:1].zero_()):8.2f} us")
