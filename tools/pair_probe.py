"""Paired-timing sanity check (GPU): two plans running the SAME kernel on C1, alternated
sample by sample like bench.py's paired ratio -- must read 1.00 -- and the Seer plan vs the
constant-model plan of its own pick."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2403_17017_b200 import gen, kernels, seer  # noqa: E402

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def one(fn):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e3


def paired(fa, fb, n=400):
    fa(); fb(); torch.cuda.synchronize()
    ta, tb = [], []
    for _ in range(n):
        ta.append(one(fa))
        tb.append(one(fb))
    return statistics.mean(ta), statistics.mean(tb)


A = gen.config("C1", device="cuda").to_device_csr(torch.float32)
x = torch.rand(A.n_cols, device="cuda")
y = torch.empty(A.n_rows, device="cuda")
model = seer.SeerModel.load(os.path.join(ROOT, "paper_2403_17017_b200", "models", "seer_b200.json"))
sp = seer.SeerPlan(model, A, x, y, 1)
sp.launch(); torch.cuda.synchronize()
kk = int(sp.outcome().kernel)
f1 = seer.SeerPlan(seer.fixed_model(kk), A, x, y, 1)
f2 = seer.SeerPlan(seer.fixed_model(kk), A, x, y, 1)
print("kernel", kernels.KERNELS[kk], sp.select_kind(), f1.select_kind())
if "--bench-like" in sys.argv:  # what bench.measure does between building the Seer plan and pairing
    for _ in range(5):
        kernels.spmv(A, x, kk, y=y)
    for k2 in range(len(kernels.KERNELS)):
        fp = seer.SeerPlan(seer.fixed_model(k2), A, x, y, 1)
        for _ in range(5):
            fp.launch()
        torch.cuda.synchronize()
        fp.close()
    f2.close()
    f2 = seer.SeerPlan(seer.fixed_model(kk), A, x, y, 1)
for name, a, b in (("fixed vs fixed", f1.launch, f2.launch), ("seer vs fixed", sp.launch, f1.launch),
                   ("fixed vs seer", f1.launch, sp.launch), ("seer vs seer", sp.launch, sp.launch)):
    ma, mb = paired(a, b)
    print(f"{name:15s} {ma:7.2f} {mb:7.2f} ratio b/a {mb / ma:.3f}", flush=True)
