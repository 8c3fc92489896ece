import os, sys, time, statistics
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from paper_2403_17017_b200 import gen, seer
from paper_2403_17017_b200.device import DeviceCSR
A = gen.config("C2", device="cuda").to_device_csr(torch.float32)
x = torch.rand(A.n_cols, device="cuda")
model = seer.SeerModel.load(os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"), "paper_2403_17017_b200/models/seer_b200.json"))
h = [t.cpu().pin_memory() for t in (A.row_offsets, A.col_indices, A.values, x)]
def run(nsets, d2h=True, steps=12):
    sets = []
    for _ in range(nsets):
        d = [torch.empty_like(t, device="cuda") for t in h] + [torch.empty(A.n_rows, device="cuda")]
        B = DeviceCSR(A.n_rows, A.n_cols, d[0], d[1], d[2])
        sets.append((d, seer.SeerPlan(model, B, d[3], d[4], 1)))
    hy = [torch.empty(A.n_rows, pin_memory=True) for _ in range(nsets)]
    copy = torch.cuda.Stream(); comp = torch.cuda.current_stream()
    freed = [torch.cuda.Event() for _ in range(nsets)]
    for e in freed: e.record(comp)
    def step(i):
        s = i % nsets
        d, plan = sets[s]
        copy.wait_event(freed[s])
        with torch.cuda.stream(copy):
            for a, b in zip(d[:4], h): a.copy_(b, non_blocking=True)
            ev = torch.cuda.Event(); ev.record(copy)
        comp.wait_event(ev)
        plan.launch(comp)
        if d2h: hy[s].copy_(d[4], non_blocking=True)
        freed[s].record(comp)
    for i in range(3): step(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp); copy.wait_event(e0)
    for i in range(steps): step(i)
    comp.wait_stream(copy); e1.record(comp); e1.synchronize()
    return e0.elapsed_time(e1) / steps
for ns in (1, 2, 3):
    for d2h in (True, False):
        print(ns, d2h, round(run(ns, d2h), 3), "ms/step", flush=True)
