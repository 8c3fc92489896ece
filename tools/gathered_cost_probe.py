"""Realised gathered-path overhead (GPU): the Seer plan of a model whose selector is a
USE_GATHERED leaf and whose gathered tree is a `kernel` leaf (selection kernel: feature pass
+ tree + cudaGraphSetConditional, then the SWITCH body) minus the same kernel's
constant-model plan (the body alone), both kp plans, L2 flushed, mean of N.  Also the
selection graph without the body (a SWITCH whose bodies are empty is not expressible, so
the feature pass alone as kp_gather_features in a graph is shown for scale)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

from kbench import MATS  # noqa: E402
from paper_2403_17017_b200 import dtree, kernels, seer  # noqa: E402

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def mean_t(fn, n=200):
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
    return statistics.mean(ts)


kern = int(sys.argv[2]) if len(sys.argv) > 2 else kernels.CSR_TM
for name in (sys.argv[1] if len(sys.argv) > 1 else "C1,u1m,C2,C3").split(","):
    m, dt = MATS[name](torch.device("cuda"))
    A = m.to_device_csr(dt)
    del m
    x = torch.rand(A.n_cols, device="cuda", dtype=dt)
    y = torch.empty(A.n_rows, device="cuda", dtype=dt)
    gm = seer.SeerModel(dtree.leaf_tree(kern, 8, 4), dtree.leaf_tree(kern, 8, 8), dtree.leaf_tree(seer.USE_GATHERED, 2, 4))
    pg = seer.SeerPlan(gm, A, x, y, 1)
    pb = seer.SeerPlan(seer.fixed_model(kern), A, x, y, 1)
    tg, tb = mean_t(pg.launch), mean_t(pb.launch)
    pg.close()
    pb.close()
    print(f"{name:6s} rows {A.n_rows:9d} {kernels.KERNELS[kern]}: gathered plan {tg:8.2f} us, body plan {tb:8.2f} us, "
          f"overhead {tg - tb:6.2f} us", flush=True)
