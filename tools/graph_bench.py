"""Per-kernel cost inside a CUDA graph (the way kp_seer_plan runs it), for A/B tests of
small-matrix latency where single eager launches are quantised by launch overhead.

    python tools/graph_bench.py [--mats C1,u1m] [--kernels 4] [--n 20] [--reps 20]

Prints, per (matrix, kernel): t1 = one SpMV as a graph (L2 flushed before the launch) and
the marginal per-iteration cost (t_n - t_1) / (n - 1) of an n-SpMV graph (warm L2).
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

from kbench import MATS  # noqa: E402
from paper_2403_17017_b200 import kernels  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mats", default="C1,u1m,rmat15,st43")
    ap.add_argument("--kernels", default="2,3,4,5")
    ap.add_argument("--n", type=int, default=20)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for name in a.mats.split(","):
        m, dt = MATS[name](dev)
        A = m.to_device_csr(dt, device=dev)
        x = (torch.rand(A.n_cols, device=dev, dtype=torch.float64) * 2 - 1).to(dt)
        y = torch.empty(A.n_rows, device=dev, dtype=dt)
        for k in [int(v) for v in a.kernels.split(",")]:
            P = kernels.prepare(A, k, cache=False) if k in kernels.NEEDS_PREP else None
            kernels.spmv(A, x, k, y=y, prepared=P)

            def gtime(n):
                cs = torch.cuda.Stream()
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cs):
                    for _ in range(n):
                        kernels.spmv(A, x, k, y=y, prepared=P)
                g.replay()
                torch.cuda.synchronize()
                ts = []
                for _ in range(a.reps):
                    flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    g.replay()
                    e1.record()
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e3)
                return statistics.median(ts)

            t1, tn = gtime(1), gtime(a.n)
            print(f"{name:8s} {kernels.KERNELS[k]:13s} t1 {t1:9.2f} us   per-iter {(tn - t1) / (a.n - 1):9.2f} us",
                  flush=True)


if __name__ == "__main__":
    main()
