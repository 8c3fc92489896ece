"""Probe: does column blocking (S column slices of the matrix, x-slice resident in L2)
cut C5's gather traffic?  Times the full-matrix merge SpMV against the sum of S sliced
SpMVs (separate y per slice, no accumulation) on the same matrix, fp32.

    python tools/probes/colslice_probe.py [--scale 26] [--slices 1,2,3,4,6,8]
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2403_17017_b200 import gen, kernels  # noqa: E402
from paper_2403_17017_b200.device import DeviceCSR  # noqa: E402


def col_slices(A, S):
    off = A.row_offsets.to(torch.int64)
    R, C = A.n_rows, A.n_cols
    bounds = [(C * s) // S for s in range(S + 1)]
    out = []
    for s in range(S):
        m = (A.col_indices >= bounds[s]) & (A.col_indices < bounds[s + 1])
        idx = torch.nonzero(m).squeeze(1)
        del m
        rows = torch.searchsorted(off, idx, right=True) - 1
        cnt = torch.bincount(rows, minlength=R)
        del rows
        o = torch.zeros(R + 1, dtype=torch.int64, device=A.device)
        torch.cumsum(cnt, 0, out=o[1:])
        out.append(DeviceCSR(R, C, o.to(torch.int32), A.col_indices[idx], A.values[idx]))
        del idx, cnt, o
    return out


def timeit(fn, reps=7):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--slices", default="1,2,3,4,6,8")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    m = gen.rmat(a.scale, 16, seed=42, device=dev, values="stochastic") if a.scale != 26 else gen.config("C5", device=dev)
    A = m.to_device_csr(torch.float32, device=dev)
    del m
    torch.cuda.empty_cache()
    x = torch.rand(A.n_cols, device=dev)
    y = torch.empty(A.n_rows, device=dev)
    print(f"rows {A.n_rows} cols {A.n_cols} nnz {A.nnz}", flush=True)
    for K in (kernels.CSR_WO, kernels.CSR_MP):
        P = kernels.prepare(A, K, cache=False) if K in kernels.NEEDS_PREP else None
        t = timeit(lambda: kernels.spmv(A, x, K, y=y, prepared=P))
        print(f"{kernels.KERNELS[K]:8s} S=1 full  {t:8.3f} ms", flush=True)
        ref = y.double().clone()
        del P
        for S in [int(v) for v in a.slices.split(",") if int(v) > 1]:
            sl = col_slices(A, S)
            Ps = [kernels.prepare(B, K, cache=False) if K in kernels.NEEDS_PREP else None for B in sl]
            ys = [torch.empty(A.n_rows, device=dev) for _ in sl]

            def run():
                for B, Pb, yb in zip(sl, Ps, ys):
                    kernels.spmv(B, x, K, y=yb, prepared=Pb)
            t = timeit(run)
            acc = torch.empty(A.n_rows, device=dev)
            dst = [torch.empty(A.n_rows, device=dev)]

            def run_b(use_acc):
                for i, (B, Pb) in enumerate(zip(sl, Ps)):
                    last = i == len(sl) - 1
                    kernels.spmv_bcast(B, x, K, dst if last else [acc], 0, prepared=Pb,
                                       acc=acc if (use_acc and i) else None)
            tb = timeit(lambda: run_b(False))
            ta = timeit(lambda: run_b(True))
            print(f"   bcast-kernel sliced no-acc {tb:8.3f} ms   with acc {ta:8.3f} ms", flush=True)
            if S == 3:
                full_b = timeit(lambda: kernels.spmv_bcast(A, x, K, dst, 0))
                print(f"   bcast-kernel full {full_b:8.3f} ms", flush=True)
            tot = sum(yb.double() for yb in ys)
            err = float(((tot - ref).abs() / (ref.abs() + 1e-30)).max())
            per = [round(timeit(lambda B=B, Pb=Pb, yb=yb: kernels.spmv(B, x, K, y=yb, prepared=Pb), 3), 3)
                   for B, Pb, yb in zip(sl, Ps, ys)]
            print(f"{kernels.KERNELS[K]:8s} S={S} sliced {t:8.3f} ms  (+ sum of {S} y: not timed)  per-slice {per}"
                  f"  nnz {[B.nnz for B in sl]}  max rel diff {err:.2e}", flush=True)
            del sl, Ps, ys, tot
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
