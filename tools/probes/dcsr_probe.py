"""Probe: how much of a column slice's time is its empty rows?  Each C5 column slice as
a full-row CSR vs the same slice with its empty rows removed (compact CSR, compact y --
no scatter), plain CSR,WO per slice.  Upper bound on what compressed-row slices could save.

    python tools/probes/dcsr_probe.py [--slices 2,3,4,6]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools", "probes"))
import torch  # noqa: E402

from colslice_probe import col_slices, timeit  # noqa: E402
from paper_2403_17017_b200 import gen, kernels  # noqa: E402
from paper_2403_17017_b200.device import DeviceCSR  # noqa: E402


def compact(B):
    off = B.row_offsets.to(torch.int64)
    ln = off[1:] - off[:-1]
    keep = torch.nonzero(ln > 0).squeeze(1)
    o = torch.zeros(keep.numel() + 1, dtype=torch.int64, device=off.device)
    torch.cumsum(ln[keep], 0, out=o[1:])
    return DeviceCSR(keep.numel(), B.n_cols, o.to(torch.int32), B.col_indices, B.values), keep.numel()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--slices", default="1,2,3,4,6")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    A = gen.config("C5", device=dev).to_device_csr(torch.float32, device=dev)
    torch.cuda.empty_cache()
    x = torch.rand(A.n_cols, device=dev)
    K = kernels.CSR_WO
    for S in [int(v) for v in a.slices.split(",")]:
        sl = col_slices(A, S) if S > 1 else [A]
        cs = [compact(B) for B in sl]
        ys = [torch.empty(A.n_rows, device=dev) for _ in sl]
        t_full = timeit(lambda: [kernels.spmv(B, x, K, y=yb) for B, yb in zip(sl, ys)])
        t_cmp = timeit(lambda: [kernels.spmv(C, x, K, y=yb) for (C, _), yb in zip(cs, ys)])
        frac = [round(n / A.n_rows, 3) for _, n in cs]
        print(f"S={S}: full-row slices {t_full:7.3f} ms   compact {t_cmp:7.3f} ms   nonempty-row fraction {frac}",
              flush=True)
        del sl, cs, ys
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
