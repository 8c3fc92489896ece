"""csr_from_coo (sparse.py:87-103): device kp_csr_from_coo vs the reference's host
algorithm on the same triples (GPU box).

    python tools/coo_bench.py [--scale 20] [--ef 16] [--reps 5]

Triples: R-MAT-free uniform (row, col) draws on a 2^scale square with ~4% forced duplicate
runs (counter hash, device-generated), fp64 values.  Device time: CUDA events around the
whole public call (keys, radix passes, run sums, offsets; the workspace allocation excluded),
median of reps.  Algorithmic bytes = n*24 (int64 row, int64 col, f64 val in) + (R+1)*8 +
nnz*(4+8) (CSR out).  Host: the reference algorithm (np.lexsort + np.add.reduceat +
bincount, oracle.csr_from_coo == kernelpick.sparse.csr_from_coo) on 1 core, best of 2.
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_17017_b200 import _lib, device, gen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--ef", type=int, default=16)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-host", action="store_true")
    a = ap.parse_args()
    n_side = 1 << a.scale
    n = n_side * a.ef
    e = torch.arange(n, dtype=torch.int64, device="cuda")
    rows = gen.randint(42, 2 * e, n_side)
    cols = gen.randint(42, 2 * e + 1, n_side)
    k = n // 25
    rows[:k] = rows[k:2 * k]
    cols[:k] = cols[k:2 * k]
    vals = gen.uniform01(43, e) * 2 - 1
    del e
    A = device.csr_from_coo(n_side, n_side, rows, cols, vals)  # warm-up (+ module load)
    nnz = A.nnz
    del A
    ts = []
    L0 = _lib.load().kp_launch_count()
    for _ in range(a.reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        A = device.csr_from_coo(n_side, n_side, rows, cols, vals)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
        del A
    launches = (_lib.load().kp_launch_count() - L0) // a.reps
    t = statistics.median(ts)
    algo = n * 24 + (n_side + 1) * 8 + nnz * 12
    out = {"op": "csr_from_coo", "n_triples": n, "shape": [n_side, n_side], "nnz": nnz, "device_ms": round(t * 1e3, 3),
           "device_gbs_algorithmic": round(algo / t / 1e9, 1), "launches_per_call": int(launches),
           "note": "device time includes the D2H read of (nnz, invalid) and the output allocation"}
    if not a.no_host:
        from oracle import oracle as orc
        r, c, v = rows.cpu().numpy(), cols.cpu().numpy(), vals.cpu().numpy()
        best = None
        for _ in range(2):
            t0 = time.perf_counter()
            orc.csr_from_coo(n_side, n_side, r, c, v)
            el = time.perf_counter() - t0
            best = el if best is None else min(best, el)
        out.update({"host_reference_ms": round(best * 1e3, 1), "host_cores": 1,
                    "speedup_vs_host_reference": round(best / t, 1)})
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
