"""Per-kernel SpMV bandwidth on favourable and config inputs (GPU).

    python tools/kbench.py [--mats C2,C3,C4,band27,band4,band2k,pl] [--reps 10] [--out f.json]

For every (matrix, kernel): preprocessing once (timed separately), then `reps` SpMVs
each bracketed by CUDA events with a 512 MB L2 flush in between.  GB/s uses the
kernel's own compulsory byte model; frac is against MEASURED_PEAKS hbm_gbs.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2403_17017_b200 import gen, kernels  # noqa: E402

MATS = {
    "C1": lambda d: (gen.config("C1", device=d), torch.float32),
    "C2": lambda d: (gen.config("C2", device=d), torch.float32),
    "C3": lambda d: (gen.config("C3", device=d), torch.float32),
    "C4": lambda d: (gen.config("C4", device=d), torch.float64),
    "band27": lambda d: (gen.banded(4_000_000, 27, device=d), torch.float32),
    "band4": lambda d: (gen.banded(32_000_000, 4, device=d), torch.float32),
    "band2k": lambda d: (gen.banded(65_536, 2048, device=d), torch.float32),
    "pl": lambda d: (gen.powerlaw_rows(4_000_000, 16.0, 1.5, device=d), torch.float32),
    "const32": lambda d: (gen.constant_rows(4_000_000, 32, device=d), torch.float32),
    "C5": lambda d: (gen.config("C5", device=d), torch.float32),
    # small / medium inputs: latency (launches, searches, fix-ups) dominates
    "u1m": lambda d: (gen.uniform_random(500_000, 500_000, 1_000_000, seed=5, device=d), torch.float32),
    "rmat15": lambda d: (gen.rmat(15, 16, device=d), torch.float32),
    "st43": lambda d: (gen.stencil27(43, device=d), torch.float32),
    # round-2 pitfall cases: a dense band, a medium-width band, a road network
    "dband": lambda d: (gen.banded(8192, 8192, device=d), torch.float32),
    "band300": lambda d: (gen.banded(6641, 307, device=d), torch.float32),
    "road": lambda d: (gen.road(3000, 0.62, device=d), torch.float32),
    "const8big": lambda d: (gen.constant_rows(64_000_000, 8, seed=78, device=d), torch.float32),
    # fp64 variants (C4 is the only fp64 BASELINE config)
    "C2d": lambda d: (gen.config("C2", device=d), torch.float64),
    "band27d": lambda d: (gen.banded(4_000_000, 27, device=d), torch.float64),
    "pld": lambda d: (gen.powerlaw_rows(4_000_000, 16.0, 1.5, device=d), torch.float64),
    "C3d": lambda d: (gen.config("C3", device=d), torch.float64),
    "band2kd": lambda d: (gen.banded(65_536, 2048, device=d), torch.float64),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mats", default="C2,C3,C4,band27,band4,band2k,pl")
    ap.add_argument("--kernels", default="0,1,2,3,4,5,6,7")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=None)
    ap.add_argument("--wave-warps", type=int, default=0,
                    help="persistent-kernel wave size in warps (0 = occupancy-derived; experiments)")
    a = ap.parse_args()
    if a.wave_warps:
        from paper_2403_17017_b200 import _lib
        _lib.load().kp_debug_set_wave_warps(a.wave_warps)
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6650.0
    dev = torch.device("cuda", 0)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    res = {}
    for name in a.mats.split(","):
        m, dt = MATS[name](dev)
        A = m.to_device_csr(dt, device=dev)
        del m
        x = (torch.rand(A.n_cols, device=dev, dtype=torch.float64) * 2 - 1).to(dt)
        y = torch.empty(A.n_rows, device=dev, dtype=dt)
        row = {"rows": A.n_rows, "nnz": A.nnz, "dtype": str(dt)}
        for k in [int(v) for v in a.kernels.split(",")]:
            lab = kernels.KERNELS[k]
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            P = kernels.prepare(A, k, cache=False) if k in kernels.NEEDS_PREP else None
            e1.record()
            torch.cuda.synchronize()
            prep = e0.elapsed_time(e1) * 1e3
            w = None
            if k == kernels.ELL_TM:
                w = int(min(int(P.buf[:64].cpu().view(torch.int64)[3]), P.ell_cap))
            for _ in range(2):
                kernels.spmv(A, x, k, y=y, prepared=P)
            ts = []
            for _ in range(a.reps):
                flush.zero_()
                e0.record()
                kernels.spmv(A, x, k, y=y, prepared=P)
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            t = statistics.median(ts)
            b = A.byte_model(k, w)
            row[lab] = {"us": round(t, 2), "prep_us": round(prep, 1), "gbs": round(b / t / 1e3, 1),
                        "frac": round(b / t / 1e3 / peak, 3)}
            print(f"{name:8s} {lab:13s} {t:10.2f} us  {b / t / 1e3:8.1f} GB/s  {b / t / 1e3 / peak:6.3f}  prep {prep:9.1f} us",
                  flush=True)
            del P
        res[name] = row
        del A, x, y
        torch.cuda.empty_cache()
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
