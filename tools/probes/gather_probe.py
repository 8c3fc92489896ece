"""Gather-floor probe (GPU): time gather_probe.so's kernels on C2's real column array and on
uniform-random columns; prints us per pass and Gnnz/s.  Run: python tools/probes/gather_probe.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2403_17017_b200 import gen  # noqa: E402

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "gather_probe.so"))
lib.gp_run.argtypes = [ctypes.c_int, ctypes.c_int] + [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_int,
                                                                                ctypes.c_void_p]
NAMES = {0: "ldg(nc)", 1: "nc.no_alloc", 2: "cg(L2 only)", 3: "ca", 4: "nc.evict_last", 5: "no gather"}


def main():
    dev = torch.device("cuda")
    A = gen.config("C2", device=dev)
    col = A.col_indices.to(torch.int32).contiguous()  # gen.Matrix holds int64
    n = col.numel() // 256 * 256
    C = A.n_cols
    val = torch.rand(n, device=dev)
    x = torch.rand(C, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    out = torch.empty(sms * 32 * 256, device=dev)
    s = torch.cuda.current_stream()
    cols = {"C2": col[:n], "uniform": torch.randint(0, C, (n,), device=dev, dtype=torch.int32),
            "sorted-C2": torch.sort(col[:n])[0].to(torch.int32)}
    cfgs = [(0, -1), (25 << 10, -1)]
    if os.environ.get("GP_ONE"):  # one launch per mode for ncu
        cfgs = [(0, -1)]
    for smem, carve in cfgs:
      lib.gp_config(smem, carve)
      for cname, cc in cols.items():
        for wv in (0, 1):
            for per_sm in ((8,) if os.environ.get("GP_ONE") else (4, 8)):
                for m in ((0, 1) if os.environ.get("GP_ONE") else (0, 1, 5)):
                    ts = []
                    for rep in range(2 if os.environ.get("GP_ONE") else 6):
                        flush.zero_()
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        rc = lib.gp_run(m, wv, cc.data_ptr(), val.data_ptr(), x.data_ptr(), out.data_ptr(), n,
                                        sms * per_sm, s.cuda_stream)
                        e1.record()
                        torch.cuda.synchronize()
                        assert rc == 0, rc
                        if rep:
                            ts.append(e0.elapsed_time(e1) * 1e3)
                    ts.sort()
                    us = ts[len(ts) // 2]
                    print(f"smem={smem >> 10:3d}K carve={carve:4d} {cname:9s} val={wv} ctas/sm={per_sm:2d} {NAMES[m]:14s} {us:7.1f} us  "
                          f"{n / us / 1e3:6.2f} Gnnz/s", flush=True)


if __name__ == "__main__":
    main()
