"""fp64 gather floor on C4's real column array (GPU): us per pass of gather64_probe.so for
2 / 3 / 4 CTAs per SM, with and without an 18 KB shared-memory footprint per CTA (the merge
kernel's).  Run: python tools/probes/gather64_probe.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2403_17017_b200 import gen  # noqa: E402

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "gather64_probe.so"))
lib.g64_run.argtypes = [ctypes.c_int, ctypes.c_int] + [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
dev = torch.device("cuda")
m = gen.config("C4", device=dev)
col = m.col_indices.to(torch.int32).contiguous()
n = col.numel() // 256 * 256
val = torch.rand(n, device=dev, dtype=torch.float64)
x = torch.rand(m.n_cols, device=dev, dtype=torch.float64)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = torch.empty(sms * 8 * 256, dtype=torch.float64, device=dev)
s = torch.cuda.current_stream()
for smem in (0, 18 << 10):
    for mb in (2, 3, 4):
        ts = []
        for rep in range(6):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rc = lib.g64_run(mb, smem, col[:n].data_ptr(), val.data_ptr(), x.data_ptr(), out.data_ptr(), n, sms * mb,
                             s.cuda_stream)
            e1.record()
            torch.cuda.synchronize()
            assert rc == 0, rc
            if rep:
                ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        print(f"C4 fp64 gathers smem={smem >> 10:2d}K ctas/sm={mb}: {ts[len(ts) // 2]:7.1f} us", flush=True)
