"""TMA gather4 vs LSU gather floor on C2's columns (GPU): us per pass.  The LSU numbers for
the same columns are in profiles/gather_floor_r01.txt (val=0: 59-68 us).
Run: python tools/probes/gather4_probe.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2403_17017_b200 import gen  # noqa: E402

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "gather4_probe.so"))
lib.g4_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                       ctypes.c_int, ctypes.c_void_p]
dev = torch.device("cuda")
m = gen.config("C2", device=dev)
col = m.col_indices.to(torch.int32).contiguous()
n = col.numel() // 256 * 256
x = torch.rand(m.n_cols, device=dev)
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = torch.empty(sms * 2 * 256, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
s = torch.cuda.current_stream()
for name, cc in (("C2", col[:n]), ("uniform", torch.randint(0, m.n_cols, (n,), device=dev, dtype=torch.int32)),
                 ("sorted-C2", torch.sort(col[:n])[0].to(torch.int32))):
    ts = []
    for rep in range(6):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = lib.g4_run(cc.data_ptr(), x.data_ptr(), m.n_cols, out.data_ptr(), n, sms, s.cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        assert rc == 0, rc
        if rep:
            ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    # check: acc over all elements equals the LSU sum
    print(f"{name:9s} TMA gather4 {ts[len(ts) // 2]:7.1f} us  ({n / ts[len(ts) // 2] / 1e3:6.1f} G gathers/s)", flush=True)
