"""Small driver for profiling the fused selection / feature kernel (K1/K15) on C2."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2403_17017_b200 import features, gen, seer  # noqa: E402

A = gen.config(sys.argv[1] if len(sys.argv) > 1 else "C2", device="cuda").to_device_csr(torch.float32)
model = seer.SeerModel.load(os.path.join(ROOT, "paper_2403_17017_b200", "models", "seer_b200.json"))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ts = {"select": [], "gather": []}
for i in range(8):
    for name, fn in (("select", lambda: seer.select_async(model, A, 1)), ("gather", lambda: features.gather_outcome(A))):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        if i >= 2:
            ts[name].append(e0.elapsed_time(e1) * 1e3)
print({k: sorted(v) for k, v in ts.items()})
