"""One SpMV launch of kernel K on a matrix, for an ncu capture (GPU).  Warms up twice, then
launches once more; capture that launch with e.g.
    ncu --set full --clock-control none --import-source on -k regex:k_csr_merge --launch-skip 2 \
        --launch-count 1 -o gpurun_out/full_C4_wo python tools/ncu_one.py C4 4
(the preparation kernels of MP/COO/ELL/Adaptive run before the warm-ups and are not matched
by a SpMV kernel regex)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

from kbench import MATS  # noqa: E402
from paper_2403_17017_b200 import kernels  # noqa: E402

name, kern = sys.argv[1], int(sys.argv[2])
m, dt = MATS[name](torch.device("cuda"))
A = m.to_device_csr(dt)
del m
x = (torch.rand(A.n_cols, device="cuda", dtype=torch.float64) * 2 - 1).to(dt)
y = torch.empty(A.n_rows, device="cuda", dtype=dt)
P = kernels.prepare(A, kern, cache=False) if kern in kernels.NEEDS_PREP else None
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    flush.zero_()
    kernels.spmv(A, x, kern, y=y, prepared=P)
torch.cuda.synchronize()
print(f"{name} {kernels.KERNELS[kern]} rows={A.n_rows} nnz={A.nnz}")
