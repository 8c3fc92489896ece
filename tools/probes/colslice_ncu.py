"""One column slice (S = 3, slice 1) of C5 through the plain merge kernel (kp_spmv) and
the fused-exchange variant (kp_spmv_bcast_acc, with acc) -- for an ncu comparison."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools", "probes"))
import torch  # noqa: E402

from colslice_probe import col_slices  # noqa: E402
from paper_2403_17017_b200 import gen, kernels  # noqa: E402

dev = torch.device("cuda", 0)
A = gen.config("C5", device=dev).to_device_csr(torch.float32, device=dev)
x = torch.rand(A.n_cols, device=dev)
B = col_slices(A, 3)[1]
del A
y = torch.empty(B.n_rows, device=dev)
acc = torch.rand(B.n_rows, device=dev)
for _ in range(2):
    kernels.spmv(B, x, kernels.CSR_WO, y=y)
    kernels.spmv_bcast(B, x, kernels.CSR_WO, [y], 0, acc=acc)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
kernels.spmv(B, x, kernels.CSR_WO, y=y)
kernels.spmv_bcast(B, x, kernels.CSR_WO, [y], 0, acc=acc)
kernels.spmv_bcast(B, x, kernels.CSR_WO, [y], 0)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
