"""One column-blocked C5 iteration at N = 1 (ShardedSeer local path, auto slices) between
cudaProfilerStart/Stop -- for an ncu capture of its merge launches (DRAM bytes vs the
byte model).  Also runs the unblocked SpMV once for comparison."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2403_17017_b200 import dist as kdist  # noqa: E402
from paper_2403_17017_b200 import gen, kernels  # noqa: E402

m = gen.config("C5", device="cuda")
A, plan, _ = kdist.shard_device(m.row_offsets, m.col_indices, m.values, m.n_cols, 0, 1, torch.float32)
R, C, Z = m.n_rows, m.n_cols, m.nnz
del m
torch.cuda.empty_cache()
run = kdist.ShardedSeer(None, A, plan, 1, R, C, Z, exchange="nccl", kernel=kernels.CSR_WO)
x = torch.rand(C, device="cuda")
y = torch.empty(R, device="cuda")
Ps = run.prepare()
for _ in range(2):
    run.spmv_into(x, [y], 0, Ps)
    kernels.spmv(A, x, kernels.CSR_WO, y=y)
torch.cuda.synchronize()
print("col_slices", run.col_slices, "byte model", A.byte_model(kernels.CSR_WO, None), flush=True)
torch.cuda.cudart().cudaProfilerStart()
run.spmv_into(x, [y], 0, Ps)          # blocked: S merge launches (+ fix-ups)
kernels.spmv(A, x, kernels.CSR_WO, y=y)  # unblocked
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
