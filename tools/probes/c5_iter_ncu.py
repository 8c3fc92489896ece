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
if "--reorder" in sys.argv:  # as bench.py's C5 distributes it
    order, newid = kdist.degree_order(m.col_indices, m.n_cols)
    m.row_offsets, m.col_indices, m.values = kdist.permute_symmetric(m.row_offsets, m.col_indices, m.values,
                                                                    order, newid)
    del order, newid
A, plan, _ = kdist.shard_device(m.row_offsets, m.col_indices, m.values, m.n_cols, 0, 1, torch.float32)
R, C, Z = m.n_rows, m.n_cols, m.nnz
del m
torch.cuda.empty_cache()
run = kdist.ShardedSeer(None, A, plan, 1, R, C, Z, exchange="nccl", kernel=kernels.CSR_WO,
                        col_slices=1 if "--reorder" in sys.argv else "auto")
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
