"""Run every kernel on the small parity matrices (for compute-sanitizer)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import test_gpu_spmv as t  # noqa: E402
from paper_2403_17017_b200 import kernels  # noqa: E402

ks = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "0,1,2,3,4,5,6,7").split(",")]
from paper_2403_17017_b200 import _lib, device  # noqa: E402
import numpy as np  # noqa: E402
# few resident warps -> many units per persistent warp (register carries, range fix-ups)
_lib.load().kp_debug_set_wave_warps(int(os.environ.get("KP_WAVE_WARPS", "0")))
# device csr_from_coo (radix sort, run sums, offsets) on a duplicate-heavy input
rng = np.random.default_rng(1)
n = 50000
rows, cols = rng.integers(0, 300, n), rng.integers(0, 200, n)
device.csr_from_coo(300, 200, rows, cols, rng.normal(size=n))
torch.cuda.synchronize()
print("csr_from_coo ok", flush=True)
for m in t.mats():
    for dt in (torch.float32, torch.float64):
        A = m.to_device_csr(dt, index="int32")
        x = torch.rand(A.n_cols, device="cuda", dtype=dt)
        for k in ks:
            print(m.name, dt, kernels.KERNELS[k], flush=True)
            kernels.spmv(A, x, k)
            torch.cuda.synchronize()
# round 2: long-row lists + tail (WM / TM), the compact column transfer, emitted-tree plans
import test_gpu_long_rows as tl  # noqa: E402
for m in tl._fixtures():
    A = m.to_device_csr(torch.float32)
    x = torch.rand(A.n_cols, device="cuda")
    for k in (kernels.CSR_WM, kernels.CSR_TM, kernels.CSR_BM):
        print(m.name, "long rows", kernels.KERNELS[k], flush=True)
        kernels.spmv(A, x, k)
        torch.cuda.synchronize()
    H = device.HostPackedCSR(A)
    d_buf, B = H.staging(A.device)
    H.upload(d_buf, B)
    torch.cuda.synchronize()
    assert torch.equal(B.col_indices, A.col_indices)
print("long rows / pack ok", flush=True)
from paper_2403_17017_b200 import gen, seer  # noqa: E402
model = seer.SeerModel.load(os.path.join(ROOT, "paper_2403_17017_b200", "models", "seer_b200.json"))
A = gen.config("C1").to_device_csr(torch.float32)
x = torch.rand(A.n_cols, device="cuda")
y = torch.empty(A.n_rows, device="cuda")
plan = seer.SeerPlan(model, A, x, y, 100)  # the bundle's gathered path (emitted trees)
plan.launch()
torch.cuda.synchronize()
print("plan", plan.select_kind(), flush=True)
plan.close()
# column-blocked shard: accumulating fused-exchange stores (acc aliasing the destination)
from paper_2403_17017_b200 import dist as kdist  # noqa: E402
m = gen.config("C5", small=True, device="cuda")
for dt in (torch.float32, torch.float64):
    A, plan, _ = kdist.shard_device(m.row_offsets, m.col_indices, m.values, m.n_cols, 0, 1, dt)
    for kern in (kernels.CSR_WO, kernels.CSR_MP):
        run = kdist.ShardedSeer(None, A, plan, 2, m.n_rows, m.n_cols, m.nnz, kernel=kern, col_slices=3)
        run.step(torch.rand(m.n_rows, device="cuda", dtype=dt))
        torch.cuda.synchronize()
        print("column blocks", dt, kernels.KERNELS[kern], flush=True)
print("all ok")
