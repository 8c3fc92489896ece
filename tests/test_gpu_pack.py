"""Device side of the compact column transfer format: kp_unpack_cols restores exactly the
columns kp_pack_cols packed, for bit widths 1..31 and ragged lengths; a HostPackedCSR
round trip feeds an SpMV that matches the oracle."""
import ctypes

import numpy as np
import pytest
import torch

from paper_2403_17017_b200 import _lib, gen, kernels
from paper_2403_17017_b200.device import HostPackedCSR

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_cols", [2, 3, 1000, 1 << 20, (1 << 20) + 1, 10_000_019, 1 << 31])
@pytest.mark.parametrize("n", [1, 33, 4097, 1_000_003])
def test_unpack_inverts_pack(n, n_cols):
    L = _lib.load()
    rng = np.random.default_rng(n ^ n_cols)
    cols = rng.integers(0, n_cols, n, dtype=np.int64).astype(np.int32)
    cols[-1] = n_cols - 1
    h = np.zeros(L.kp_pack_cols_bytes(n, n_cols) // 4, dtype=np.uint32)
    assert L.kp_pack_cols(cols.ctypes.data_as(ctypes.c_void_p), n, n_cols, h.ctypes.data_as(ctypes.c_void_p), 0) == 0
    d = torch.from_numpy(h.view(np.int32)).cuda()
    out = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(L.kp_unpack_cols(d.data_ptr(), n, n_cols, out.data_ptr(), s), "unpack")
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), cols)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_host_packed_round_trip_spmv(dtype, orc):
    m = gen.config("C2", small=True)
    A = m.to_device_csr(dtype)
    H = HostPackedCSR(A)
    assert H.bits == 12 and sum(H.sizes) < A.nnz * (4 + A.values.element_size()) + 4 * (A.n_rows + 1)
    d_buf, B = H.staging(A.device)
    H.upload(d_buf, B)
    torch.cuda.synchronize()
    assert torch.equal(B.col_indices, A.col_indices) and torch.equal(B.values, A.values)
    assert torch.equal(B.row_offsets, A.row_offsets)
    x = (torch.rand(A.n_cols, dtype=torch.float64) * 2 - 1).to(dtype).cuda()
    y = kernels.spmv(B, x, kernels.CSR_WO)
    off, col, val = A.to_host()
    yref, absy = orc.spmv_csr(off, col, val, x.cpu().numpy())
    ok, r = orc.spmv_check(y.cpu().numpy(), yref, absy, 1e-5 if dtype == torch.float32 else 1e-12)
    assert ok, r
