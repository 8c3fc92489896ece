"""Every SpMV kernel vs the fp64-accumulating CPU oracle, normwise tolerance
|y - y_ref|_i <= tol * sum_j |a_ij x_j| with tol = 1e-5 (fp32) / 1e-12 (fp64)."""
import numpy as np
import pytest
import torch

from paper_2403_17017_b200 import gen, kernels
from paper_2403_17017_b200.device import DeviceCSR

pytestmark = pytest.mark.gpu
TOL = {torch.float32: 1e-5, torch.float64: 1e-12}


def _edge_matrices():
    ms = []
    # all rows empty but one; empty leading/trailing rows; single row; single column
    def mk(name, R, C, rows, cols):
        return gen.from_coo(name, R, C, torch.tensor(rows, dtype=torch.int64), torch.tensor(cols, dtype=torch.int64), 9)
    ms.append(mk("one_entry", 1000, 1000, [500], [3]))
    ms.append(mk("single_row", 1, 6000, [0] * 3000, list(range(0, 6000, 2))[:3000]))
    ms.append(mk("single_col", 3000, 1, list(range(3000)), [0] * 3000))
    ms.append(mk("empty_ends", 5000, 100, [2000, 2000, 2001, 2999], [1, 5, 7, 99]))
    # row lengths straddling tile / chunk / long-row thresholds
    lens = [0, 1, 255, 256, 257, 1023, 1024, 1025, 2047, 2048, 2049, 8191, 8192, 8193, 20000, 0, 3, 0]
    rows = np.repeat(np.arange(len(lens)), lens)
    cols = np.concatenate([np.arange(l) for l in lens])
    ms.append(mk("thresholds", len(lens), 20001, rows.tolist(), cols.tolist()))
    ms.append(gen.powerlaw_rows(30000, 12.0, 1.3, seed=4))
    ms.append(gen.constant_rows(50000, 3, seed=2))
    ms.append(gen.banded(40000, 27))
    # known mean <= 4 (CSR,BM's thread-per-row variant) with a few long rows mixed in
    ms.append(gen.road(120, 0.6))
    ms.append(gen.circuit(20000, 3, 0.02))
    return ms


MATS = None


def mats():
    global MATS
    if MATS is None:
        MATS = [gen.config(c, small=True) for c in ("C1", "C2", "C3", "C4", "C5")] + _edge_matrices()
        for m in MATS:
            m.to_sparse_csr()  # every fixture must be a canonical, in-range CSR
    return MATS


def _check(m, A, kern, y, orc):
    off, col, val = A.to_host()
    x = XS[(m.name, A.values.dtype)]
    yref, absy = orc.spmv_csr(off, col, val, x.cpu().numpy())
    ok, ratio = orc.spmv_check(y.cpu().numpy(), yref, absy, TOL[A.values.dtype])
    assert ok, f"{m.name} {kernels.KERNELS[kern]} {A.values.dtype} {A.row_offsets.dtype}: ratio {ratio}"


XS = {}


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("index", ["int32", "int64"])
@pytest.mark.parametrize("kern", range(8))
def test_kernel_parity(kern, dtype, index, orc):
    for m in mats():
        A = m.to_device_csr(dtype, index=index)
        key = (m.name, dtype)
        if key not in XS:
            g = torch.Generator().manual_seed(3)
            XS[key] = (torch.rand(m.n_cols, generator=g, dtype=torch.float64) * 2 - 1).to(dtype).cuda()
        x = XS[key]
        y = torch.full((A.n_rows,), float("nan"), dtype=dtype, device="cuda")
        kernels.spmv(A, x, kern, y=y)
        torch.cuda.synchronize()
        _check(m, A, kern, y, orc)
        # determinism: bit-identical on a re-run (no float atomics)
        y2 = kernels.spmv(A, x, kern)
        assert torch.equal(y, y2)


def test_ell_hybrid_tail_small_cap(orc):
    m = gen.config("C4", small=True)
    A = m.to_device_csr(torch.float32)
    P = kernels.prepare(A, kernels.ELL_TM, ell_cap=4, cache=False)
    x = (torch.rand(A.n_cols, dtype=torch.float64) * 2 - 1).float().cuda()
    XS[(m.name + "_ell", torch.float32)] = x
    y = kernels.spmv(A, x, kernels.ELL_TM, prepared=P)
    off, col, val = A.to_host()
    yref, absy = orc.spmv_csr(off, col, val, x.cpu().numpy())
    assert orc.spmv_check(y.cpu().numpy(), yref, absy, 1e-5)[0]


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("cap", [1, 3, 17, 4096])
def test_ell_tail_lists(cap, dtype, orc):
    """K12's tail lists: rows longer than the width W go to the warp list, rows with more
    than kEllLongTail (4096) elements past W to the CTA list; the sweep keeps their first W
    elements and k_ell_tail adds the rest.  Lengths straddle W and W + 4096 for each cap;
    re-runs are bit-identical (the lists' order is atomic-dependent, the sums are not)."""
    lens = [0, 1, 2, 3, 4, 5, 16, 17, 18, 40, 4096, 4097, 4099, 4100, 4113, 9000, 30000, 0, 7, 100000]
    lens = lens * 3
    rows = np.repeat(np.arange(len(lens)), lens)
    cols = np.concatenate([(np.arange(l) * 7919) % 150000 for l in lens])
    m = gen.from_coo("elltail", len(lens), 150000, torch.tensor(rows), torch.tensor(cols), 11)
    A = m.to_device_csr(dtype)
    P = kernels.prepare(A, kernels.ELL_TM, ell_cap=cap, cache=False)
    x = (torch.rand(A.n_cols, dtype=torch.float64, generator=torch.Generator().manual_seed(5)) * 2 - 1).to(dtype).cuda()
    y = torch.full((A.n_rows,), float("nan"), dtype=dtype, device="cuda")
    kernels.spmv(A, x, kernels.ELL_TM, y=y, prepared=P)
    off, col, val = A.to_host()
    yref, absy = orc.spmv_csr(off, col, val, x.cpu().numpy())
    ok, r = orc.spmv_check(y.cpu().numpy(), yref, absy, TOL[dtype])
    assert ok, (cap, r)
    hdr = P.buf[:128].cpu().view(torch.int64)
    W = min(int(hdr[3]), cap)
    assert int(hdr[7]) == sum(1 for v in lens if v > W)                    # n_tail
    assert int(hdr[8]) == sum(1 for v in lens if v - W > 4096)             # n_long
    for _ in range(2):
        assert torch.equal(kernels.spmv(A, x, kernels.ELL_TM, prepared=P), y)


def test_c2_full_size_every_kernel_agrees(orc):
    """Full-size C2 (R-MAT s20): every kernel vs the oracle (sampled-free full check)."""
    m = gen.config("C2", device="cuda")
    A = m.to_device_csr(torch.float32)
    x = (torch.rand(A.n_cols, device="cuda", dtype=torch.float64) * 2 - 1).float()
    off, col, val = A.to_host()
    yref, absy = orc.spmv_csr(off, col, val, x.cpu().numpy())
    for k in range(8):
        y = kernels.spmv(A, x, k)
        ok, r = orc.spmv_check(y.cpu().numpy(), yref, absy, 1e-5)
        assert ok, (kernels.KERNELS[k], r)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("warps", [1, 3, 7, 64])
def test_persistent_ranges_many_units_per_warp(warps, dtype, orc):
    """Force few resident warps so each warp walks many consecutive units (register
    carries across units, rows spanning warp ranges -> fix-up runs) on every fixture."""
    from paper_2403_17017_b200 import _lib
    L = _lib.load()
    prev = L.kp_debug_set_wave_warps(warps)
    try:
        for m in mats():
            A = m.to_device_csr(dtype)
            key = (m.name, dtype)
            if key not in XS:
                g = torch.Generator().manual_seed(3)
                XS[key] = (torch.rand(m.n_cols, generator=g, dtype=torch.float64) * 2 - 1).to(dtype).cuda()
            for kern in (kernels.kernel_index("CSR,MP"), kernels.kernel_index("CSR,WO"), kernels.kernel_index("COO,WM")):
                y = torch.full((A.n_rows,), float("nan"), dtype=dtype, device="cuda")
                kernels.spmv(A, XS[key], kern, y=y, prepared=kernels.prepare(A, kern, cache=False)
                             if kern in kernels.NEEDS_PREP else None)
                torch.cuda.synchronize()
                _check(m, A, kern, y, orc)
    finally:
        L.kp_debug_set_wave_warps(prev)


def test_coo_misaligned_user_arrays(orc):
    """kp_spmv on col / val pointers that are not 16-byte aligned (a caller's view into a
    larger buffer): COO,WM takes its scalar-load path instead of faulting."""
    import ctypes
    from paper_2403_17017_b200 import _lib
    m = gen.config("C2", small=True)
    A = m.to_device_csr(torch.float32)
    colb = torch.empty(A.nnz + 1, dtype=torch.int32, device="cuda")
    valb = torch.empty(A.nnz + 1, dtype=torch.float32, device="cuda")
    colb[1:].copy_(A.col_indices)
    valb[1:].copy_(A.values)
    st = _lib.kp_csr(A.n_rows, A.n_cols, A.nnz, A.off_type, A.val_type, A.row_offsets.data_ptr(),
                     colb[1:].data_ptr(), valb[1:].data_ptr())
    x = (torch.rand(A.n_cols, dtype=torch.float64) * 2 - 1).float().cuda()
    P = kernels.prepare(A, kernels.COO_WM, cache=False)
    ws = kernels.spmv_workspace(A, kernels.COO_WM)
    y = torch.empty(A.n_rows, dtype=torch.float32, device="cuda")
    _lib.check(_lib.load().kp_spmv(kernels.COO_WM, ctypes.byref(st), ctypes.byref(P.struct), x.data_ptr(),
                                   y.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_handle()), "kp_spmv")
    torch.cuda.synchronize()
    off, col, val = A.to_host()
    yref, absy = orc.spmv_csr(off, col, val, x.cpu().numpy())
    assert orc.spmv_check(y.cpu().numpy(), yref, absy, 1e-5)[0]


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_wide_x_half_wave(dtype, orc):
    """x larger than 64 MB: the persistent kernels (merge, COO) run half a wave of warps
    (DRAM-bound gathers); every kernel still matches the oracle."""
    R, C, Z = 200_000, 20_000_000, 6_000_000
    g = torch.Generator().manual_seed(11)
    rows = torch.randint(0, R, (Z,), generator=g)
    cols = torch.randint(0, C, (Z,), generator=g)
    m = gen.from_coo("wide_x", R, C, rows, cols, 5)
    A = m.to_device_csr(dtype)
    x = (torch.rand(C, generator=g, dtype=torch.float64) * 2 - 1).to(dtype).cuda()
    off, col, val = A.to_host()
    yref, absy = orc.spmv_csr(off, col, val, x.cpu().numpy())
    for k in range(8):
        y = torch.full((A.n_rows,), float("nan"), dtype=dtype, device="cuda")
        kernels.spmv(A, x, k, y=y)
        ok, r = orc.spmv_check(y.cpu().numpy(), yref, absy, TOL[dtype])
        assert ok, (kernels.KERNELS[k], r)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("index", ["int32", "int64"])
def test_tm_medium_row_stages(dtype, index, orc):
    """CSR,TM enlarged stages (mean row length > ~9: capacity from the known mean, two
    consumer threads per row) on ragged row counts, means around and above the largest
    stage (per-tile fallback to direct walks), and skewed tiles that overflow their stage."""
    ms = [gen.banded(10_001, 10), gen.banded(70_003, 27), gen.constant_rows(33_333, 40, seed=6),
          gen.banded(5_000, 60), gen.stencil27(23)]
    # mean ~27 with a few 5000-long rows: the tiles holding them overflow the stage
    R = 20_000
    lens = np.full(R, 27)
    lens[[17, 9000, 19_999]] = 5000
    rows = np.repeat(np.arange(R), lens)
    cols = np.concatenate([np.sort(np.random.default_rng(l + i).choice(20_000, l, replace=False))
                           for i, l in enumerate(lens)])
    ms.append(gen.from_coo("skewed_tiles", R, 20_000, torch.tensor(rows), torch.tensor(cols), 5))
    for m in ms:
        A = m.to_device_csr(dtype, index=index)
        key = (m.name, dtype)
        if key not in XS:
            g = torch.Generator().manual_seed(5)
            XS[key] = (torch.rand(m.n_cols, generator=g, dtype=torch.float64) * 2 - 1).to(dtype).cuda()
        y = torch.full((A.n_rows,), float("nan"), dtype=dtype, device="cuda")
        kernels.spmv(A, XS[key], kernels.CSR_TM, y=y)
        torch.cuda.synchronize()
        _check(m, A, kernels.CSR_TM, y, orc)
        assert torch.equal(y, kernels.spmv(A, XS[key], kernels.CSR_TM))
