"""Long-row deferral of the row-mapped schedules (CSR,WM / CSR,TM, kp_spmv.cu DeferWs):
rows past the schedule's threshold are listed by the sweep and finished by k_long_rows
(PDL tail).  Checked: y vs the fp64 oracle on matrices whose long rows straddle the
warp / CTA split of the tail, bit-identical repeats (the list counter re-zeroes itself),
the workspace left zeroed, and no list at all when no row can be long (n_cols <= T)."""
import ctypes

import numpy as np
import pytest
import torch

from paper_2403_17017_b200 import _lib, gen, kernels

pytestmark = pytest.mark.gpu
TOL = {torch.float32: 1e-5, torch.float64: 1e-12}


def _mk(name, lens, n_cols, seed=3):
    rows = np.repeat(np.arange(len(lens)), lens)
    rng = np.random.default_rng(seed)
    cols = np.concatenate([np.sort(rng.choice(n_cols, l, replace=False)) if l else np.zeros(0, np.int64)
                           for l in lens])
    return gen.from_coo(name, len(lens), n_cols, torch.tensor(rows, dtype=torch.int64),
                        torch.tensor(cols, dtype=torch.int64), seed)


def _fixtures():
    base = [5] * 3000
    lens = list(base)
    # rows on both sides of the WM / TM thresholds (64 x G, 128), of the tail's warp / CTA
    # split (4096), of its CTA / cluster split (65536) and past it
    for i, l in enumerate([127, 128, 129, 255, 256, 257, 4095, 4096, 4097, 30000, 65536, 65537, 90000, 0, 1]):
        lens[100 + 191 * i] = l
    return [_mk("long_rows", lens, 100000), gen.powerlaw_rows(40000, 10.0, 1.2, seed=9),
            gen.config("C4", small=True), gen.config("C2", small=True)]


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("index", ["int32", "int64"])
@pytest.mark.parametrize("kern", [kernels.CSR_WM, kernels.CSR_TM])
def test_long_rows_parity_and_repeat(kern, dtype, index, orc):
    for m in _fixtures():
        A = m.to_device_csr(dtype, index=index)
        g = torch.Generator().manual_seed(7)
        x = (torch.rand(A.n_cols, generator=g, dtype=torch.float64) * 2 - 1).to(dtype).cuda()
        y1 = kernels.spmv(A, x, kern)
        y2 = kernels.spmv(A, x, kern)
        torch.cuda.synchronize()
        assert torch.equal(y1, y2), (m.name, kernels.KERNELS[kern])
        off, col, val = A.to_host()
        yref, absy = orc.spmv_csr(off, col, val, x.cpu().numpy())
        ok, r = orc.spmv_check(y1.cpu().numpy(), yref, absy, TOL[dtype])
        assert ok, (m.name, kernels.KERNELS[kern], dtype, index, r)
        ws = kernels.spmv_workspace(A, kern)
        if ws is not None:  # the tail re-zeroed its counters
            assert int(ws[:16].count_nonzero()) == 0  # count, n_huge, n_giant, done, (m.name, kernels.KERNELS[kern])


def test_no_list_when_rows_cannot_be_long():
    L = _lib.load()
    m = gen.banded(5000, 27)  # n_cols 5000 > both thresholds: a list is sized
    narrow = _mk("narrow", [50] * 2000, 100)  # no row can exceed 100 <= both thresholds
    for mm, want_zero in ((narrow, True), (m, False)):
        A = mm.to_device_csr(torch.float32)
        for k in (kernels.CSR_WM, kernels.CSR_TM):
            nb = ctypes.c_size_t(1)
            _lib.check(L.kp_spmv_workspace_bytes(k, ctypes.byref(A.struct), ctypes.byref(nb)), "ws")
            assert (nb.value == 0) == want_zero, (mm.name, kernels.KERNELS[k], nb.value)
