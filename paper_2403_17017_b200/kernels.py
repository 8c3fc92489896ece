"""The SpMV kernel family Seer selects between, and its preprocessing.

Vocabulary order is PAPER.md Table III (:311-318) and never changes: tree class
indices and the lowest-index tie-break of ``fastest_kernel`` depend
on it.  Every call runs the sm_100a kernels in libkpb200.so (csrc/kp_spmv.cu);
there is no CPU path.
"""

from __future__ import annotations

import ctypes
import math

from . import _lib
from .device import DeviceCSR, as_device

KERNELS = ("Adaptive-CSR", "CSR,BM", "CSR,MP", "CSR,WM", "CSR,WO", "CSR,TM", "COO,WM", "ELL,TM")
ADAPTIVE_CSR, CSR_BM, CSR_MP, CSR_WM, CSR_WO, CSR_TM, COO_WM, ELL_TM = range(8)
# kernels whose one-time preprocessing is charged to the first iteration
NEEDS_PREP = frozenset({ADAPTIVE_CSR, CSR_MP, COO_WM, ELL_TM})
# SPEC.md:190 file-name convention: csr_tm.csv <-> "CSR,TM"
FILE_NAMES = {k: KERNELS[k].lower().replace(",", "_").replace("-", "_") for k in range(8)}


def kernel_index(k) -> int:
    if isinstance(k, str):
        return KERNELS.index(k)
    k = int(k)
    if not 0 <= k < len(KERNELS):
        raise ValueError(f"kernel index {k} out of range")
    return k


class Prepared:
    """A kernel's preprocessed format living in one device buffer."""

    def __init__(self, kernel: int, buf, struct: _lib.kp_prepared, ell_cap: int = 0):
        self.kernel = kernel
        self.buf = buf
        self.struct = struct
        self.ell_cap = ell_cap

    @property
    def nbytes(self) -> int:
        return 0 if self.buf is None else int(self.buf.numel())


def default_ell_cap(A: DeviceCSR, budget_bytes: int | None = None) -> int:
    """Reserved ELL width: 2x the mean row length + 8, at most 128 slots (a thread walking
    more is ELL's pitfall: a dense 8192-wide band ran 71x behind CSR,BM at width 8192), and
    within a memory budget.  Rows longer than the actual width are finished by the ELL tail
    kernel (warp / CTA per row), so any cap is correct."""
    torch = _lib.require_cuda()
    if A.n_rows == 0:
        return 1
    mean = A.nnz / A.n_rows
    cap = min(int(math.ceil(2 * mean)) + 8, 128)
    if budget_bytes is None:
        free, _ = torch.cuda.mem_get_info(A.device)
        budget_bytes = free // 4
    per_col = A.n_rows * (4 + A.values.element_size())
    return max(1, min(cap, budget_bytes // max(per_col, 1)))


def prepare(A, kernel, *, ell_cap: int | None = None, stream=None, cache: bool = True) -> Prepared:
    """Run the kernel's preprocessing (K10-K13) on the device; cached on ``A``."""
    torch = _lib.require_cuda()
    A = as_device(A)
    k = kernel_index(kernel)
    if cache and k in A._prepared:
        return A._prepared[k]
    L = _lib.load()
    cap = 0
    if k == ELL_TM:
        cap = int(ell_cap) if ell_cap else default_ell_cap(A)
    nbytes = ctypes.c_size_t(0)
    _lib.check(L.kp_prepare_bytes(k, ctypes.byref(A.struct), cap, ctypes.byref(nbytes)), "kp_prepare_bytes")
    buf = torch.empty(max(int(nbytes.value), 256), dtype=torch.uint8, device=A.device)
    st = _lib.kp_prepared()
    with torch.cuda.device(A.device):
        _lib.check(L.kp_prepare(k, ctypes.byref(A.struct), cap, buf.data_ptr(), buf.numel(), ctypes.byref(st),
                                _lib.stream_handle(stream, A.device)), "kp_prepare")
    P = Prepared(k, buf, st, cap)
    if cache:
        A._prepared[k] = P
    return P


_ws_cache: dict = {}


def spmv_workspace(A: DeviceCSR, kernel: int, stream=None):
    """SpMV scratch (carries of the split-row kernels, the long-row list of CSR,WM / CSR,TM),
    one per (device, kernel, stream): launches on different streams may overlap and must not
    share it.  Zeroed at allocation (the C-ABI contract: kernels leave it zeroed).  Grows to
    the largest matrix."""
    torch = _lib.require_cuda()
    nbytes = ctypes.c_size_t(0)
    _lib.check(_lib.load().kp_spmv_workspace_bytes(kernel, ctypes.byref(A.struct), ctypes.byref(nbytes)),
               "kp_spmv_workspace_bytes")
    n = int(nbytes.value)
    if n == 0:
        return None
    key = (A.device, kernel, _lib.stream_handle(stream, A.device))
    ws = _ws_cache.get(key)
    if ws is None or ws.numel() < n:
        ws = torch.zeros(n, dtype=torch.uint8, device=A.device)
        _ws_cache[key] = ws
    return ws


def spmv(A, x, kernel, *, y=None, prepared: Prepared | None = None, stream=None):
    """y = A.x with the chosen kernel (index or label).  Preprocesses on first use."""
    torch = _lib.require_cuda()
    A = as_device(A)
    k = kernel_index(kernel)
    check_vector(x, A, A.n_cols, "x")
    x = x.contiguous()
    if y is None:
        y = torch.empty(A.n_rows, dtype=A.values.dtype, device=A.device)
    else:
        check_vector(y, A, A.n_rows, "y", out=True)
    if k in NEEDS_PREP and prepared is None:
        prepared = prepare(A, k, stream=stream)
    ws = spmv_workspace(A, k, stream)
    P = ctypes.byref(prepared.struct) if prepared is not None else None
    with torch.cuda.device(A.device):
        rc = _lib.load().kp_spmv(k, ctypes.byref(A.struct), P, x.data_ptr(), y.data_ptr(),
                                 0 if ws is None else ws.data_ptr(), 0 if ws is None else ws.numel(),
                                 _lib.stream_handle(stream, A.device))
    _lib.check(rc, f"kp_spmv[{KERNELS[k]}]")
    return y


def check_vector(v, A, n: int, name: str, out: bool = False) -> None:
    """x / y contract of the C-ABI: a CUDA tensor on A's device with A's value dtype and
    at least ``n`` elements (exactly n for an input); outputs must also be contiguous,
    since the kernels write n elements through the raw pointer."""
    ok = (v.is_cuda and v.device == A.device and v.dtype == A.values.dtype and
          (v.numel() >= n if out else v.numel() == n) and (v.is_contiguous() or not out))
    if not ok:
        raise ValueError(f"{name} must be a {'contiguous ' if out else ''}CUDA tensor on {A.device} with "
                         f"{'>= ' if out else ''}{n} elements of {A.values.dtype} (got {tuple(v.shape)} "
                         f"{v.dtype} on {v.device})")


def spmv_bcast(A, x, kernel, dests, self_index: int, *, prepared: Prepared | None = None, stream=None,
               acc=None, rows=None):
    """kp_spmv_bcast: y = A.x written from the kernel's own epilogue into every tensor of
    ``dests`` (this rank's slice of each rank's next-x buffer; peer-mapped symmetric memory
    or local tensors), ``dests[self_index]`` being the local copy.  Merge-path kernels only.
    ``acc`` (n_rows elements, may be ``dests[self_index]``): y = acc + A.x instead
    (kp_spmv_bcast_acc, the column-blocked iteration of dist.ShardedSeer).  ``rows`` (int32,
    n_rows entries): row r of A is row rows[r] of the single destination / acc (a
    compressed-row block accumulating in place)."""
    torch = _lib.require_cuda()
    A = as_device(A)
    k = kernel_index(kernel)
    if k not in (CSR_MP, CSR_WO):
        raise ValueError("fused exchange is implemented for the merge-path kernels (CSR,MP / CSR,WO)")
    if not 1 <= len(dests) <= _lib.KP_MAX_PEERS or not 0 <= self_index < len(dests):
        raise ValueError("1..8 destinations and a valid self index")
    check_vector(x, A, A.n_cols, "x")
    for d in dests:
        if d.dtype != A.values.dtype or d.numel() < A.n_rows or not d.is_contiguous() or not d.is_cuda:
            raise ValueError("each destination needs n_rows contiguous elements of the matrix value dtype")
    if k in NEEDS_PREP and prepared is None:
        prepared = prepare(A, k, stream=stream)
    if acc is not None and (acc.dtype != A.values.dtype or acc.numel() < A.n_rows or not acc.is_contiguous()
                            or not acc.is_cuda):
        raise ValueError("acc needs n_rows contiguous elements of the matrix value dtype")
    if rows is not None:
        if rows.dtype != torch.int32 or rows.numel() != A.n_rows or not rows.is_contiguous() or not rows.is_cuda:
            raise ValueError("rows needs n_rows contiguous int32 entries on the device")
        if len(dests) != 1 or (acc is not None and acc.data_ptr() != dests[0].data_ptr()):
            raise ValueError("a row map scatters into one destination, accumulating in place")
    pe = _lib.kp_peers()
    for i, d in enumerate(dests):
        pe.y[i] = d.data_ptr()
    pe.n, pe.self = len(dests), int(self_index)
    ws = spmv_workspace(A, k, stream)
    P = ctypes.byref(prepared.struct) if prepared is not None else None
    with torch.cuda.device(A.device):
        _lib.check(_lib.load().kp_spmv_bcast_acc(k, ctypes.byref(A.struct), P, x.data_ptr(),
                                                 0 if acc is None else acc.data_ptr(),
                                                 0 if rows is None else rows.data_ptr(), ctypes.byref(pe),
                                                 0 if ws is None else ws.data_ptr(), 0 if ws is None else ws.numel(),
                                                 _lib.stream_handle(stream, A.device)),
                   f"kp_spmv_bcast_acc[{KERNELS[k]}]")
