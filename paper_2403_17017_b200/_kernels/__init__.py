"""Drop-in replacement for the reference backend ``kernelpick._kernels``
(/root/reference/pkg/src/kernelpick/_kernels/__init__.py:1-28).

Same three names, same return types:

* ``BACKEND`` -- ``"cuda"`` (the reference reports "compiled" or "pure");
* ``length_stats(row_offsets) -> (min, max, sum, sumsq)`` as Python ints
  (_core.pyx:15-33, _pure.py:11-21), int64 wrapping semantics;
* ``wave_ceil_max_sum(row_offsets, divisor, wave_rows) -> int`` (_core.pyx:36-56).

``row_offsets`` may be any array-like (numpy, read-only arrays included -- the
reference's compiled backend rejects those) which is uploaded, or
a CUDA ``torch.Tensor`` (int32/int64) used in place.  Both run kernel K1/K2 of
libkpb200.so on the GPU; there is no CPU fallback (the call raises
``BackendUnavailable`` without a GPU).  Invalid divisor / wave_rows raise
``ValueError`` (the reference backends diverge there).
"""

from __future__ import annotations

import numpy as np

from .. import _lib

BACKEND = "cuda"


def _device_offsets(row_offsets):
    torch = _lib.require_cuda()
    if isinstance(row_offsets, torch.Tensor) and row_offsets.is_cuda:
        t = row_offsets.contiguous()
        if t.dtype not in (torch.int32, torch.int64):
            t = t.to(torch.int64)
    else:
        a = np.ascontiguousarray(np.asarray(row_offsets), dtype=np.int64)
        t = torch.from_numpy(a.copy() if not a.flags.writeable else a).cuda()
    off_type = _lib.KP_I32 if t.dtype == torch.int32 else _lib.KP_I64
    return torch, t, off_type


def length_stats(row_offsets) -> tuple[int, int, int, int]:
    """(min, max, sum, sum of squares) of per-row entry counts (K1 on the GPU)."""
    torch, t, off_type = _device_offsets(row_offsets)
    from ..device import reduce_workspace
    out = torch.empty(4, dtype=torch.int64, device=t.device)
    with torch.cuda.device(t.device):
        rc = _lib.load().kp_length_stats(t.data_ptr(), off_type, t.numel(), out.data_ptr(),
                                         reduce_workspace(t.device).data_ptr(), _lib.stream_handle(None, t.device))
    _lib.check(rc, "kp_length_stats")
    lo, hi, s1, s2 = out.cpu().tolist()
    return int(lo), int(hi), int(s1), int(s2)


def wave_ceil_max_sum(row_offsets, divisor: int, wave_rows: int) -> int:
    """Sum over consecutive waves of `wave_rows` rows of max ceil(len / divisor) (K2)."""
    if int(divisor) <= 0 or int(wave_rows) <= 0:
        raise ValueError("divisor and wave_rows must be positive")
    torch, t, off_type = _device_offsets(row_offsets)
    from ..device import reduce_workspace
    out = torch.empty(1, dtype=torch.int64, device=t.device)
    with torch.cuda.device(t.device):
        rc = _lib.load().kp_wave_ceil_max_sum(t.data_ptr(), off_type, t.numel(), int(divisor), int(wave_rows),
                                              out.data_ptr(), reduce_workspace(t.device).data_ptr(),
                                              _lib.stream_handle(None, t.device))
    _lib.check(rc, "kp_wave_ceil_max_sum")
    return int(out.item())


__all__ = ["BACKEND", "length_stats", "wave_ceil_max_sum"]
