"""Gathered (dynamically computed) row-density features with measured collection cost.

Drop-in for /root/reference/pkg/src/kernelpick/features.py:35-87:
``GatheredFeatures`` (same fields and ``as_vector`` order max/min/mean/var),
``row_density`` and ``gather_features(m, clock)``.

``gather_features`` runs ONE fused kernel (csrc/kp_reduce.cu, K1): the integer
(min, max, sum of squares) pass over row_offsets and the fp64 epilogue of
features.py:74-85 on the device, rounding op by op like Python floats (no FMA), so
every feature is bit-identical to the reference's on the same offsets.
``collection_time`` is measured by the injected clock around the device pass (use
``clock.CudaEventClock`` for device time).  The Kendall-tau / correlation-table
diagnostics of features.py:90-180 are offline analysis (out of
scope for the runtime path).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

from . import _lib
from .clock import perf_clock

Clock = Callable[[], float]


@dataclass(frozen=True)
class GatheredFeatures:
    """Statistics from an extra pass over the data, plus the cost of that pass."""

    max_row_density: float
    min_row_density: float
    mean_row_density: float
    var_row_density: float
    collection_time: float

    def as_vector(self) -> tuple[float, float, float, float]:
        return (self.max_row_density, self.min_row_density, self.mean_row_density, self.var_row_density)


def row_density(m, row: int) -> float:
    """Stored entries of ``row`` divided by the column count."""
    if m.n_cols == 0:
        raise ValueError("row density undefined for a zero-column matrix")
    if not 0 <= row < m.n_rows:
        raise IndexError(f"row {row} out of range for {m.n_rows}-row matrix")
    off = m.row_offsets
    return int(off[row + 1] - off[row]) / m.n_cols


def _offsets_on_device(m):
    """(tensor, off_type) for a DeviceCSR, a CUDA tensor view, or a host matrix."""
    from .device import DeviceCSR
    torch = _lib.require_cuda()
    if isinstance(m, DeviceCSR):
        return m.row_offsets, m.off_type
    off = m.row_offsets
    if isinstance(off, torch.Tensor) and off.is_cuda:
        t = off.contiguous()
    else:
        import numpy as np
        a = np.ascontiguousarray(off, dtype=np.int64)
        t = torch.from_numpy(a if a.flags.writeable else a.copy()).cuda()
    return t, (_lib.KP_I32 if t.dtype == torch.int32 else _lib.KP_I64)


def gather_outcome(m, out=None, stream=None):
    """Enqueue the fused feature kernel; returns the device kp_outcome buffer (96 B)."""
    torch = _lib.require_cuda()
    from .device import reduce_workspace
    t, off_type = _offsets_on_device(m)
    if out is None:
        out = torch.empty(_lib.OUTCOME_BYTES, dtype=torch.uint8, device=t.device)
    with torch.cuda.device(t.device):
        rc = _lib.load().kp_gather_features(t.data_ptr(), off_type, int(m.n_rows), int(m.n_cols), out.data_ptr(),
                                            reduce_workspace(t.device, stream).data_ptr(),
                                            _lib.stream_handle(stream, t.device))
    _lib.check(rc, "kp_gather_features")
    return out


def decode_outcome(buf, stream=None) -> _lib.kp_outcome:
    """Host copy of a device (or host) kp_outcome.  ``stream``: the stream the outcome was
    written on -- the copy is ordered after it (the D2H itself runs on the buffer device's
    current stream, which waits for ``stream`` first)."""
    if hasattr(buf, "cpu"):
        if stream is not None and buf.is_cuda:
            import torch
            torch.cuda.current_stream(buf.device).wait_stream(stream)
        raw = bytes(buf.cpu().numpy().tobytes())
    else:
        raw = bytes(buf)
    return _lib.kp_outcome.from_buffer_copy(raw)


def gather_features(m, clock: Clock | None = None) -> GatheredFeatures:
    """One pass over row offsets: max/min/mean/population variance of per-row
    densities, timed by ``clock`` (features.py:64-87)."""
    if m.n_rows == 0:
        raise ValueError("cannot gather features of an empty matrix")
    if m.n_cols == 0:
        raise ValueError("cannot gather features of a zero-column matrix")
    clock = clock or perf_clock
    torch = _lib.require_cuda()
    t0 = clock()
    buf = gather_outcome(m)
    o = decode_outcome(buf)  # D2H of 96 bytes: synchronises on the pass
    elapsed = clock() - t0
    if o.status == _lib.KP_ERANGE:
        raise OverflowError("row length / column count beyond 2**53: Python int division semantics "
                            "would not be a single double division")
    del torch
    return GatheredFeatures(o.max_d, o.min_d, o.mean_d, o.var_d, elapsed)

