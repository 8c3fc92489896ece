"""Injectable time sources (reference: /root/reference/pkg/src/kernelpick/clock.py:11-29).

``perf_clock`` and ``FixedClock`` keep the reference's call shape ``() -> float``.
``CudaEventClock`` is the B200 addition: each call records a CUDA event on the
current stream and returns seconds since the clock's first event, measured on the
device (the call synchronises on the event it just recorded).  Passing it to
``gather_features`` times the feature pass as the GPU saw it, without host jitter.
"""

from __future__ import annotations

import time


def perf_clock() -> float:
    """Host wall clock (time.perf_counter)."""
    return time.perf_counter()


class FixedClock:
    """Every call advances by ``tick``: any measured duration is exactly ``tick``."""

    def __init__(self, start: float = 0.0, tick: float = 1e-7):
        self._t = start
        self.tick = tick

    def __call__(self) -> float:
        self._t += self.tick
        return self._t


class CudaEventClock:
    """Device-side clock: seconds between CUDA events on the current stream."""

    def __init__(self, stream=None):
        import torch
        self._torch = torch
        self._stream = stream
        self._origin = None

    def __call__(self) -> float:
        torch = self._torch
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(self._stream)
        ev.synchronize()
        if self._origin is None:
            self._origin = ev
            return 0.0
        return self._origin.elapsed_time(ev) * 1e-3
