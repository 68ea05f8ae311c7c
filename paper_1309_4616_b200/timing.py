"""Optional device-side timing of Newton-Leja series (CUDA events recorded on
the launching stream around each asynchronously enqueued series, before the
single host read-back).  Used by bench.py for the live roofline numbers."""

from __future__ import annotations

import torch

_active = None


class SeriesTimer:
    def __init__(self):
        self.records: list[tuple[torch.cuda.Event, torch.cuda.Event, int]] = []
        self.device_ms: list[tuple[float, int]] = []  # series timed inside a fused step call

    def __enter__(self):
        global _active
        self._prev, _active = _active, self
        return self

    def __exit__(self, *exc):
        global _active
        _active = self._prev

    def add(self, start, end, matvecs: int) -> None:
        self.records.append((start, end, int(matvecs)))

    def add_ms(self, ms: float, matvecs: int) -> None:
        self.device_ms.append((float(ms), int(matvecs)))

    def passes(self) -> int:
        """HBM passes of the recorded series when each pass fuses two nodes."""
        ms = [m for _, _, m in self.records] + [m for _, m in self.device_ms]
        return sum((m + 1) // 2 for m in ms)

    def totals(self):
        """(seconds spent in series, matvecs) over all recorded series."""
        torch.cuda.synchronize()
        ms = sum(s.elapsed_time(e) for s, e, _ in self.records) + sum(t for t, _ in self.device_ms)
        return ms * 1e-3, sum(m for _, _, m in self.records) + sum(m for _, m in self.device_ms)


def active():
    return _active


def event():
    ev = torch.cuda.Event(enable_timing=True)
    ev.record()
    return ev
