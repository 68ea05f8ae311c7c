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
        self.pass_counts: list[tuple[int, int]] = []  # (matvecs, passes) of every recorded series

    def __enter__(self):
        global _active
        self._prev, _active = _active, self
        return self

    def __exit__(self, *exc):
        global _active
        _active = self._prev

    def add(self, start, end, matvecs: int, passes: int | None = None) -> None:
        self.records.append((start, end, int(matvecs)))
        self.pass_counts.append((int(matvecs), int(passes if passes is not None else matvecs)))

    def add_ms(self, ms: float, matvecs: int, passes: int | None = None) -> None:
        self.device_ms.append((float(ms), int(matvecs)))
        self.pass_counts.append((int(matvecs), int(passes if passes is not None else matvecs)))

    def passes(self) -> int:
        """Sweeps over the operand of the recorded series (the series'
        own count: a two-node series may end with a one-node pass)."""
        return sum(p for _, p in self.pass_counts)

    def pass_mix(self) -> tuple[int, int]:
        """(two-node passes, one-node passes) of the recorded series."""
        two = sum(m - p for m, p in self.pass_counts)
        return two, sum(p for _, p in self.pass_counts) - two

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
