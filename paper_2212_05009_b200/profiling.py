"""Per-kernel spans timed with CUDA events on the launching stream.

`KernelTimer` is installed around an epoch (eager or while capturing a CUDA
graph: inside a capture the events become external event nodes, so every
replay re-times them).  Each span carries the kernel's *algorithmic* bytes
(DESIGN.md §5), so achieved GB/s = bytes / span time.
"""

from __future__ import annotations

import ctypes
from contextlib import contextmanager
from dataclasses import dataclass

from . import _lib

_ACTIVE = None


@dataclass
class Span:
    name: str
    algo_bytes: int
    flops: int
    ev0: int
    ev1: int


class KernelTimer:
    def __init__(self):
        self.spans: list[Span] = []
        self._pool: list[int] = []

    def _event(self) -> int:
        ev = ctypes.c_void_p()
        _lib.call("gcnb_event_create", ctypes.byref(ev))
        self._pool.append(ev.value)
        return ev.value

    def record(self, name: str, algo_bytes: int, flops: int, stream: int):
        cap = ctypes.c_int32(0)
        _lib.call("gcnb_stream_is_capturing", stream, ctypes.byref(cap))
        ev0, ev1 = self._event(), self._event()
        _lib.call("gcnb_event_record", ev0, stream, cap.value)
        return Span(name, int(algo_bytes), int(flops), ev0, ev1), cap.value

    def results(self) -> list[tuple[str, int, int, float]]:
        """[(name, algo_bytes, flops, ms)] for the last execution (call after a sync)."""
        out = []
        ms = ctypes.c_float(0.0)
        for s in self.spans:
            _lib.call("gcnb_event_elapsed_ms", s.ev0, s.ev1, ctypes.byref(ms))
            out.append((s.name, s.algo_bytes, s.flops, float(ms.value)))
        return out

    def close(self) -> None:
        for ev in self._pool:
            _lib.call("gcnb_event_destroy", ev)
        self._pool.clear()
        self.spans.clear()


@contextmanager
def active(timer: KernelTimer | None):
    global _ACTIVE
    prev, _ACTIVE = _ACTIVE, timer
    try:
        yield timer
    finally:
        _ACTIVE = prev


@contextmanager
def span(name: str, algo_bytes: int, flops: int, stream: int):
    t = _ACTIVE
    if t is None:
        yield
        return
    sp, external = t.record(name, algo_bytes, flops, stream)
    yield
    _lib.call("gcnb_event_record", sp.ev1, stream, external)
    t.spans.append(sp)
