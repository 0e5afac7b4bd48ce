"""Per-kernel spans timed with CUDA events on the launching stream.

`KernelTimer` is installed around an epoch (eager or while capturing a CUDA
graph: inside a capture the events become external event nodes, so every
replay re-times them).  Each span carries the kernel's *algorithmic* bytes
(every gathered neighbour row counted, no cache reuse) and its
*compulsory* bytes (each input and output element touched once — the HBM
lower bound the roofline fraction is taken against).
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
    comp_bytes: int = 0


class KernelTimer:
    def __init__(self):
        self.spans: list[Span] = []
        self._pool: list[int] = []

    def _event(self) -> int:
        ev = ctypes.c_void_p()
        _lib.call("gcnb_event_create", ctypes.byref(ev))
        self._pool.append(ev.value)
        return ev.value

    def record(self, name: str, algo_bytes: int, flops: int, stream: int, comp_bytes: int | None = None):
        cap = ctypes.c_int32(0)
        _lib.call("gcnb_stream_is_capturing", stream, ctypes.byref(cap))
        ev0, ev1 = self._event(), self._event()
        _lib.call("gcnb_event_record", ev0, stream, cap.value)
        comp = int(algo_bytes if comp_bytes is None else comp_bytes)
        return Span(name, int(algo_bytes), int(flops), ev0, ev1, comp), cap.value

    def results(self) -> list[tuple[str, int, int, float, int]]:
        """[(name, algo_bytes, flops, ms, compulsory_bytes)] for the last execution (call after a sync)."""
        out = []
        ms = ctypes.c_float(0.0)
        for s in self.spans:
            _lib.call("gcnb_event_elapsed_ms", s.ev0, s.ev1, ctypes.byref(ms))
            out.append((s.name, s.algo_bytes, s.flops, float(ms.value), s.comp_bytes))
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
def span(name: str, algo_bytes: int, flops: int, stream: int, comp_bytes: int | None = None):
    t = _ACTIVE
    if t is None:
        yield
        return
    sp, external = t.record(name, algo_bytes, flops, stream, comp_bytes)
    yield
    _lib.call("gcnb_event_record", sp.ev1, stream, external)
    t.spans.append(sp)
