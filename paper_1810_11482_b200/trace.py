"""Optional per-operation tracing (``Runtime(record_events=True)``).

Mirrors the reference's event log (/root/reference/pkg/src/offloadrt/
device.py:71-83,330-350: ``EventRecord`` + ``DeviceObject.event_log()``)
with device time: every traced op is bracketed by two CUDA timing events on
its stream; ``event_log()`` resolves them to milliseconds since the device's
first traced op.  Engines are named ``"<device>-s<stream>"`` like the
reference's stream worker threads.  Off by default — tracing adds two event
records per operation.
"""

from __future__ import annotations

import ctypes
import itertools
import threading
from dataclasses import dataclass, field

from . import _native


@dataclass
class EventRecord:
    """One executed operation, as seen by its device."""

    seq: int
    device: str
    op: str  # 'write' | 'read' | 'run' | 'copy'
    stream: int
    engine: str
    start: float  # ms since the first traced op on this device
    end: float
    amount: int = 0  # bytes for copies, work items for kernels
    meta: dict = field(default_factory=dict)


class Tracer:
    def __init__(self, device):
        self.device = device
        self._lock = threading.Lock()
        self._seq = itertools.count()
        self._base = None
        self._pending: list = []
        self._done: list = []

    def _event(self) -> ctypes.c_void_p:
        e = ctypes.c_void_p()
        _native.check(_native.load().ofl_event_create(self.device.ordinal, ctypes.byref(e)), "trace event")
        return e

    def begin(self, stream) -> ctypes.c_void_p:
        lib = _native.load()
        with self._lock:
            if self._base is None:
                self._base = self._event()
                lib.ofl_event_record(self._base, stream.ptr)
        e = self._event()
        lib.ofl_event_record(e, stream.ptr)
        return e

    def end(self, stream, start_event, op: str, amount: int = 0, meta=None) -> None:
        e = self._event()
        _native.load().ofl_event_record(e, stream.ptr)
        with self._lock:
            self._pending.append((next(self._seq), op, stream.sid, start_event, e, amount, meta or {}))

    def event_log(self) -> list:
        """Records of every traced op so far (waits for them to finish)."""
        lib = _native.load()
        with self._lock:
            pending, self._pending = self._pending, []
            base = self._base
        ms = ctypes.c_float()
        name = self.device.info.name
        for seq, op, sid, e0, e1, amount, meta in pending:
            lib.ofl_event_elapsed_ms(base, e0, ctypes.byref(ms))
            t0 = ms.value
            lib.ofl_event_elapsed_ms(base, e1, ctypes.byref(ms))
            self._done.append(EventRecord(seq, name, op, sid, f"{name}-s{sid}", t0, ms.value,
                                          amount, meta))
            lib.ofl_event_destroy(e0)
            lib.ofl_event_destroy(e1)
        with self._lock:
            return sorted(self._done, key=lambda r: r.seq)
