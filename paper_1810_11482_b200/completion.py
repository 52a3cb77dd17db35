"""Tokens for stream-ordered device operations, and the completion thread.

Replaces the reference's per-stream worker threads that fulfil promises
after running each operation (/root/reference/pkg/src/offloadrt/device.py:
129-157, futures.py:76-89).  Here the device runs the operation; the token
only records *where* on which stream it sits (a ticket, include/ofl.h), and
completion is observed on demand:

* ``done()``  -> ``ofl_query``  (cudaEventQuery on a lazily placed marker)
* ``get()``   -> ``ofl_wait``   (cudaEventSynchronize; no thread handoff)
* ``then()``  -> ``ofl_notify`` (cudaLaunchHostFunc pushes the token id into
  a queue and signals an eventfd; one completion thread blocked in
  ``os.read`` drains ids in batches and fulfils the tokens — no polling)

A token may carry a ``finish`` function run exactly once when the operation
is known complete (e.g. turning a pinned staging block into the ``bytes``
the reference's ``enqueue_read`` returns); an exception from it fails the
token, which is how host-side post-conditions surface.
"""

from __future__ import annotations

import ctypes
import itertools
import os
import select
import threading
import time
from typing import Any, Callable, Optional

from . import _native
from .errors import InternalError
from .futures import _PENDING, _READY, DEVICE_TOKEN_TYPES, CompletionToken, _lock

_ids = itertools.count(1)
_pending: dict[int, "DeviceToken"] = {}
_pending_lock = threading.Lock()
_thread: Optional[threading.Thread] = None
_thread_lock = threading.Lock()


# With nothing completing for this long, the completion thread checks the
# streams of the tokens it waits for: a sticky device fault stops the CUDA
# host-function callbacks, so without this a then() on a faulted stream
# would never fire.  Idle-time only — busy streams are never polled.
WATCHDOG_S = 1.0


def _watchdog() -> None:
    with _pending_lock:
        items = list(_pending.items())
    for tid, tok in items:
        if tok._state == _PENDING:
            tok._poll()  # ofl_query: a fault fails the token (and its continuations)
        if tok._state != _PENDING:
            with _pending_lock:
                _pending.pop(tid, None)


def _completion_loop(fd: int) -> None:
    lib = _native.load()
    cap = 1024
    buf = (ctypes.c_uint64 * cap)()
    count = ctypes.c_int(0)
    while True:
        try:
            ready, _, _ = select.select([fd], [], [], WATCHDOG_S)
            if not ready:
                if _pending:
                    _watchdog()
                continue
            os.read(fd, 8)
        except InterruptedError:
            continue
        while True:
            lib.ofl_drain(buf, cap, ctypes.byref(count))
            n = count.value
            if n == 0:
                break
            with _pending_lock:
                toks = [_pending.pop(buf[i], None) for i in range(n)]
            for tok in toks:
                if tok is not None:
                    try:
                        tok._finish_now()
                    except BaseException:  # noqa: BLE001 - a raw callback raised;
                        pass  # the thread must survive to complete other tokens


def _ensure_thread() -> None:
    global _thread
    if _thread is not None:
        return
    with _thread_lock:
        if _thread is None:
            fd = _native.load().ofl_completion_fd()
            if fd < 0:
                raise InternalError("completion eventfd unavailable")
            t = threading.Thread(
                target=_completion_loop, args=(fd,), name="ofl-completion", daemon=True
            )
            t.start()
            _thread = t


class DeviceToken(CompletionToken):
    """Token of one stream-ordered operation: (stream, ticket)."""

    __slots__ = ("_stream", "_ticket", "_finish", "_claimed")

    def __init__(self, stream, ticket: int, finish: Optional[Callable[[], Any]] = None):
        # CompletionToken.__init__ inlined: this runs once per device op
        self._state = _PENDING
        self._value = None
        self._error = None
        self._callbacks = None
        self._stream = stream
        self._ticket = ticket
        self._finish = finish
        self._claimed = False

    def _finish_now(self) -> None:
        """The operation is complete on the device: produce the value.
        Exactly one caller runs ``finish``; the others return at once."""
        with _lock:
            if self._state != _PENDING or self._claimed:
                return
            self._claimed = True
            fin = self._finish
            if fin is None:  # no host-side work: complete under the same lock
                self._state = _READY
                callbacks = self._callbacks
                self._callbacks = None
            else:
                self._finish = None
        if fin is None:
            if callbacks:
                for cb in callbacks:
                    cb(self)
            return
        try:
            value = fin()
        except BaseException as exc:  # noqa: BLE001 - delivered through the token
            self._try_complete(error=exc)
            return
        self._try_complete(value=value)

    def _group_key(self):
        return (self._stream, self._ticket)

    def _fail(self, status: int, what: str) -> None:
        with _lock:
            if self._claimed:
                return
            self._claimed = True
            self._finish = None
        self._try_complete(error=_native.error_for(status, what))

    def _poll(self) -> bool:
        if self._state != _PENDING:
            return True
        s = self._stream
        fast = _native._fast
        if fast is not None:  # ofl_query checks the done watermark first
            r = fast.query(s.ptr, self._ticket)
            if r < 0:
                self._fail(-r, "device operation failed")
                return True
            if not r:
                return False
        elif s.done_ticket() < self._ticket:
            ready = ctypes.c_int(0)
            status = s.lib.ofl_query(s.ptr, self._ticket, ctypes.byref(ready))
            if status:
                self._fail(status, "device operation failed")
                return True
            if not ready.value:
                return False
        self._finish_now()
        return self._state != _PENDING

    def _block(self, timeout: Optional[float]) -> bool:
        if self._state != _PENDING:
            return True
        if timeout is not None:
            # wait for the completion callback in slices, querying the stream
            # in between so that a device fault (which stops callbacks)
            # surfaces as an error instead of a timeout
            event = threading.Event()
            self._on_done(lambda _t: event.set())
            deadline = time.monotonic() + timeout
            while True:
                left = deadline - time.monotonic()
                if event.wait(min(0.05, max(left, 0.0))) or self._poll():
                    return True
                if left <= 0:
                    return False
        s = self._stream
        fast = _native._fast
        if fast is not None:
            status = fast.wait(s.ptr, self._ticket)
        else:
            status = s.lib.ofl_wait(s.ptr, self._ticket)
        if status:
            self._fail(status, "device operation failed")
        else:
            self._finish_now()
        if self._state == _PENDING:  # another thread is running finish()
            self._wait_quiet(None)
        return True

    def _arm(self) -> None:
        _ensure_thread()
        tid = next(_ids)
        with _pending_lock:
            _pending[tid] = self
        s = self._stream
        status = s.lib.ofl_notify(s.ptr, self._ticket, tid)
        if status:
            with _pending_lock:
                _pending.pop(tid, None)
            self._fail(status, "completion notify failed")


class PipelinedToken(DeviceToken):
    """Device token whose ``finish`` itself waits for the operation, piece by
    piece: a chunked read (``ofl_collect`` waits for each chunk's event and
    copies it out while the later chunks are still on the link).  ``get()``
    starts the finish at once instead of first waiting for the whole
    operation, so the host copies overlap the DMA; the finish fails the
    token if the device faulted (the chunk events report it)."""

    __slots__ = ()

    def _block(self, timeout: Optional[float]) -> bool:
        if self._state != _PENDING:
            return True
        if timeout is not None:
            return DeviceToken._block(self, timeout)
        self._finish_now()
        if self._state == _PENDING:  # another thread is running finish()
            self._wait_quiet(None)
        return True


DEVICE_TOKEN_TYPES.add(DeviceToken)
DEVICE_TOKEN_TYPES.add(PipelinedToken)
