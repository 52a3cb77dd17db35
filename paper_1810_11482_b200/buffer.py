"""Device-resident buffers.

Replaces the reference BufferObject (/root/reference/pkg/src/offloadrt/
buffer.py:22-66): untyped bytes, zero-initialised at creation, every access
bounds-checked against [0, size).  The bytes live in HBM (cudaMalloc); writes
and reads are stream-ordered cudaMemcpyAsync (see hostmem.py for the host
side of each copy); kernels see typed views by pointer + element count.
"""

from __future__ import annotations

import ctypes
import threading

from . import _native, hostmem
from .completion import DeviceToken, PipelinedToken
from .device import DeviceObject
from .errors import BadArgsError, OobAccessError
from .futures import CompletionToken, make_ready
from .bindings import ticket_slot as _ticket_slot

ELEM_SIZE = {"buffer_f64": 8, "buffer_u32": 4, "buffer_f32": 4}


def check_range(offset: int, size: int, total: int, what: str) -> None:
    if offset < 0 or size < 0:
        raise BadArgsError(f"{what}: negative offset or size")
    if offset + size > total:
        raise OobAccessError(
            f"{what}: range [{offset}, {offset + size}) exceeds buffer of {total} bytes"
        )


class BufferObject:
    """Owning-side buffer: a device allocation and the device whose streams
    order access to it."""

    __slots__ = ("device", "size_bytes", "ptr", "__weakref__")

    def __init__(self, device: DeviceObject, size_bytes: int, shareable: bool = False):
        if size_bytes <= 0:
            raise BadArgsError("buffer size must be positive")
        self.device = device
        self.size_bytes = size_bytes
        self.ptr = 0
        self.ptr = device.allocate(size_bytes, shareable)

    def __del__(self):
        if self.ptr:
            try:
                self.device.release(self.ptr, self.size_bytes)
            except Exception:  # noqa: BLE001 - interpreter teardown
                pass
            self.ptr = 0

    def elements(self, kind: str) -> int:
        """Element count of the typed view; a tail shorter than one element
        is unaddressable (reference buffer.py:57-66)."""
        try:
            return self.size_bytes // ELEM_SIZE[kind]
        except KeyError:
            raise BadArgsError(f"not a buffer kind: {kind}") from None

    # -- copies ------------------------------------------------------------------
    def enqueue_write(self, offset: int, data, stream: int = 0) -> CompletionToken:
        addr, n, owner = hostmem.host_view(data)
        if offset < 0 or offset + n > self.size_bytes:
            check_range(offset, n, self.size_bytes, "write")
        dev = self.device
        st = dev._streams.get(stream) or dev.stream(stream)
        lib = st.lib
        ticket = _ticket_slot()
        dst = self.ptr + offset
        if n == 0 or type(owner) is hostmem.PinnedArray or hostmem.is_pinned(addr, n):
            fast = _native._fast
            if fast is not None:
                t = fast.h2d(st.ptr, dst, addr, n)
                if t < 0:
                    raise_status(-t, "write")
                if n:
                    st.keep(t, owner)
                return DeviceToken(st, t)
            status = lib.ofl_h2d(st.ptr, dst, addr, n, ctypes.byref(ticket))
            if status:
                raise_status(status, "write")
            if n:
                st.keep(ticket.value, owner)
        elif n <= hostmem.SMALL_PAGEABLE:
            # the driver stages pageable data before returning
            status = lib.ofl_h2d(st.ptr, dst, addr, n, ctypes.byref(ticket))
            if status:
                raise_status(status, "write")
        else:
            # pipelined multi-threaded staging in libofl (csrc/ofl_staging.cu)
            status = lib.ofl_h2d_pageable(st.ptr, dst, addr, n, ctypes.byref(ticket))
            if status:
                raise_status(status, "write")
        return DeviceToken(st, ticket.value)

    def write_pinned(self, offset: int, data, stream: int = 0) -> CompletionToken:
        """enqueue_write of a ``pinned_empty`` array (zero-copy DMA): the
        handles' fast path, range already checked by the handle."""
        fast = _native._fast
        if fast is None or not data.flags.c_contiguous:
            return self.enqueue_write(offset, data, stream)
        n = data.nbytes
        dev = self.device
        st = dev._streams.get(stream) or dev.stream(stream)
        t = fast.h2d(st.ptr, self.ptr + offset, data._address(), n)
        if t < 0:
            raise_status(-t, "write")
        if n:
            st.keep(t, data)
        return DeviceToken(st, t)

    def enqueue_read(self, offset: int, size: int, stream: int = 0) -> CompletionToken:
        """Token for the bytes of [offset, offset+size) at this stream position."""
        check_range(offset, size, self.size_bytes, "read")
        if size == 0:
            return make_ready(b"")
        st = self.device.stream(stream)
        if size >= hostmem.CHUNKED_READ:
            return self._read_chunked(st, offset, size, None)
        block = hostmem.pool.get(size)
        ticket = ctypes.c_uint64()
        status = st.lib.ofl_d2h(st.ptr, block.addr, self.ptr + offset, size, ctypes.byref(ticket))
        if status:
            hostmem.pool.put(block)
            raise_status(status, "read")
        landing = _Landing(block, size)
        tok = DeviceToken(st, ticket.value, landing.take)
        # the block goes back to the pool only after the copy completed and
        # its bytes were taken (or the token was dropped unobserved)
        st.keep(ticket.value, landing.release_later)
        return tok

    def enqueue_read_into(self, offset: int, out, stream: int = 0) -> CompletionToken:
        """Copy [offset, offset+len(out)) into the writable host buffer `out`
        at this stream position.  Zero-copy when `out` is pinned
        (hostmem.pinned_empty).  The token's value is `out`."""
        addr, n, owner = hostmem.writable_view(out)
        check_range(offset, n, self.size_bytes, "read")
        st = self.device.stream(stream)
        ticket = ctypes.c_uint64()
        if n == 0:
            return make_ready(out)
        if hostmem.is_pinned(addr, n):
            status = st.lib.ofl_d2h(st.ptr, addr, self.ptr + offset, n, ctypes.byref(ticket))
            if status:
                raise_status(status, "read")
            st.keep(ticket.value, owner)
            return DeviceToken(st, ticket.value, lambda: out)
        if n >= hostmem.CHUNKED_READ:
            return self._read_chunked(st, offset, n, (addr, owner, out))
        block = hostmem.pool.get(n)
        status = st.lib.ofl_d2h(st.ptr, block.addr, self.ptr + offset, n, ctypes.byref(ticket))
        if status:
            hostmem.pool.put(block)
            raise_status(status, "read")
        landing = _Landing(block, n, into=addr, keep=owner)
        st.keep(ticket.value, landing.release_later)
        return DeviceToken(st, ticket.value, lambda: (landing.take(), out)[1])

    def _read_chunked(self, st, offset: int, n: int, into) -> CompletionToken:
        """Large read to pageable memory: chunked D2H into a pinned staging
        block (one event per chunk); the token's finish step copies each
        chunk out on the copy threads as soon as it lands (ofl_collect), into
        a new ``bytes`` (into=None) or into the caller's buffer."""
        block = hostmem.pool.get(n)
        handle = ctypes.c_void_p()
        ticket = ctypes.c_uint64()
        status = st.lib.ofl_d2h_chunked(st.ptr, block.addr, self.ptr + offset, n,
                                        hostmem.READ_CHUNK, ctypes.byref(handle),
                                        ctypes.byref(ticket))
        if status:
            hostmem.pool.put(block)
            raise_status(status, "read")
        landing = _ChunkedLanding(st.lib, block, n, handle.value, into)
        st.keep(ticket.value, landing.release_later)
        return PipelinedToken(st, ticket.value, landing.take)

    def enqueue_read_rows_into(self, offset: int, out, row_bytes: int, rows: int,
                               dst_offset: int, dst_pitch: int, stream: int = 0):
        """Copy `rows` consecutive rows of `row_bytes` starting at `offset`
        into the pinned host buffer `out`, row i at byte dst_offset +
        i*dst_pitch (one strided DMA; cudaMemcpy2DAsync).  Token value: out."""
        addr, n, owner = hostmem.writable_view(out)
        span = rows * row_bytes
        check_range(offset, span, self.size_bytes, "read")
        if rows and (dst_pitch < row_bytes or dst_offset < 0
                     or dst_offset + (rows - 1) * dst_pitch + row_bytes > n):
            raise BadArgsError("row read does not fit the destination")
        if span == 0:
            return make_ready(out)
        if not hostmem.is_pinned(addr, n):
            raise BadArgsError("enqueue_read_rows_into needs a pinned destination (pinned_empty)")
        st = self.device.stream(stream)
        ticket = ctypes.c_uint64()
        status = st.lib.ofl_d2h_rows(st.ptr, addr + dst_offset, dst_pitch, self.ptr + offset,
                                     row_bytes, rows, ctypes.byref(ticket))
        if status:
            raise_status(status, "read")
        st.keep(ticket.value, owner)
        return DeviceToken(st, ticket.value, lambda: out)


class _Landing:
    """A staging block receiving a device->host copy.  `take` (after
    completion) extracts the data; the block is recycled once both the copy
    is complete (stream purge) and the data has been taken."""

    __slots__ = ("block", "size", "into", "keep_obj", "data", "taken", "purged", "lock")

    def __init__(self, block, size: int, into: int = 0, keep=None):
        self.lock = threading.Lock()
        self.block = block
        self.size = size
        self.into = into
        self.keep_obj = keep
        self.data = None
        self.taken = False
        self.purged = False

    def _extract(self):
        if self.into:
            hostmem.memcpy(self.into, self.block.addr, self.size)
            return None
        return hostmem.bytes_from(self.block.addr, self.size)

    def take(self):
        # only called once the copy is complete (token finish), so the block
        # can go back to the pool right away
        with self.lock:
            if not self.taken:
                self.data = self._extract()
                self.taken = True
            self._recycle()
            data, self.data = self.data, None
        return data

    def release_later(self):
        # copy is complete; if nobody took the data yet, keep the block until
        # they do (the token holds this landing through its finish function)
        with self.lock:
            self.purged = True
            if self.taken:
                self._recycle()

    def _recycle(self):
        if self.block is not None:
            hostmem.pool.put(self.block)
            self.block = None

    def __del__(self):
        # token dropped unobserved after the copy completed
        if self.block is not None and self.purged:
            try:
                hostmem.pool.put(self.block)
            except Exception:  # noqa: BLE001
                pass


class _ChunkedLanding:
    """A chunked read in flight (ofl_d2h_chunked): `take` collects it (waits
    for each chunk, copies it out in parallel) and recycles the staging
    block; dropped unobserved, the handle and block are released once the
    stream has passed the read."""

    __slots__ = ("lib", "block", "size", "handle", "into", "lock", "taken", "purged")

    def __init__(self, lib, block, size: int, handle: int, into):
        self.lib, self.block, self.size, self.handle, self.into = lib, block, size, handle, into
        self.lock = threading.Lock()
        self.taken = False
        self.purged = False

    def take(self):
        with self.lock:
            if self.taken:
                raise RuntimeError("read collected twice")
            self.taken = True
            try:
                if self.into is None:
                    fast = _native._fast
                    if fast is not None:
                        out = fast.collect_bytes(self.handle, self.size)
                        if type(out) is int:
                            raise_status(-out, "read")
                        return out
                    out = bytearray(self.size)
                    raw = (ctypes.c_char * self.size).from_buffer(out)
                    status = self.lib.ofl_collect(self.handle, ctypes.addressof(raw))
                    del raw
                    if status:
                        raise_status(status, "read")
                    return bytes(out)
                addr, _owner, result = self.into
                status = self.lib.ofl_collect(self.handle, addr)
                if status:
                    raise_status(status, "read")
                return result
            finally:
                self._release()

    def release_later(self):
        with self.lock:
            self.purged = True
            if not self.taken:
                return  # the token's finish step will collect it
            self._release()

    def _release(self):
        if self.handle:
            self.lib.ofl_read_release(self.handle)
            self.handle = 0
        if self.block is not None:
            hostmem.pool.put(self.block)
            self.block = None

    def __del__(self):
        # token dropped unobserved after the copy completed
        if self.handle and self.purged:
            try:
                self._release()
            except Exception:  # noqa: BLE001
                pass


def raise_status(status: int, what: str):
    from . import _native

    raise _native.error_for(status, what)
