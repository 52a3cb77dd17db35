"""Pinned host memory: user-visible pinned arrays and the staging pool.

The reference copies host data three times per write (handles.py:88,
buffer.py:42,44-45 of /root/reference/pkg/src/offloadrt).  Here a write is:

* zero-copy DMA when the source lies in pinned memory this runtime handed out
  (``pinned_empty``) — the array is kept alive until the copy completes;
* a direct ``cudaMemcpyAsync`` from pageable memory for small payloads (the
  driver stages them before the call returns, so the caller may reuse them);
* one host copy into a pinned staging block, then an async DMA, for large
  pageable payloads (the block returns to the pool once the copy is done).

Reads land in pinned memory (staging block or a pinned user array), because
a device->pageable copy would block the calling thread.
"""

from __future__ import annotations

import bisect
import ctypes
import threading
import weakref
from typing import Optional

import numpy as np

from . import _native

SMALL_PAGEABLE = 256 * 1024  # below this, let the driver stage pageable data
CHUNKED_READ = 4 << 20       # reads to pageable memory from this size: chunked, collected in parallel
READ_CHUNK = 8 << 20         # D2H piece of a chunked read
_MIN_CLASS = 4096

_ranges_lock = threading.Lock()
# (starts, ends) of the pinned allocations, sorted; replaced as a whole under
# the lock (copy on write), so a lookup reads one consistent pair without it
_ranges: tuple = ((), ())


def _register_range(start: int, size: int) -> None:
    global _ranges
    with _ranges_lock:
        starts, ends = list(_ranges[0]), list(_ranges[1])
        i = bisect.bisect_left(starts, start)
        starts.insert(i, start)
        ends.insert(i, start + size)
        _ranges = (tuple(starts), tuple(ends))


def _unregister_range(start: int) -> None:
    global _ranges
    with _ranges_lock:
        starts, ends = list(_ranges[0]), list(_ranges[1])
        i = bisect.bisect_left(starts, start)
        if i < len(starts) and starts[i] == start:
            del starts[i]
            del ends[i]
            _ranges = (tuple(starts), tuple(ends))


def is_pinned(addr: int, size: int) -> bool:
    """True if [addr, addr+size) lies inside one pinned allocation."""
    starts, ends = _ranges
    if not starts:
        return False
    i = bisect.bisect_right(starts, addr) - 1
    return i >= 0 and addr + size <= ends[i]


def _host_alloc(nbytes: int) -> int:
    lib = _native.load()
    p = ctypes.c_void_p()
    _native.check(lib.ofl_host_alloc(max(1, nbytes), ctypes.byref(p)), "pinned allocation")
    return p.value


def _free(addr: int) -> None:
    _unregister_range(addr)
    try:
        _native.load().ofl_host_free(addr)
    except Exception:  # noqa: BLE001 - interpreter teardown
        pass


def _as_array(addr: int, nbytes: int) -> np.ndarray:
    buf = (ctypes.c_uint8 * nbytes).from_address(addr)
    return np.frombuffer(buf, dtype=np.uint8)


def pinned_empty(nbytes: int, dtype=np.uint8) -> np.ndarray:
    """A numpy array in page-locked memory.  Writes from / reads into it are
    zero-copy DMA.  Freed when the array (and every view of it) is gone."""
    dtype = np.dtype(dtype)
    count = nbytes // dtype.itemsize if dtype.itemsize else 0
    size = max(1, count * dtype.itemsize)
    addr = _host_alloc(size)
    _register_range(addr, size)
    owner = (ctypes.c_uint8 * size).from_address(addr)
    # every numpy view keeps `owner` alive through its .base chain
    weakref.finalize(owner, _free, addr)
    raw = np.frombuffer(owner, dtype=np.uint8)
    return raw[: count * dtype.itemsize].view(dtype).view(PinnedArray)


class PinnedArray(np.ndarray):
    """ndarray living in page-locked memory from ``pinned_empty``.  Its
    address is looked up once per array object (numpy's own accessors cost
    over a microsecond, which matters on the per-op path)."""

    def __array_finalize__(self, obj):
        self._ofl_addr = None

    def _address(self) -> int:
        addr = getattr(self, "_ofl_addr", None)
        if addr is None:
            addr = self.ctypes.data
            self._ofl_addr = addr
        return addr


def _bytes_data_offset() -> int:
    """Offset of a bytes object's payload from id(obj) (CPython layout),
    verified against ctypes; 0 when the layout is not the expected one."""
    probe = b"offset-probe"
    off = bytes.__basicsize__ - 1
    real = ctypes.cast(ctypes.c_char_p(probe), ctypes.c_void_p).value
    return off if id(probe) + off == real else 0


_BYTES_OFF = _bytes_data_offset()


def pinned_like(src) -> np.ndarray:
    """Pinned copy of an array-like (same dtype and shape)."""
    a = np.ascontiguousarray(src)
    out = pinned_empty(a.nbytes, a.dtype).reshape(a.shape)
    np.copyto(out, a)
    return out


class Block:
    """One reusable pinned staging block."""

    __slots__ = ("addr", "size", "array")

    def __init__(self, addr: int, size: int):
        self.addr = addr
        self.size = size
        self.array = _as_array(addr, size)


class StagingPool:
    """Power-of-two size classes of pinned blocks, reused forever."""

    def __init__(self):
        self._lock = threading.Lock()
        self._free: dict[int, list[Block]] = {}

    @staticmethod
    def _cls(nbytes: int) -> int:
        c = _MIN_CLASS
        while c < nbytes:
            c <<= 1
        return c

    def get(self, nbytes: int) -> Block:
        c = self._cls(nbytes)
        with self._lock:
            lst = self._free.get(c)
            if lst:
                return lst.pop()
        addr = _host_alloc(c)
        return Block(addr, c)

    def put(self, block: Block) -> None:
        with self._lock:
            self._free.setdefault(block.size, []).append(block)


pool = StagingPool()


def host_view(data) -> tuple[int, int, object]:
    """(address, nbytes, owner) of a C-contiguous host buffer; owner keeps the
    memory alive.  Non-buffer objects go through bytes() like the reference's
    BufferHandle.enqueue_write (handles.py:88)."""
    t = type(data)
    if t is bytes:
        n = len(data)
        if n == 0:
            return 0, 0, data
        if _BYTES_OFF:
            return id(data) + _BYTES_OFF, n, data
        return ctypes.cast(ctypes.c_char_p(data), ctypes.c_void_p).value, n, data
    if t is PinnedArray and data.flags.c_contiguous:
        return data._address(), data.nbytes, data
    if isinstance(data, np.ndarray) and data.flags.c_contiguous:
        return data.ctypes.data, data.nbytes, data
    try:
        mv = memoryview(data)
    except TypeError:
        b = bytes(data)
        return host_view(b)
    if not mv.c_contiguous:
        return host_view(mv.tobytes())
    arr = np.frombuffer(mv.cast("B"), dtype=np.uint8) if mv.nbytes else np.zeros(0, np.uint8)
    return (arr.ctypes.data if arr.size else 0), arr.nbytes, arr


def writable_view(out) -> tuple[int, int, object]:
    """(address, nbytes, owner) of a writable C-contiguous host buffer."""
    if type(out) is PinnedArray and out.flags.c_contiguous and out.flags.writeable:
        return out._address(), out.nbytes, out
    if isinstance(out, np.ndarray):
        if not out.flags.c_contiguous or not out.flags.writeable:
            raise ValueError("output array must be C-contiguous and writable")
        return out.ctypes.data, out.nbytes, out
    mv = memoryview(out)
    if mv.readonly or not mv.c_contiguous:
        raise ValueError("output buffer must be C-contiguous and writable")
    arr = np.frombuffer(mv.cast("B"), dtype=np.uint8)
    return (arr.ctypes.data if arr.size else 0), arr.nbytes, arr


def memcpy(dst: int, src: int, nbytes: int) -> None:
    """Host copy; large ones run on libofl's copy threads (GIL released)."""
    if nbytes >= (4 << 20):
        _native.load().ofl_host_memcpy(dst, src, nbytes)
    elif nbytes:
        ctypes.memmove(dst, src, nbytes)


def bytes_from(addr: int, nbytes: int) -> bytes:
    """A new bytes object holding [addr, addr+nbytes): allocated zeroed
    (calloc-backed for large sizes) and filled in place before anyone else
    can see it — one copy, on the copy threads."""
    if nbytes < (4 << 20) or not _BYTES_OFF:
        return ctypes.string_at(addr, nbytes)
    out = bytes(nbytes)
    memcpy(id(out) + _BYTES_OFF, addr, nbytes)
    return out


