"""CUDA devices: discovery snapshot, streams, allocation.

Replaces the reference DeviceObject (/root/reference/pkg/src/offloadrt/
device.py:188-367), whose streams are FIFO queues drained by one OS thread
each.  Here a stream id maps to a non-blocking CUDA stream owned by
libofl.so; FIFO order per stream and overlap across streams come from the
hardware, and no host thread sits between the caller and the device.

Kept semantics: stream ids are plain ints, 0 is the default stream and
``create_stream`` hands out 1, 2, ... (device.py:232-233); any id may be
used and is materialised on first use; ``synchronize`` covers the streams
that exist at call time (device.py:316-328).
"""

from __future__ import annotations

import ctypes
import itertools
import os
import threading
from collections import deque
from dataclasses import dataclass
from typing import Optional

from . import _native
from .completion import DeviceToken
from .errors import BadArgsError
from .futures import CompletionToken, make_ready, when_all
from .trace import Tracer

DEFAULT_STREAM = 0


@dataclass(frozen=True)
class DeviceInfo:
    """Discovery snapshot (reference device.py:37-48).  Capability compares
    lexicographically on (major, minor)."""

    name: str
    capability: tuple
    memory_bytes: int
    compute_units: int

    def meets(self, major: int, minor: int) -> bool:
        return tuple(self.capability) >= (major, minor)

    def _key(self) -> tuple:
        return (self.name, tuple(self.capability), self.memory_bytes, self.compute_units)

    # equal to any snapshot with the same fields — the reference's own
    # DeviceInfo included (a daemon's view decoded by the reference's client
    # equals this object, reference tests/test_transport.py:54-59)
    def __eq__(self, other) -> bool:
        try:
            return self._key() == (other.name, tuple(other.capability), other.memory_bytes,
                                   other.compute_units)
        except (AttributeError, TypeError):
            return NotImplemented

    def __hash__(self) -> int:
        return hash(self._key())


@dataclass(frozen=True)
class PhysicalInfo:
    ordinal: int
    product: str
    capability: tuple
    memory_bytes: int
    sms: int
    l2_bytes: int


def query_physical(ordinal: int) -> PhysicalInfo:
    lib = _native.load()
    name = ctypes.create_string_buffer(256)
    major, minor, sms = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    mem, l2 = ctypes.c_uint64(), ctypes.c_uint64()
    _native.check(
        lib.ofl_device_props(
            ordinal, name, 256, ctypes.byref(major), ctypes.byref(minor), ctypes.byref(mem),
            ctypes.byref(sms), ctypes.byref(l2),
        ),
        f"device {ordinal} properties",
    )
    return PhysicalInfo(
        ordinal, name.value.decode(), (major.value, minor.value), mem.value, sms.value, l2.value
    )


def pci_bus_id(ordinal: int) -> str:
    """The GPU's PCI address as sysfs spells it ("0000:1b:00.0")."""
    buf = ctypes.create_string_buffer(64)
    _native.check(_native.load().ofl_device_pci_bus_id(ordinal, buf, 64), "pci bus id")
    return buf.value.decode()


def _cpulist(text: str) -> set:
    cpus: set = set()
    for part in text.strip().split(","):
        if part:
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
    return cpus


def local_cpus(ordinal: int, sysfs: str = "/sys/bus/pci/devices") -> Optional[set]:
    """CPUs of the GPU's NUMA node (sysfs ``local_cpulist``), or None when the
    platform does not say."""
    try:
        with open(os.path.join(sysfs, pci_bus_id(ordinal), "local_cpulist")) as f:
            return _cpulist(f.read()) or None
    except (OSError, ValueError):
        return None


def bind_host_to_device(ordinal: int) -> Optional[dict]:
    """Restrict this process's threads (present and future) to the CPUs
    nearest to GPU `ordinal`, so pinned staging memory allocated afterwards
    lands on that NUMA node and the copy threads run next to its PCIe root
    (one process per GPU on a multi-socket host).  A no-op (None) when the
    GPU's CPUs are unknown or already all we may use."""
    cpus = local_cpus(ordinal)
    if not cpus or not hasattr(os, "sched_setaffinity"):
        return None
    allowed = os.sched_getaffinity(0)
    use = cpus & allowed
    if not use or use == allowed:
        return None
    for tid in os.listdir("/proc/self/task"):
        try:
            os.sched_setaffinity(int(tid), use)
        except OSError:
            pass  # a thread that exited meanwhile
    return {"pci_bus_id": pci_bus_id(ordinal), "cpus": len(use), "of": len(allowed)}


class Stream:
    """One CUDA stream plus host objects that must outlive its in-flight
    operations (pinned sources, staging blocks)."""

    __slots__ = ("ptr", "lib", "device", "sid", "_keep", "_purge_lock", "err_slots")

    def __init__(self, device: "DeviceObject", sid: int):
        self.lib = _native.load()
        self.device = device
        self.sid = sid
        self._purge_lock = threading.Lock()
        p = ctypes.c_void_p()
        _native.check(self.lib.ofl_stream_create(device.ordinal, ctypes.byref(p)), "stream create")
        self.ptr = p.value
        self._keep: deque = deque()
        self.err_slots = None  # jit._ErrSlots, created on the first NVRTC launch

    def done_ticket(self) -> int:
        return self.lib.ofl_stream_done(self.ptr)

    def wait_ticket(self, ticket: int) -> int:
        """Block until `ticket` completed; returns the C status."""
        fast = _native._fast
        if fast is not None:
            return fast.wait(self.ptr, ticket)
        return self.lib.ofl_wait(self.ptr, ticket)

    def error(self, status: int) -> Exception:
        return _native.error_for(status, f"{self.device.info.name} stream {self.sid}")

    def query_ticket(self, ticket: int) -> bool:
        fast = _native._fast
        if fast is not None:
            return fast.query(self.ptr, ticket) > 0
        ready = ctypes.c_int(0)
        status = self.lib.ofl_query(self.ptr, ticket, ctypes.byref(ready))
        return bool(ready.value) and not status

    def tail(self) -> int:
        return self.lib.ofl_stream_tail(self.ptr)

    def keep(self, ticket: int, release) -> None:
        """Hold `release` (an object, or a callable run on release) until the
        stream has completed `ticket`."""
        keep = self._keep
        keep.append((ticket, release))
        if len(keep) & 15 == 0:
            self.purge()

    def purge(self) -> None:
        keep = self._keep
        if not keep:
            return
        released = []
        with self._purge_lock:  # check-then-pop must not interleave
            done = self.lib.ofl_stream_done(self.ptr)
            if keep[0][0] > done and len(keep) > 256:
                # long pipelines without observers: advance the watermark
                ready = ctypes.c_int(0)
                self.lib.ofl_query(self.ptr, keep[0][0], ctypes.byref(ready))
                done = self.lib.ofl_stream_done(self.ptr)
            while keep and keep[0][0] <= done:
                released.append(keep.popleft()[1])
        for rel in released:
            if callable(rel):
                rel()

    def token(self, ticket: int, finish=None) -> DeviceToken:
        return DeviceToken(self, ticket, finish)

    def tail_token(self) -> CompletionToken:
        t = self.tail()
        return DeviceToken(self, t) if t else make_ready(None)

    def destroy(self) -> None:
        if self.ptr:
            self.lib.ofl_stream_destroy(self.ptr)  # synchronises the stream first
            self.ptr = None
            while self._keep:
                _, rel = self._keep.popleft()
                if callable(rel):
                    rel()
            slots, self.err_slots = self.err_slots, None
            if slots is not None:
                slots.free()


class DeviceObject:
    """One logical device of a Runtime, bound to a physical CUDA ordinal."""

    def __init__(self, info: DeviceInfo, physical: PhysicalInfo, record_events: bool = False):
        self.info = info
        self.physical = physical
        self.ordinal = physical.ordinal
        self.backend = "cuda"
        self.record_events = record_events
        self.tracer = Tracer(self) if record_events else None
        self._lock = threading.Lock()
        self._streams: dict[int, Stream] = {}
        self._stream_ids = itertools.count(1)
        self._allocated = 0
        self._closed = False

    # -- streams -------------------------------------------------------------
    def create_stream(self) -> int:
        return next(self._stream_ids)

    def stream(self, sid: int) -> Stream:
        s = self._streams.get(sid)
        if s is not None:
            return s
        if not isinstance(sid, int) or isinstance(sid, bool) or sid < 0:
            raise BadArgsError(f"invalid stream id {sid!r}")
        with self._lock:
            s = self._streams.get(sid)
            if s is None:
                if self._closed:
                    raise BadArgsError(f"{self.info.name} is closed")
                s = Stream(self, sid)
                self._streams[sid] = s
        return s

    def synchronize(self) -> CompletionToken:
        """Completes when everything enqueued so far on every existing stream
        has completed (streams created later are not covered)."""
        with self._lock:
            streams = list(self._streams.values())
        return when_all([s.tail_token() for s in streams])

    # -- memory ----------------------------------------------------------------
    def allocate(self, size: int, shareable: bool = False) -> int:
        """Zero-filled device memory: from the stream-ordered pool, or (for
        buffers exported to other processes through CUDA IPC) cudaMalloc."""
        lib = _native.load()
        p = ctypes.c_void_p()
        alloc = lib.ofl_malloc_shareable if shareable else lib.ofl_malloc
        status = alloc(self.ordinal, size, ctypes.byref(p))
        if status:
            raise _native.error_for(status, f"{self.info.name}: allocation of {size} bytes")
        with self._lock:
            self._allocated += size
        return p.value

    def release(self, ptr: int, size: int) -> None:
        try:
            _native.load().ofl_free(self.ordinal, ptr)
        finally:
            with self._lock:
                self._allocated -= size

    @property
    def allocated_bytes(self) -> int:
        return self._allocated

    def trim_memory(self) -> None:
        """Return the memory released buffers still hold to the device (waits
        for frees queued behind in-flight work; ofl_trim_memory)."""
        _native.check(_native.load().ofl_trim_memory(self.ordinal), "trim memory")

    def event_log(self) -> list:
        """Traced operations (Runtime(record_events=True)); empty otherwise."""
        return self.tracer.event_log() if self.tracer is not None else []

    def close(self) -> None:
        with self._lock:
            streams = list(self._streams.values())
            self._streams.clear()
            self._closed = True
        for s in streams:
            s.destroy()


def physical_devices() -> list[PhysicalInfo]:
    n = _native.device_count()
    return [query_physical(i) for i in range(n)]


def describe(index: int, phys: PhysicalInfo, name: Optional[str] = None) -> DeviceInfo:
    return DeviceInfo(name or f"cuda{index}", phys.capability, phys.memory_bytes, phys.sms)
