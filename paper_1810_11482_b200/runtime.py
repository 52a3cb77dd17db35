"""Runtime wiring: CUDA devices, the registry, and the dispatch seam.

``CudaDispatch`` is the drop-in for the reference's ``LocalDispatch``
(/root/reference/pkg/src/offloadrt/runtime.py:30-120): the same method set
with the same signatures and error convention — resolution and execution
failures come back as failed tokens, synchronous methods raise.  Below it,
instead of per-stream worker threads and numba, sit CUDA streams, HBM
buffers and sm_100a kernels in libofl.so (include/ofl.h).

``Runtime(backend="cuda", devices=...)`` mirrors the reference constructor
(runtime.py:131-159).  ``devices`` is None (every visible GPU), a count, or a
list of CUDA ordinals; several logical devices may share one GPU (useful to
exercise multi-device code paths on a single B200).  There is no CPU
backend: without libofl.so or a CUDA device the constructor raises.
"""

from __future__ import annotations

import ctypes
import os
import weakref
from typing import Optional, Sequence, Union

from . import _native
from .buffer import BufferObject
from .device import DeviceInfo, DeviceObject, describe, physical_devices
from .errors import BadArgsError, InternalError, UnknownGidError
from .futures import CompletionToken, make_failed, make_ready
from .handles import BufferHandle, DeviceHandle, ProgramHandle, copy
from .program import ProgramObject, launch_items
from .registry import GlobalId, LocalityInfo, ObjectKind, Registry

DeviceSpec = Union[int, Sequence[int], None]


class CudaDispatch:
    """Executes operations on objects owned by this process's CUDA devices."""

    def __init__(self, registry: Registry):
        self._registry = registry
        self._objects = registry._objects  # hot-path lookups

    @staticmethod
    def _tokenized(fn) -> CompletionToken:
        try:
            return fn()
        except Exception as exc:  # noqa: BLE001 - delivered through the token
            return make_failed(exc)

    def _device(self, gid: GlobalId) -> DeviceObject:
        return self._registry.resolve_local(gid, ObjectKind.DEVICE)

    def _buffer(self, gid: GlobalId) -> BufferObject:
        obj = self._objects.get(gid)
        if obj is None or gid.kind != ObjectKind.BUFFER:
            return self._registry.resolve_local(gid, ObjectKind.BUFFER)
        return obj

    def _program(self, gid: GlobalId) -> ProgramObject:
        obj = self._objects.get(gid)
        if obj is None or gid.kind != ObjectKind.PROGRAM:
            return self._registry.resolve_local(gid, ObjectKind.PROGRAM)
        return obj

    # -- devices -------------------------------------------------------------
    def device_info(self, device_gid: GlobalId) -> CompletionToken:
        return self._tokenized(lambda: make_ready(self._device(device_gid).info))

    def create_stream(self, device_gid: GlobalId) -> int:
        return self._device(device_gid).create_stream()

    def synchronize(self, device_gid: GlobalId) -> CompletionToken:
        return self._tokenized(lambda: self._device(device_gid).synchronize())

    # -- buffers -------------------------------------------------------------
    def create_buffer(self, device_gid: GlobalId, size: int, shareable: bool = False) -> CompletionToken:
        """`shareable` (extension): a buffer another process can map through
        CUDA IPC (collectives.ProcessPeerGroup, bench.ProcessHeatSlabs)."""
        def start():
            device = self._device(device_gid)
            buf = BufferObject(device, size, shareable)
            return make_ready(self._registry.register(ObjectKind.BUFFER, buf))

        return self._tokenized(start)

    @staticmethod
    def _traced(dev, stream, op, amount, fn):
        """Run one enqueue, bracketed by trace events when the device records
        events (Runtime(record_events=True); reference device.py:330-350)."""
        tr = dev.tracer
        if tr is None:
            return fn()
        st = dev.stream(stream)
        e0 = tr.begin(st)
        tok = fn()
        tr.end(st, e0, op, amount)
        return tok

    def write(self, buffer_gid, offset, data, stream, device=None) -> CompletionToken:
        try:
            buf = self._buffer(buffer_gid)
            if buf.device.tracer is None:
                return buf.enqueue_write(offset, data, stream)
            n = memoryview(data).nbytes if not isinstance(data, bytes) else len(data)
            return self._traced(buf.device, stream, "write", n,
                                lambda: buf.enqueue_write(offset, data, stream))
        except Exception as exc:  # noqa: BLE001
            return make_failed(exc)

    def read(self, buffer_gid, offset, size, stream, device=None) -> CompletionToken:
        try:
            buf = self._buffer(buffer_gid)
            return self._traced(buf.device, stream, "read", size,
                                lambda: buf.enqueue_read(offset, size, stream))
        except Exception as exc:  # noqa: BLE001
            return make_failed(exc)

    def read_rows_into(self, buffer_gid, offset, out, row_bytes, rows, dst_offset, dst_pitch,
                       stream, device=None) -> CompletionToken:
        try:
            buf = self._buffer(buffer_gid)
            return self._traced(buf.device, stream, "read", rows * row_bytes,
                                lambda: buf.enqueue_read_rows_into(offset, out, row_bytes, rows,
                                                                   dst_offset, dst_pitch, stream))
        except Exception as exc:  # noqa: BLE001
            return make_failed(exc)

    def read_into(self, buffer_gid, offset, out, stream, device=None) -> CompletionToken:
        try:
            buf = self._buffer(buffer_gid)
            return self._traced(buf.device, stream, "read", memoryview(out).nbytes,
                                lambda: buf.enqueue_read_into(offset, out, stream))
        except Exception as exc:  # noqa: BLE001
            return make_failed(exc)

    def copy(self, src_gid, src_off, dst_gid, dst_off, size) -> CompletionToken:
        """Device-side copy on the default streams: the copy runs on the
        source's stream after the destination stream's prior work, and the
        destination stream waits for it (no host round trip)."""

        def start():
            src = self._buffer(src_gid)
            dst = self._buffer(dst_gid)
            s_st = src.device.stream(0)
            d_st = dst.device.stream(0)
            lib = s_st.lib
            d_tail = d_st.tail()
            if d_tail:
                _native.check(lib.ofl_stream_wait(s_st.ptr, d_st.ptr, d_tail), "copy ordering")
            ticket = ctypes.c_uint64()
            _native.check(
                lib.ofl_p2p(
                    s_st.ptr, dst.ptr + dst_off, dst.device.ordinal, src.ptr + src_off,
                    src.device.ordinal, size, ctypes.byref(ticket),
                ),
                "copy",
            )
            if d_st is not s_st:
                _native.check(lib.ofl_stream_wait(d_st.ptr, s_st.ptr, ticket.value), "copy ordering")
            return s_st.token(ticket.value)

        return self._tokenized(start)

    # -- programs --------------------------------------------------------------
    def create_program(self, device_gid: GlobalId, source: str) -> CompletionToken:
        def start():
            program = ProgramObject(self._device(device_gid), source)
            return make_ready(self._registry.register(ObjectKind.PROGRAM, program))

        return self._tokenized(start)

    def build(self, program_gid: GlobalId, kernel_name: str) -> CompletionToken:
        return self._tokenized(lambda: self._program(program_gid).build(kernel_name))

    def run(self, program_gid, kernel_name, grid, block, stream, args, device=None, items=None):
        """`items` may be passed by a caller that already validated the
        launch shape (the handle does); otherwise it is derived here."""
        try:
            program = self._program(program_gid)
            if items is None:
                items = launch_items(grid, block)
            # buffer gids are resolved in the same pass as the kind checks
            if program.device.tracer is None:
                return program.run(kernel_name, items, stream, args, grid, block, self._buffer)
            return self._traced(
                program.device, stream, "run", items,
                lambda: program.run(kernel_name, items, stream, args, grid, block, self._buffer),
            )
        except Exception as exc:  # noqa: BLE001
            return make_failed(exc)

    # -- lifetime ----------------------------------------------------------------
    def unregister(self, gid: GlobalId) -> CompletionToken:
        return self._tokenized(lambda: make_ready(self._registry.unregister(gid)))


# the reference's name for the local dispatch surface (runtime.py:30-120),
# so code importing offloadrt.runtime.LocalDispatch switches over unchanged
LocalDispatch = CudaDispatch


class Runtime:
    """One process: its CUDA devices, registry and dispatch table.  Use as a
    context manager or call close()."""

    def __init__(
        self,
        backend: str = "cuda",
        devices: DeviceSpec = None,
        locality_id: int = 0,
        record_events: bool = False,
        device_names: Optional[Sequence[str]] = None,
    ):
        if backend != "cuda":
            raise BadArgsError(
                f"unknown backend {backend!r}: this runtime executes on CUDA devices only"
            )
        _native.load()
        phys = physical_devices()
        if not phys:
            raise InternalError(f"no CUDA device available: {_native.last_error()}")
        if devices is None:
            ordinals = list(range(len(phys)))
        elif isinstance(devices, int):
            if devices < 1:
                raise BadArgsError("device count must be positive")
            ordinals = [i % len(phys) for i in range(devices)]
        else:
            ordinals = [int(d) for d in devices]
            for d in ordinals:
                if not 0 <= d < len(phys):
                    raise BadArgsError(f"CUDA device {d} does not exist ({len(phys)} visible)")
        self.registry = Registry(locality_id)
        self.local = CudaDispatch(self.registry)
        self._devices: list[tuple[GlobalId, DeviceObject]] = []
        self._connections: dict = {}      # locality id -> transport.RemoteLocality
        self._remote_devices: dict = {}   # locality id -> [(gid, DeviceInfo)]
        self._closed = False
        for i, o in enumerate(ordinals):
            name = device_names[i] if device_names else None
            obj = DeviceObject(describe(i, phys[o], name), phys[o], record_events)
            gid = self.registry.register(ObjectKind.DEVICE, obj)
            self._devices.append((gid, obj))

    def dispatch(self, gid: GlobalId):
        """The dispatch serving gid: this process's CUDA devices, or the
        proxy of the connected locality that minted it (reference
        runtime.py:178-184)."""
        if gid.locality_id == self.registry.self_locality_id:
            return self.local
        proxy = self._connections.get(gid.locality_id)
        if proxy is None:
            raise UnknownGidError(f"{gid} names an unknown locality")
        return proxy

    def local_program(self, gid: GlobalId):
        """(registry, generation, weakref to the ProgramObject) for a program
        owned by this process, else None — the handles' fast launch path
        (handles.py); the resolution stays valid while ``registry.generation``
        is unchanged, and while it is the registry keeps the object alive, so
        the weak reference resolves.  A weak reference, so that a handle's
        cache never keeps an unregistered object's device memory alive."""
        if gid.locality_id != self.registry.self_locality_id:
            return None
        try:
            reg = self.registry
            return reg, reg.generation, weakref.ref(self.local._program(gid))
        except Exception:  # noqa: BLE001 - the general path reports it
            return None

    def local_buffer(self, gid: GlobalId):
        """(registry, generation, weakref to the BufferObject) for a buffer
        owned by this process, else None — the handles' fast paths
        (handles.py); see local_program for why the reference is weak."""
        if gid.locality_id != self.registry.self_locality_id:
            return None
        try:
            reg = self.registry
            return reg, reg.generation, weakref.ref(self.local._buffer(gid))
        except Exception:  # noqa: BLE001 - the general path reports it
            return None

    def get_all_devices(self, major: int = 0, minor: int = 0) -> CompletionToken:
        """Every device with capability >= (major, minor): this process's in
        ordinal order, then connected localities' ordered by locality id
        (reference runtime.py:188-200)."""
        out = [DeviceHandle(g, o.info, self) for g, o in self._devices if o.info.meets(major, minor)]
        for lid in sorted(self._remote_devices):
            out.extend(DeviceHandle(g, i, self) for g, i in self._remote_devices[lid]
                       if i.meets(major, minor))
        return make_ready(out)

    def local_device_table(self) -> list[tuple[GlobalId, DeviceInfo]]:
        return [(g, o.info) for g, o in self._devices]

    def device_objects(self) -> list[DeviceObject]:
        return [o for _, o in self._devices]

    def trim_memory(self) -> None:
        """Return the memory that released buffers still hold (stream-ordered
        pool blocks, cached VMM mappings) to every local device."""
        for _, o in self._devices:
            o.trim_memory()

    def local_device_object(self, gid: GlobalId) -> Optional[DeviceObject]:
        for g, o in self._devices:
            if g == gid:
                return o
        return None

    def connect(self, address: str) -> LocalityInfo:
        """Connect to a daemon at ``host:port`` (this package's ``serve`` or
        the reference's ``offloadd``); its devices join discovery and its
        gids dispatch to the connection (reference runtime.py:204-216)."""
        from . import transport

        proxy = transport.connect(address)
        info = LocalityInfo(proxy.locality_id, address)
        try:
            self.registry.add_locality(info, proxy)
        except ValueError:
            proxy.close()
            raise
        self._connections[proxy.locality_id] = proxy
        self._remote_devices[proxy.locality_id] = proxy.devices
        return info

    def close(self) -> None:
        if self._closed:
            return
        self._closed = True
        for proxy in self._connections.values():
            proxy.close()
        for _, obj in self._devices:
            obj.close()

    def __enter__(self) -> "Runtime":
        return self

    def __exit__(self, *exc) -> None:
        self.close()


__all__ = ["Runtime", "CudaDispatch", "DeviceHandle", "BufferHandle", "ProgramHandle", "copy"]
