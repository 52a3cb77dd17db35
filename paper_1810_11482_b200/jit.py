"""NVRTC path for kernels without a hand-written binding.

``build()`` falls back here when a kernel's canonical form is not one of the
workloads (bindings.py): the IR is lowered to CUDA C (kernel/cuda_codegen.py),
compiled for sm_100a by NVRTC inside libofl.so (csrc/ofl_jit.cu) once per
(source, device), and launched stream-ordered like every other operation.
A 16-byte error record per launch (reset on the stream before the kernel,
copied back after it) carries the executor's abort protocol
(/root/reference/pkg/src/offloadrt/kernel/codegen.py:10-13,38-41): the
token fails with OobAccessError (index) or InternalError (division by zero,
cast range) for the smallest failing gtid.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import _native, hostmem
from .completion import DeviceToken
from .errors import CompileError, InternalError, OobAccessError
from .kernel import cuda_codegen

_cache: dict = {}
_cache_lock = threading.Lock()
_SLOTS = 4096
_THREADS = 256


def _nvrtc_hint() -> bytes:
    try:
        import nvidia.cuda_nvrtc  # type: ignore

        for base in nvidia.cuda_nvrtc.__path__:
            for name in ("libnvrtc.so.12", "libnvrtc.so"):
                p = os.path.join(base, "lib", name)
                if os.path.exists(p):
                    return p.encode()
    except Exception:  # noqa: BLE001
        pass
    return b""


def compile_kernel(ir, ordinal: int):
    """Compiled handle for (kernel, device); cached per generated source."""
    src = cuda_codegen.generate(ir)
    key = (src, ordinal)
    with _cache_lock:
        got = _cache.get(key)
    if got is not None:
        return got
    lib = _native.load()
    lib.ofl_jit_available(_nvrtc_hint())
    handle = ctypes.c_void_p()
    log = ctypes.create_string_buffer(8192)
    status = lib.ofl_jit_compile(ordinal, src.encode(), b"ofl_k", ctypes.byref(handle), log, 8192)
    if status:
        raise CompileError(f"kernel {ir.name!r}: NVRTC failed: {_native.last_error()[:2000]}", 0, 0)
    with _cache_lock:
        _cache.setdefault(key, handle.value)
        return _cache[key]


class _ErrSlots:
    """Per-stream ring of 16-byte device error records, owned by the Stream
    (freed in Stream.destroy).  Slots are taken under a lock: two threads
    launching on one stream never share a record."""

    __slots__ = ("device", "base", "next", "lock")

    def __init__(self, device):
        self.device = device
        self.base = device.allocate(_SLOTS * 16)
        self.next = 0
        self.lock = threading.Lock()

    def take(self) -> int:
        with self.lock:
            k = self.next
            self.next = (k + 1) % _SLOTS
        return self.base + 16 * k

    def free(self) -> None:
        if self.base:
            self.device.release(self.base, _SLOTS * 16)
            self.base = 0


_slots_lock = threading.Lock()


def _err_slot(stream) -> int:
    s = stream.err_slots
    if s is None:
        with _slots_lock:
            s = stream.err_slots
            if s is None:
                s = _ErrSlots(stream.device)
                stream.err_slots = s
    return s.take()


def launch(handle: int, ir, st, values: list, items: int, grid_volume: int, block_volume: int):
    """Enqueue one generic launch; returns a DeviceToken whose completion
    checks the error record."""
    lib = st.lib
    keep = []
    for (_, kind), v in zip(ir.params, values):
        if kind.startswith("buffer_"):
            keep.append(ctypes.c_void_p(v.ptr))
            keep.append(ctypes.c_uint64(v.size_bytes // (8 if kind == "buffer_f64" else 4)))
        elif kind == "scalar_f64":
            keep.append(ctypes.c_double(v))
        else:
            keep.append(ctypes.c_uint32(v))
    err = _err_slot(st)
    keep += [ctypes.c_uint64(items), ctypes.c_uint32(grid_volume & 0xFFFFFFFF),
             ctypes.c_uint32(block_volume & 0xFFFFFFFF), ctypes.c_void_p(err)]
    params = (ctypes.c_void_p * len(keep))(*[ctypes.addressof(k) for k in keep])
    t = ctypes.c_uint64()
    _native.check(lib.ofl_fill_ones(st.ptr, err, 16, ctypes.byref(t)), "error record reset")
    sms = st.device.physical.sms
    blocks = min((items + _THREADS - 1) // _THREADS, sms * 32)
    _native.check(lib.ofl_jit_launch(st.ptr, handle, params, blocks, _THREADS, ctypes.byref(t)),
                  f"launch of {ir.name!r}")
    block = hostmem.pool.get(16)
    status = lib.ofl_d2h(st.ptr, block.addr, err, 16, ctypes.byref(t))
    if status:
        hostmem.pool.put(block)
        _native.check(status, "error record read")
    from .buffer import _Landing

    landing = _Landing(block, 16)
    st.keep(t.value, landing.release_later)

    def finish():
        rec = np.frombuffer(landing.take(), dtype=np.uint64)
        if rec[0] == np.uint64(0xFFFFFFFFFFFFFFFF):
            return None
        detail = int(rec[0]) & 0xFFFFFFFF
        code = int(rec[1]) & 0xFF
        if code == cuda_codegen.CODE_OOB:
            raise OobAccessError(f"kernel buffer index {detail} out of range")
        if code == cuda_codegen.CODE_DIV0:
            raise InternalError("division by zero in kernel")
        raise InternalError("u32() cast out of representable range")

    return DeviceToken(st, t.value, finish)
