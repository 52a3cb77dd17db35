"""ctypes binding of libofl.so (the C-ABI declared in include/ofl.h).

This is the only module that touches the native library.  There is no CPU
fallback: if the library is missing or no CUDA device is usable, every
entry into the CUDA backend raises :class:`~.errors.InternalError`.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, c_char_p, c_double, c_int, c_uint32, c_uint64, c_void_p

from .errors import (
    BadArgsError,
    CompileError,
    InternalError,
    OobAccessError,
    OutOfMemoryError,
    UnknownGidError,
)

OFL_OK = 0
OFL_ERR_UNKNOWN_GID = 1
OFL_ERR_BAD_ARGS = 2
OFL_ERR_COMPILE = 3
OFL_ERR_OOB_ACCESS = 4
OFL_ERR_INTERNAL = 5
OFL_ERR_OOM = 6
OFL_ERR_CUDA = 7
OFL_ERR_NCCL = 8

STREAM_COPY, STREAM_SCALE, STREAM_ADD, STREAM_TRIAD = 0, 1, 2, 3
DT_U32, DT_F64, DT_F32 = 0, 1, 2
OP_SUM, OP_MAX = 0, 1

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OFL_LIB", os.path.join(_HERE, "lib", "libofl.so"))

_c_stream = c_void_p
_u64p = POINTER(c_uint64)

# name -> (restype, argtypes)
_SIGNATURES = {
    "ofl_abi_version": (c_int, []),
    "ofl_last_error": (c_char_p, []),
    "ofl_kernel_launches": (c_uint64, []),
    "ofl_device_count": (c_int, [POINTER(c_int)]),
    "ofl_device_props": (
        c_int,
        [c_int, c_char_p, c_int, POINTER(c_int), POINTER(c_int), _u64p, POINTER(c_int), _u64p],
    ),
    "ofl_device_pci_bus_id": (c_int, [c_int, c_char_p, c_int]),
    "ofl_stream_create": (c_int, [c_int, POINTER(c_void_p)]),
    "ofl_stream_destroy": (c_int, [_c_stream]),
    "ofl_stream_tail": (c_uint64, [_c_stream]),
    "ofl_stream_done": (c_uint64, [_c_stream]),
    "ofl_stream_handle": (c_void_p, [_c_stream]),
    "ofl_malloc": (c_int, [c_int, c_uint64, POINTER(c_void_p)]),
    "ofl_malloc_shareable": (c_int, [c_int, c_uint64, POINTER(c_void_p)]),
    "ofl_free": (c_int, [c_int, c_void_p]),
    "ofl_trim_memory": (c_int, [c_int]),
    "ofl_host_alloc": (c_int, [c_uint64, POINTER(c_void_p)]),
    "ofl_host_free": (c_int, [c_void_p]),
    "ofl_h2d": (c_int, [_c_stream, c_void_p, c_void_p, c_uint64, _u64p]),
    "ofl_d2h": (c_int, [_c_stream, c_void_p, c_void_p, c_uint64, _u64p]),
    "ofl_ipc_handle": (c_int, [c_void_p, c_char_p]),
    "ofl_ipc_open": (c_int, [c_int, c_char_p, POINTER(c_void_p)]),
    "ofl_ipc_close": (c_int, [c_int, c_void_p]),
    "ofl_gate_signal": (c_int, [_c_stream, c_void_p, c_uint64, _u64p]),
    "ofl_gate_wait": (c_int, [_c_stream, c_void_p, c_int, c_uint64, c_void_p, _u64p]),
    "ofl_d2h_rows": (c_int, [_c_stream, c_void_p, c_uint64, c_void_p, c_uint64, c_uint64, _u64p]),
    "ofl_d2d": (c_int, [_c_stream, c_void_p, c_void_p, c_uint64, _u64p]),
    "ofl_h2d_pageable": (c_int, [_c_stream, c_void_p, c_void_p, c_uint64, _u64p]),
    "ofl_host_memcpy": (c_int, [c_void_p, c_void_p, c_uint64]),
    "ofl_d2h_chunked": (c_int, [_c_stream, c_void_p, c_void_p, c_uint64, c_uint64,
                                ctypes.POINTER(c_void_p), _u64p]),
    "ofl_collect": (c_int, [c_void_p, c_void_p]),
    "ofl_read_release": (c_int, [c_void_p]),
    "ofl_p2p": (c_int, [_c_stream, c_void_p, c_int, c_void_p, c_int, c_uint64, _u64p]),
    "ofl_stream_wait": (c_int, [_c_stream, _c_stream, c_uint64]),
    "ofl_query": (c_int, [_c_stream, c_uint64, POINTER(c_int)]),
    "ofl_wait": (c_int, [_c_stream, c_uint64]),
    "ofl_notify": (c_int, [_c_stream, c_uint64, c_uint64]),
    "ofl_completion_fd": (c_int, []),
    "ofl_completion_post": (c_int, [c_uint64]),
    "ofl_drain": (c_int, [_u64p, c_int, POINTER(c_int)]),
    "ofl_event_create": (c_int, [c_int, POINTER(c_void_p)]),
    "ofl_event_record": (c_int, [c_void_p, _c_stream]),
    "ofl_event_elapsed_ms": (c_int, [c_void_p, c_void_p, POINTER(ctypes.c_float)]),
    "ofl_event_destroy": (c_int, [c_void_p]),
    "ofl_stream_op": (
        c_int,
        [_c_stream, c_int, c_void_p, c_void_p, c_void_p, c_double, c_uint64, _u64p],
    ),
    "ofl_stencil": (c_int, [_c_stream, c_void_p, c_void_p, c_uint64, c_uint64, _u64p]),
    "ofl_heat": (c_int, [_c_stream, c_void_p, c_void_p, c_uint64, c_uint64, c_int, _u64p]),
    "ofl_stencil2d": (c_int, [_c_stream, c_void_p, c_void_p, c_uint32, c_uint32, c_uint64,
                              c_uint64, _u64p]),
    "ofl_stencil2d_slab": (c_int, [_c_stream, c_void_p, c_void_p, c_uint32, c_uint32, c_uint32,
                                   c_uint32, c_void_p, c_int, c_void_p, c_int, _u64p]),
    "ofl_xchg_bytes": (c_int, []),
    "ofl_dot_f32_allreduce": (c_int, [_c_stream, c_void_p, c_void_p, c_void_p, c_uint64, c_int,
                                      c_int, POINTER(c_void_p), POINTER(c_int), c_uint64, _u64p]),
    "ofl_heat_slab": (c_int, [_c_stream, c_void_p, c_void_p, c_uint64, c_int, c_uint64, c_uint64,
                              c_void_p, c_int, c_void_p, c_int, c_uint64, _u64p]),
    "ofl_mandelbrot": (
        c_int,
        [
            _c_stream, c_void_p, c_uint32, c_uint32, c_double, c_double, c_double, c_double,
            c_double, c_uint32, c_uint64, c_uint32, c_uint32, c_int, _u64p,
        ],
    ),
    "ofl_sum_u32": (c_int, [_c_stream, c_void_p, c_void_p, c_uint64, _u64p]),
    "ofl_dot_f32": (c_int, [_c_stream, c_void_p, c_void_p, c_void_p, c_uint64, _u64p]),
    "ofl_partition": (c_int, [_c_stream, c_void_p, c_uint32, c_uint64, _u64p]),
    "ofl_bench_raw_chain": (
        c_int,
        [
            _c_stream, c_void_p, c_void_p, c_uint64, c_void_p, c_void_p, c_void_p, c_uint64,
            c_uint64, c_int, POINTER(c_double),
        ],
    ),
    "ofl_bench_fp64_peak": (c_int, [_c_stream, POINTER(c_double)]),
    "ofl_jit_available": (c_int, [c_char_p]),
    "ofl_jit_compile": (c_int, [c_int, c_char_p, c_char_p, POINTER(c_void_p), c_char_p, c_int]),
    "ofl_jit_launch": (c_int, [_c_stream, c_void_p, POINTER(c_void_p), c_uint64, c_int, _u64p]),
    "ofl_jit_destroy": (c_int, [c_void_p]),
    "ofl_fill_ones": (c_int, [_c_stream, c_void_p, c_uint64, _u64p]),
    "ofl_nccl_available": (c_int, [c_char_p]),
    "ofl_nccl_unique_id": (c_int, [c_char_p]),
    "ofl_nccl_init_all": (c_int, [c_int, POINTER(c_int), POINTER(c_void_p)]),
    "ofl_nccl_init_rank": (c_int, [c_int, c_int, c_int, c_char_p, POINTER(c_void_p)]),
    "ofl_allreduce": (
        c_int, [c_void_p, _c_stream, c_void_p, c_void_p, c_uint64, c_int, c_int, _u64p],
    ),
    "ofl_allreduce_group": (
        c_int,
        [
            c_int, POINTER(c_void_p), POINTER(c_void_p), POINTER(c_void_p), POINTER(c_void_p),
            c_uint64, c_int, c_int, _u64p,
        ],
    ),
    "ofl_comm_destroy": (c_int, [c_void_p]),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None
_lib_lock = threading.Lock()
# csrc/oflcall.c: vectorcall entry points for the per-operation hot calls
# (ofl_h2d, ofl_stream_op, ofl_wait), bound to the loaded library; None when the module
# is not built (the ctypes prototypes then serve those calls too)
_fast = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libofl.so and attach prototypes.  Raises InternalError when the
    library has not been built — the CUDA backend has no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(path):
                raise InternalError(
                    f"libofl.so not found at {path}; run __graft_entry__.build() "
                    "(the CUDA backend has no CPU fallback)"
                )
            lib = ctypes.CDLL(path)
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _bind_fast(lib)
            _lib = lib
    return _lib


def _bind_fast(lib) -> None:
    global _fast
    try:
        from . import _oflcall
    except ImportError:
        _fast = None
        return
    addr = lambda fn: ctypes.cast(fn, ctypes.c_void_p).value  # noqa: E731
    _oflcall.bind(addr(lib.ofl_h2d), addr(lib.ofl_stream_op), addr(lib.ofl_wait),
                  addr(lib.ofl_query), addr(lib.ofl_collect))
    _fast = _oflcall


def fastcall():
    """The bound _oflcall module (or None); call after load()."""
    return _fast


def last_error() -> str:
    msg = load().ofl_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def error_for(status: int, what: str = "") -> Exception:
    """Exception for a non-zero C status (codes per errors.py:92-96 of the
    reference, extended with OOM / CUDA / NCCL)."""
    msg = last_error()
    if what:
        msg = f"{what}: {msg}" if msg else what
    if status == OFL_ERR_UNKNOWN_GID:
        return UnknownGidError(msg)
    if status == OFL_ERR_BAD_ARGS:
        return BadArgsError(msg)
    if status == OFL_ERR_COMPILE:
        return CompileError(msg)
    if status == OFL_ERR_OOB_ACCESS:
        return OobAccessError(msg)
    if status == OFL_ERR_OOM:
        return OutOfMemoryError(msg)
    return InternalError(msg)


def check(status: int, what: str = "") -> None:
    if status:
        raise error_for(status, what)


def device_count() -> int:
    n = c_int(0)
    status = load().ofl_device_count(ctypes.byref(n))
    if status:
        return 0
    return n.value


def nccl_library_path() -> str:
    """The NCCL that torch would load (if the torch wheel ships one)."""
    try:
        import nvidia.nccl  # type: ignore

        for base in nvidia.nccl.__path__:
            cand = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                return cand
    except Exception:  # noqa: BLE001
        pass
    return ""
