"""CPU oracle for the hot path — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only tests/, ``__graft_entry__.smoke()`` and bench.py (its ``cpu_baseline``
leg and ``--impl reference``) may import this package.  It is the checker
the CUDA path is compared against, never the thing measured or shipped; the
product package (paper_1810_11482_b200) does not import it.

Two restatements of the reference's arithmetic (/root/reference/pkg/src/
offloadrt: bench/kernels/*.k run by kernel/codegen.py's sequential executor,
validators bench/harness.py:123-158, tests/oracles.py:13-69):

* ``ofl_oracle.c`` (this wrapper): plain C, -ffp-contract=off, optionally
  multi-threaded over independent items — fast enough for full sizes and
  used as the CPU baseline;
* ``numpy_oracle.py``: vectorised numpy / pure-Python loops for small cases.

Pinning: both are checked against golden vectors produced by importing and
running the reference itself (tests/golden/make_golden.py ->
tests/golden/golden.json) and against the reference tests' known answers.
The fp32 dot product has no reference kernel (the kernel language has no
f32); it is pinned by the reference executor running the same arithmetic on
f64 buffers holding the fp32 values (``dot_seq`` in make_golden.py, results
in tests/golden/golden_long.json), which ``dot_f32_seq`` reproduces bit for
bit and ``dot_f32`` (fixed 2^16 chunks) within 1e-12 relative.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build() -> str:
    """Compile liboracle.so with the committed recipe (oracle/Makefile)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return LIB


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        vp, u64, u32, i32, f64 = (
            ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_double,
        )
        L.oracle_stream.argtypes = [i32, vp, vp, vp, f64, u64, i32]
        L.oracle_stream.restype = None
        L.oracle_stencil.argtypes = [vp, vp, u64, u64, i32]
        L.oracle_stencil.restype = None
        L.oracle_stencil2d.argtypes = [vp, vp, u32, u32, u64, i32]
        L.oracle_stencil2d.restype = None
        L.oracle_heat.argtypes = [vp, vp, u64, u64, i32]
        L.oracle_heat.restype = None
        L.oracle_mandelbrot.argtypes = [vp, u32, u32, f64, f64, f64, f64, f64, u32, u64, u32, u32, i32]
        L.oracle_mandelbrot.restype = None
        L.oracle_sum_u32.argtypes = [vp, u64, i32]
        L.oracle_sum_u32.restype = u32
        L.oracle_dot_f32.argtypes = [vp, vp, u64, i32]
        L.oracle_dot_f32.restype = f64
        L.oracle_dot_f32_seq.argtypes = [vp, vp, u64]
        L.oracle_dot_f32_seq.restype = f64
        L.oracle_partition.argtypes = [vp, u32, u64, i32]
        L.oracle_partition.restype = None
        L.oracle_max_threads.argtypes = []
        L.oracle_max_threads.restype = i32
        _lib = L
    return _lib


def max_threads() -> int:
    return lib().oracle_max_threads()


def _p(a: np.ndarray) -> int:
    assert a.flags.c_contiguous
    return a.ctypes.data


STREAM_OPS = {"copy": 0, "scale": 1, "add": 2, "triad": 3}


def stream(op: str, b: np.ndarray, c=None, s: float = 0.0, out=None, threads: int = 1):
    """STREAM kernel over f64 vectors: copy a=b, scale a=s*b, add a=b+c,
    triad a=b+s*c."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    c = b if c is None else np.ascontiguousarray(c, dtype=np.float64)
    a = np.empty_like(b) if out is None else out
    lib().oracle_stream(STREAM_OPS[op], _p(a), _p(b), _p(c), float(s), b.size, threads)
    return a


def stencil(x: np.ndarray, items=None, out=None, threads: int = 1) -> np.ndarray:
    """One stencil.k step; items beyond min(n, items) keep `out`'s content."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = x.size
    y = np.zeros_like(x) if out is None else out
    lib().oracle_stencil(_p(x), _p(y), n, n if items is None else items, threads)
    return y


def stencil2d(x: np.ndarray, w: int, h: int, items=None, out=None, threads: int = 1) -> np.ndarray:
    """One stencil2d.k step over a row-major w x h grid; items beyond
    min((w*h) mod 2^32, items) keep `out`'s content."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros_like(x) if out is None else out
    cells = (w * h) & 0xFFFFFFFF
    lib().oracle_stencil2d(_p(x), _p(y), w, h, cells if items is None else items, threads)
    return y


def heat2d(x: np.ndarray, w: int, h: int, steps: int, threads: int = 1) -> np.ndarray:
    """`steps` stencil2d.k applications ping-ponging; returns the final state."""
    a = np.array(x, dtype=np.float64, copy=True)
    b = a.copy()
    for _ in range(steps):
        stencil2d(a, w, h, out=b, threads=threads)
        a, b = b, a
    return a


def heat(x: np.ndarray, steps: int, threads: int = 1) -> np.ndarray:
    """`steps` stencil.k applications; returns the final state."""
    a = np.array(x, dtype=np.float64, copy=True)
    b = np.zeros_like(a)
    lib().oracle_heat(_p(a), _p(b), a.size, steps, threads)
    return a if steps % 2 == 0 else b


def mandelbrot(width: int, height: int, viewport=(-2.0, 1.0, -1.5, 1.5), esc: float = 4.0,
               max_iter: int = 256, items=None, row_first: int = 0, row_step: int = 1,
               threads: int = 1, out=None) -> np.ndarray:
    re0, re1, im0, im1 = viewport
    total = (width * height) & 0xFFFFFFFF
    o = np.zeros(total, dtype=np.uint32) if out is None else out
    lib().oracle_mandelbrot(
        _p(o), width, height, re0, re1, im0, im1, esc, max_iter,
        total if items is None else items, row_first, row_step, threads,
    )
    return o


def sum_u32(values: np.ndarray, threads: int = 1) -> int:
    v = np.ascontiguousarray(values, dtype=np.uint32)
    return int(lib().oracle_sum_u32(_p(v), v.size, threads))


def dot_f32(a: np.ndarray, b: np.ndarray, threads: int = 1) -> float:
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    return float(lib().oracle_dot_f32(_p(a), _p(b), min(a.size, b.size), threads))


def dot_f32_seq(a: np.ndarray, b: np.ndarray) -> float:
    """The reference executor's order (one work item, index order); pinned
    bit for bit by tests/golden/golden_long.json."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    return float(lib().oracle_dot_f32_seq(_p(a), _p(b), min(a.size, b.size)))


def partition(offset: int, count: int, threads: int = 1) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    lib().oracle_partition(_p(out), offset, count, threads)
    return out
