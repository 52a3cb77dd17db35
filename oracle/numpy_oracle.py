"""Second, independent restatement in numpy / pure Python — TEST
INFRASTRUCTURE.  Used to cross-check the C oracle on small inputs.

Follows the reference's validators (/root/reference/pkg/src/offloadrt/bench/
harness.py:123-158) and sequential oracles (pkg/tests/oracles.py:13-69);
every expression keeps the .k evaluation order.
"""

from __future__ import annotations

import math

import numpy as np

M32 = 0xFFFFFFFF


def stencil(x: np.ndarray) -> np.ndarray:
    """harness.py:123-126."""
    x = np.asarray(x, dtype=np.float64)
    y = x.copy()
    y[1:-1] = 0.5 * x[:-2] + x[1:-1] + 0.5 * x[2:]
    return y


def stencil2d(x: np.ndarray, w: int, h: int) -> np.ndarray:
    """kernels/stencil2d.k restated over the whole grid (w, h >= 1)."""
    X = np.asarray(x, dtype=np.float64).reshape(h, w)
    Y = X.copy()
    if h > 2 and w > 2:
        Y[1:-1, 1:-1] = 0.25 * (((X[:-2, 1:-1] + X[1:-1, :-2]) + X[1:-1, 2:]) + X[2:, 1:-1])
    return Y.ravel()


def stencil_seq(x) -> list:
    """tests/oracles.py:13-20 restated."""
    out = list(x)
    for i in range(1, len(x) - 1):
        out[i] = 0.5 * x[i - 1] + x[i] + 0.5 * x[i + 1]
    return out


def heat(x: np.ndarray, steps: int) -> np.ndarray:
    y = np.asarray(x, dtype=np.float64)
    for _ in range(steps):
        y = stencil(y)
    return y


def stream(op: str, b, c=None, s: float = 0.0) -> np.ndarray:
    b = np.asarray(b, dtype=np.float64)
    if op == "copy":
        return b.copy()
    if op == "scale":
        return s * b
    c = np.asarray(c, dtype=np.float64)
    if op == "add":
        return b + c
    return b + s * c


def sum_u32(values) -> int:
    """harness.py:129-130."""
    return int(np.asarray(values, dtype=np.uint64).sum()) & M32


def mandelbrot_pixel(cre: float, cim: float, max_iter: int, esc: float = 4.0) -> int:
    """tests/oracles.py:30-42 restated."""
    zr = zi = 0.0
    count = 0
    for _ in range(max_iter):
        if zr * zr + zi * zi > esc:
            break
        t = zr * zr - zi * zi + cre
        zi = 2.0 * zr * zi + cim
        zr = t
        count += 1
    return count


def mandelbrot(width: int, height: int, viewport=(-2.0, 1.0, -1.5, 1.5), max_iter: int = 256,
               esc: float = 4.0) -> np.ndarray:
    """Vectorised escape time (harness.py:133-158 restated)."""
    re0, re1, im0, im1 = viewport
    idx = np.arange(width * height, dtype=np.int64)
    px = (idx % width).astype(np.float64)
    py = (idx // width).astype(np.float64)
    cre = re0 + (px + 0.5) * (re1 - re0) / float(width)
    cim = im0 + (py + 0.5) * (im1 - im0) / float(height)
    zr = np.zeros(idx.size)
    zi = np.zeros(idx.size)
    count = np.zeros(idx.size, dtype=np.uint32)
    live = np.ones(idx.size, dtype=bool)
    for _ in range(max_iter):
        live &= ~(zr * zr + zi * zi > esc)
        if not live.any():
            break
        a, b = zr[live], zi[live]
        t = a * a - b * b + cre[live]
        zi[live] = 2.0 * a * b + cim[live]
        zr[live] = t
        count[live] += 1
    return count


def partition(offset: int, count: int) -> np.ndarray:
    """tests/oracles.py:58-64 restated."""
    out = np.empty(count)
    for k in range(count):
        v = float((offset + k) & M32)
        out[k] = math.sqrt(math.sin(v) * math.sin(v) + math.cos(v) * math.cos(v))
    return out


def dot_f32(a, b, chunk: int = 1 << 16) -> float:
    """fp64-accumulated dot of fp32 vectors, chunked like the C oracle."""
    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float32)
    total = 0.0
    for lo in range(0, a.size, chunk):
        total += float(np.dot(a[lo : lo + chunk].astype(np.float64), b[lo : lo + chunk].astype(np.float64)))
    return total
