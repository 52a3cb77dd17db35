"""Native implementations behind recognised kernels.

``build()`` type-checks a kernel and looks its canonical form up here
(kernel/canon.py).  Each binding launches one hand-written sm_100a kernel of
libofl.so with the exact semantics of the reference's sequential executor
(/root/reference/pkg/src/offloadrt/kernel/codegen.py:107-128): work items
gtid = 0 .. grid*block-1 each run the body.  Items are independent in every
bound kernel, so the device order is free.

Host-side pre-checks reproduce the executor's kernel aborts: the first
out-of-bounds buffer index (in gtid order, store index before loads as the
executor evaluates them) fails the token with OobAccessError carrying that
index.  Unlike the sequential executor no partial writes happen before the
abort — the kernel is not launched at all.

Builtin programs (``BUILTIN_KERNELS``) extend the language's reach where the
reference has no way to express the workload: fp32 data (the language has no
f32, /root/reference/pkg/src/offloadrt/kernel/lang.py:29) and the multi-step
heat equation with temporal blocking.
"""

from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass, field
from functools import lru_cache
from typing import Callable, Optional

from . import _native
from .errors import BadArgsError
from .kernel import parse_and_validate
from .kernel.canon import canonical

M32 = 0xFFFFFFFF
_HERE = os.path.dirname(os.path.abspath(__file__))


@dataclass(frozen=True)
class Binding:
    name: str
    kinds: tuple  # parameter kinds, in order
    # launch(stream, values, items, ticket_ref) -> status, or raises
    launch: Callable
    # first out-of-bounds index (or None) given values and items
    oob: Optional[Callable] = None
    # plan(values, items) -> (fn, args) with fn(stream_ptr, *args) -> ticket
    # | -status, or None (anything unusual, e.g. an out-of-bounds access:
    # launch() reports it): the handles' run fast path for the
    # per-future-overhead-critical kernels, cacheable while the registry
    # generation holds
    plan: Optional[Callable] = None
    # per parameter: 0 buffer, 1 scalar_f64, 2 scalar_u32 (the run fast path)
    codes: tuple = field(default=(), init=False, compare=False)

    def __post_init__(self):
        object.__setattr__(self, "codes", tuple(0 if k.startswith("buffer") else (1 if k == "scalar_f64" else 2)
                           for k in self.kinds))


def _first_oob(candidates, failing) -> Optional[int]:
    """Smallest gtid among candidates whose accesses fail; returns the failing
    index reported for it."""
    for g in sorted(set(c for c in candidates if c is not None and c >= 0)):
        idx = failing(g)
        if idx is not None:
            return idx
    return None


# -- STREAM ----------------------------------------------------------------------


def _stream_binding(name: str, op: int, kinds: tuple) -> Binding:
    has_c = op in (_native.STREAM_ADD, _native.STREAM_TRIAD)
    has_s = op in (_native.STREAM_SCALE, _native.STREAM_TRIAD)

    def unpack(v):
        a, b = v[0], v[1]
        c = v[2] if has_c else None
        s = v[3] if op == _native.STREAM_TRIAD else (v[2] if has_s else 0.0)
        n = v[-1]
        return a, b, c, s, n

    def oob(v, items):
        m = v[-1] if v[-1] < items else items
        lo = min(v[0].size_bytes, v[1].size_bytes, v[2].size_bytes if has_c else 1 << 62) >> 3
        return lo if m > lo else None

    fast = _native.fastcall()

    def launch(st, v, items, ticket):
        a, b, c, s, n = unpack(v)
        if fast is not None:
            t = fast.stream_op(st.ptr, op, a.ptr, b.ptr, c.ptr if c is not None else b.ptr,
                               s, n if n < items else items)
            if t < 0:
                return -t
            ticket.value = t
            return 0
        return st.lib.ofl_stream_op(
            st.ptr, op, a.ptr, b.ptr, c.ptr if c is not None else b.ptr, s,
            n if n < items else items, ticket,
        )

    plan = None
    if fast is not None:
        stream_op = fast.stream_op

        def plan(v, items):
            a, b = v[0], v[1]
            c = v[2] if has_c else b
            n = v[-1]
            m = n if n < items else items
            if m > (a.size_bytes >> 3) or m > (b.size_bytes >> 3) or m > (c.size_bytes >> 3):
                return None  # launch() reports the out-of-bounds index
            s = v[3] if op == _native.STREAM_TRIAD else (v[2] if has_s else 0.0)
            return stream_op, (op, a.ptr, b.ptr, c.ptr, s, m)

    return Binding(name, kinds, launch, oob, plan)


# -- stencil ---------------------------------------------------------------------


def _stencil_oob(v, items):
    x, y, n = v
    m = min(n, items)
    if m == 0:
        return None
    lx, ly = x.elements("buffer_f64"), y.elements("buffer_f64")

    def failing(g):
        if g >= m:
            return None
        if g >= ly:
            return g  # store index is checked first
        if g == 0 or g == ((n - 1) & M32):
            return g if g >= lx else None
        for idx in (g - 1, g, g + 1):
            if idx >= lx:
                return idx
        return None

    return _first_oob([0, 1, lx - 1, lx, ly, m - 1], failing)


def _stencil_launch(st, v, items, ticket):
    x, y, n = v
    m = min(n, items)
    if m and x is y:
        raise BadArgsError(
            "stencil: in-place update (x is y) is order-dependent; use two buffers"
        )
    return st.lib.ofl_stencil(st.ptr, x.ptr, y.ptr, n, m, ticket)


# -- stencil2d -------------------------------------------------------------------


def _stencil2d_oob(v, items):
    """First out-of-range access in the reference executor's order: items run
    in gtid order; per item the store index is checked, then the loads left
    to right (boundary: u[g]; interior: u[g-w], u[g-1], u[g+1], u[g+w])."""
    x, y, w, h = v
    cells = (w * h) & M32
    m = min(cells, items)
    if m == 0:
        return None
    lx, ly = x.elements("buffer_f64"), y.elements("buffer_f64")
    if lx >= cells and ly >= cells:
        return None

    def boundary(g):
        row, col = divmod(g, w)
        return row == 0 or row == h - 1 or col == 0 or col == w - 1

    def first_interior_from(g):
        g = max(g, 0)
        row, col = divmod(g, w)
        if row == 0:
            row, col = 1, 1
        elif col == 0:
            col = 1
        elif col == w - 1:
            row, col = row + 1, 1
        if row >= h - 1 or col >= w - 1:
            return None
        return row * w + col

    def first_boundary_from(g):
        return g if boundary(g) else (g // w) * w + w - 1

    cand = [ly, first_boundary_from(lx) if lx < m else None,
            first_interior_from(lx - w), first_interior_from(lx - 1),
            first_interior_from(lx + 1), first_interior_from(lx)]

    def failing(g):
        if g >= m:
            return None
        if g >= ly:
            return g
        loads = (g,) if boundary(g) else (g - w, g - 1, g + 1, g + w)
        for idx in loads:
            if idx >= lx:
                return idx
        return None

    return _first_oob(cand, failing)


def _stencil2d_launch(st, v, items, ticket):
    x, y, w, h = v
    cells = (w * h) & M32
    m = min(cells, items)
    if m and x is y:
        raise BadArgsError(
            "stencil2d: in-place update (u is u_next) is order-dependent; use two buffers"
        )
    if w * h >= 1 << 32:
        raise BadArgsError("stencil2d: grids of 2^32 cells or more are not supported")
    return st.lib.ofl_stencil2d(st.ptr, x.ptr, y.ptr, w, h, m, x.elements("buffer_f64"), ticket)


# -- mandelbrot ------------------------------------------------------------------


def _mandel_oob(v, items):
    out, width, height = v[0], v[1], v[2]
    total = (width * height) & M32
    m = min(total, items)
    lo = out.elements("buffer_u32")
    return lo if m > lo else None


def _mandel_launch(st, v, items, ticket):
    out, width, height, re0, re1, im0, im1, esc, max_iter = v
    return st.lib.ofl_mandelbrot(
        st.ptr, out.ptr, width, height, float(re0), float(re1), float(im0), float(im1),
        float(esc), max_iter, items, 0, 1, 0, ticket,
    )


# -- sum -------------------------------------------------------------------------


def _sum_oob(v, items):
    inp, res, n = v
    if n > inp.elements("buffer_u32"):
        return inp.elements("buffer_u32")
    if res.elements("buffer_u32") < 1:
        return 0
    return None


def _sum_launch(st, v, items, ticket):
    inp, res, n = v
    return st.lib.ofl_sum_u32(st.ptr, inp.ptr, res.ptr, n, ticket)


# -- partition -------------------------------------------------------------------


def _partition_oob(v, items):
    out, offset, count = v
    m = min(count, items)
    lo = out.elements("buffer_f64")
    return lo if m > lo else None


def _partition_launch(st, v, items, ticket):
    out, offset, count = v
    return st.lib.ofl_partition(st.ptr, out.ptr, offset, min(count, items), ticket)


# -- builtins (no .k form) -------------------------------------------------------


def _dot_oob(v, items):
    a, b, out, n = v
    m = min(n, items)
    lo = min(a.elements("buffer_f32"), b.elements("buffer_f32"))
    if m > lo:
        return lo
    if out.elements("buffer_f64") < 1:
        return 0
    return None


def _dot_launch(st, v, items, ticket):
    a, b, out, n = v
    return st.lib.ofl_dot_f32(st.ptr, a.ptr, b.ptr, out.ptr, min(n, items), ticket)


def heat_block() -> int:
    """Most steps fused per HBM pass by the heat builtin (default 96 — the
    fastest measured cap for the production pass kernel, profiles/
    r02_heat_sweep.txt; the C side spreads the steps evenly over the fewest
    passes of the right parity).  OFL_HEAT_TB overrides it for the parity
    tests of other schedules; bench.py refuses to run with it set."""
    return max(1, min(128, int(os.environ.get("OFL_HEAT_TB", "96"))))


def _heat_oob(v, items):
    x, y, n, steps = v
    lo = min(x.elements("buffer_f64"), y.elements("buffer_f64"))
    return lo if n > lo else None


def _heat_launch(st, v, items, ticket):
    x, y, n, steps = v
    if items < n:
        raise BadArgsError("heat: the launch must cover all n cells")
    if x is y:
        raise BadArgsError("heat: x and y must be distinct buffers")
    if n == 0 or steps == 0:
        return st.lib.ofl_d2d(st.ptr, x.ptr, x.ptr, 0, ticket)
    return st.lib.ofl_heat(st.ptr, x.ptr, y.ptr, n, steps, heat_block(), ticket)


def _rows_exec(v, items) -> int:
    """Rows a mandelbrot_rows launch computes: row_first + k*row_step below
    the image height and holding a pixel gtid < min(items, width*height)."""
    width, height = v[1], v[2]
    row_first, row_step = v[9], v[10]
    limit = min(items, (width * height) & M32)
    if limit == 0 or width == 0 or row_step == 0 or row_first >= height:
        return 0
    last = min(height - 1, (limit - 1) // width)
    return 0 if last < row_first else (last - row_first) // row_step + 1


def _rows_oob(v, items):
    need = _rows_exec(v, items) * v[1]
    lo = v[0].elements("buffer_u32")
    return lo if need > lo else None


def _rows_launch(st, v, items, ticket):
    out, width, height, re0, re1, im0, im1, esc, max_iter, row_first, row_step = v
    if row_step == 0:
        raise BadArgsError("mandelbrot_rows: row_step must be >= 1")
    return st.lib.ofl_mandelbrot(
        st.ptr, out.ptr, width, height, float(re0), float(re1), float(im0), float(im1),
        float(esc), max_iter, min(items, (width * height) & M32), row_first, row_step, 1, ticket,
    )


BUILTIN_KERNELS = {
    # fp32 dot product with fp64 accumulation into out[0]
    "dot_f32": Binding(
        "dot_f32", ("buffer_f32", "buffer_f32", "buffer_f64", "scalar_u32"), _dot_launch, _dot_oob
    ),
    # `steps` applications of stencil.k, ping-ponging x <-> y; the result is
    # in x for even steps, in y for odd steps
    "heat": Binding(
        "heat", ("buffer_f64", "buffer_f64", "scalar_u32", "scalar_u32"), _heat_launch, _heat_oob
    ),
    # mandelbrot.k over rows row_first + k*row_step only, packed densely
    # (multi-GPU cyclic row split); as in mandelbrot.k only pixels
    # gtid < min(grid*block, width*height) are computed
    "mandelbrot_rows": Binding(
        "mandelbrot_rows",
        ("buffer_u32", "scalar_u32", "scalar_u32", "scalar_f64", "scalar_f64", "scalar_f64",
         "scalar_f64", "scalar_f64", "scalar_u32", "scalar_u32", "scalar_u32"),
        _rows_launch,
        _rows_oob,
    ),
}

BUILTIN_PARAM_NAMES = {
    "dot_f32": ("a", "b", "out", "n"),
    "heat": ("x", "y", "n", "steps"),
    "mandelbrot_rows": ("out", "width", "height", "re0", "re1", "im0", "im1", "esc",
                        "max_iter", "row_first", "row_step"),
}


# -- canonical-form table --------------------------------------------------------


def _source(name: str) -> str:
    with open(os.path.join(_HERE, "kernels", f"{name}.k"), encoding="utf-8") as fh:
        return fh.read()


def kernel_source(name: str) -> str:
    """Source text of a bundled kernel program (stream, stencil, stencil2d,
    mandelbrot, sum, partition)."""
    return _source(name)


@lru_cache(maxsize=None)
def _table() -> dict:
    specs = {
        ("stream", "copy"): lambda k: _stream_binding("copy", _native.STREAM_COPY, k),
        ("stream", "scale"): lambda k: _stream_binding("scale", _native.STREAM_SCALE, k),
        ("stream", "add"): lambda k: _stream_binding("add", _native.STREAM_ADD, k),
        ("stream", "triad"): lambda k: _stream_binding("triad", _native.STREAM_TRIAD, k),
        ("stencil", "stencil"): lambda k: Binding("stencil", k, _stencil_launch, _stencil_oob),
        ("stencil2d", "stencil2d"): lambda k: Binding("stencil2d", k, _stencil2d_launch,
                                                      _stencil2d_oob),
        ("mandelbrot", "mandelbrot"): lambda k: Binding("mandelbrot", k, _mandel_launch, _mandel_oob),
        ("sum", "sum"): lambda k: Binding("sum", k, _sum_launch, _sum_oob),
        ("partition", "partition"): lambda k: Binding(
            "partition", k, _partition_launch, _partition_oob
        ),
    }
    table = {}
    parsed: dict = {}
    for (src, kname), make in specs.items():
        if src not in parsed:
            parsed[src] = parse_and_validate(_source(src))
        ir = parsed[src][kname]
        form = canonical(ir)
        table[form] = make(form[0])
    return table


def lookup(ir) -> Optional[Binding]:
    return _table().get(canonical(ir))


_tls = threading.local()


def ticket_slot():
    """Per-thread reusable c_uint64 the C side writes the ticket into."""
    try:
        return _tls.ticket
    except AttributeError:
        _tls.ticket = ctypes.c_uint64()
        return _tls.ticket
