"""Bound kernels' out-of-range pre-checks against a brute-force restatement
of the reference executor's abort protocol (kernel/codegen.py: items run in
gtid order; per item the store index is checked first, then the loads left
to right; the first failing index is reported).  CPU only: the checks are
host logic and need no device."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1810_11482_b200 import bindings

M32 = 0xFFFFFFFF


class FakeBuf:
    def __init__(self, elems: int):
        self.n = elems

    def elements(self, kind: str) -> int:
        return self.n


def brute_stencil2d(w, h, lx, ly, items):
    cells = (w * h) & M32
    for g in range(min(cells, items)):
        if g >= ly:
            return g
        row, col = divmod(g, w)
        if row == 0 or row == h - 1 or col == 0 or col == w - 1:
            loads = (g,)
        else:
            loads = ((g - w) & M32, g - 1, g + 1, (g + w) & M32)
        for idx in loads:
            if idx >= lx:
                return idx
    return None


def brute_stencil(n, lx, ly, items):
    for g in range(min(n, items)):
        if g >= ly:
            return g
        loads = (g,) if g == 0 or g == ((n - 1) & M32) else (g - 1, g, g + 1)
        for idx in loads:
            if idx >= lx:
                return idx
    return None


def test_stencil2d_oob_matches_executor_order():
    rng = np.random.default_rng(0)
    for _ in range(3000):
        w = int(rng.integers(1, 12))
        h = int(rng.integers(1, 12))
        cells = w * h
        lx = int(rng.integers(0, cells + 3))
        ly = int(rng.integers(0, cells + 3))
        items = int(rng.integers(0, cells + 5))
        got = bindings._stencil2d_oob((FakeBuf(lx), FakeBuf(ly), w, h), items)
        assert got == brute_stencil2d(w, h, lx, ly, items), (w, h, lx, ly, items)


def test_stencil_oob_matches_executor_order():
    rng = np.random.default_rng(1)
    for _ in range(3000):
        n = int(rng.integers(1, 40))
        lx = int(rng.integers(0, n + 3))
        ly = int(rng.integers(0, n + 3))
        items = int(rng.integers(0, n + 5))
        got = bindings._stencil_oob((FakeBuf(lx), FakeBuf(ly), n), items)
        assert got == brute_stencil(n, lx, ly, items), (n, lx, ly, items)


@pytest.mark.parametrize("name", ["stream", "stencil", "stencil2d", "mandelbrot", "sum", "partition"])
def test_every_bundled_kernel_binds(name):
    """Each bundled .k program is recognised by canonical form and bound to
    its sm_100a kernel (never silently sent to the generic path)."""
    from paper_1810_11482_b200.kernel import parse_and_validate

    irs = parse_and_validate(bindings.kernel_source(name))
    for ir in irs.values():
        assert bindings.lookup(ir) is not None, (name, ir.name)
