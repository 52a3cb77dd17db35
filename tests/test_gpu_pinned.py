"""Config 2 and config 4 on the B200 against outputs the REFERENCE produced
(tests/golden/golden_long.json, written by ``make_golden.py --long`` running
offloadrt's host backend): the full 2^28-cell x 1000-step heat equation
(stencil.k iterated, ping-pong; harness.py:199-230 inputs) bit for bit, the
2^20 x 1000 case bit for bit, and the fp32 dot product within 1e-12
relative of the reference executor's sequential fp64 sum of the exact
products (the BASELINE tolerance is 1e-5)."""

from __future__ import annotations

import hashlib
import json
import math
import os

import numpy as np
import pytest

from flows import device_heat

pytestmark = pytest.mark.gpu

LONG = os.path.join(os.path.dirname(__file__), "golden", "golden_long.json")


def _long():
    with open(LONG) as fh:
        return json.load(fh)


def _heat_cases():
    return [(c["n"], c["steps"]) for c in _long()["heat"]]


@pytest.mark.parametrize("n,steps", _heat_cases())
def test_heat_builtin_matches_reference(dev, n, steps):
    case = next(c for c in _long()["heat"] if c["n"] == n and c["steps"] == steps)
    x = np.random.default_rng(case["seed"]).random(n)
    out = device_heat(dev, x, steps)
    del x
    assert hashlib.sha256(out).hexdigest() == case["sha256"]
    assert float(np.frombuffer(out, np.float64).sum()) == case["sum"]


def test_dot_f32_matches_reference(dev):
    prog = dev.create_builtin_program().get()
    prog.build("dot_f32").get()
    for case in _long()["dot"]:
        n = case["n"]
        rng = np.random.default_rng(case["seed"])
        a = rng.random(n, dtype=np.float32)
        b = rng.random(n, dtype=np.float32)
        A, B, R = dev.create_buffer(n * 4).get(), dev.create_buffer(n * 4).get(), dev.create_buffer(8).get()
        A.enqueue_write(0, a)
        B.enqueue_write(0, b)
        prog.run([A, B, R, n], "dot_f32", (math.ceil(n / 256), 1, 1), (256, 1, 1))
        got = float(np.frombuffer(R.enqueue_read(0, 8).get(), np.float64)[0])
        ref = case["result"]
        assert abs(got - ref) <= 1e-5 * ref      # BASELINE's stated fp32 tolerance
        assert abs(got - ref) <= 1e-12 * ref     # what fp64 accumulation gives


@pytest.mark.parametrize("n,steps", _heat_cases())
def test_heat_chunks_match_reference(dev, n, steps):
    """bench.HeatChunks (independent halo-extended pieces, transfers
    overlapped with the steps) reproduces the reference's field bit for bit."""
    from paper_1810_11482_b200 import pinned_empty
    from paper_1810_11482_b200.bench import HeatChunks

    case = next(c for c in _long()["heat"] if c["n"] == n and c["steps"] == steps)
    x = pinned_empty(n * 8, np.float64)
    x[:] = np.random.default_rng(case["seed"]).random(n)
    out = pinned_empty(n * 8, np.float64)
    HeatChunks(dev, n, steps, chunks=16, sets=3)(x, out)
    assert hashlib.sha256(out).hexdigest() == case["sha256"]


@pytest.mark.parametrize("n,steps,chunks,sets", [
    (3, 5, 4, 2),          # smaller than one halo: a single piece
    (1000, 7, 9, 2),       # ragged pieces
    (4097, 0, 5, 3),       # zero steps: the input comes back
    (20011, 333, 7, 1),    # one buffer pair for every piece (stream order reuses it)
    (65536, 1, 64, 4),     # one step, many pieces
])
def test_heat_chunks_edge_cases(dev, n, steps, chunks, sets):
    import oracle
    from paper_1810_11482_b200 import pinned_empty
    from paper_1810_11482_b200.bench import HeatChunks

    x = pinned_empty(n * 8, np.float64)
    x[:] = np.random.default_rng(n + steps).random(n)
    out = pinned_empty(n * 8, np.float64)
    HeatChunks(dev, n, steps, chunks=chunks, sets=sets)(x, out)
    assert np.array_equal(out.view(np.uint64), oracle.heat(np.array(x), steps).view(np.uint64))


def test_heat_chunks_pageable_host_arrays(dev):
    """Plain numpy arrays in and out (staged writes, chunked reads into the
    caller's array), two buffer pairs reused in stream order."""
    import oracle
    from paper_1810_11482_b200.bench import HeatChunks

    n, steps = 3 << 20, 40
    x = np.random.default_rng(11).random(n)
    out = np.zeros(n)
    HeatChunks(dev, n, steps, chunks=12, sets=2)(x, out)
    assert np.array_equal(out.view(np.uint64), oracle.heat(x.copy(), steps).view(np.uint64))
