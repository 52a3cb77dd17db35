"""Pin the CPU oracle to the reference: every golden vector in
tests/golden/golden.json was produced by running the reference package
itself (tests/golden/make_golden.py).  Both restatements (C and numpy) must
reproduce them exactly (bit-for-bit; partition within the reference's own
1e-12 bound)."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import oracle
from oracle import numpy_oracle as npo


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_stencil_hand_case(golden):
    case = golden["stencil"][0]
    x = np.array(case["input"])
    assert oracle.stencil(x).tolist() == case["output"] == [1.0, 4.0, 6.0, 4.0]
    assert npo.stencil(x).tolist() == case["output"]
    assert npo.stencil_seq(list(x)) == case["output"]


@pytest.mark.parametrize("idx", [1, 2, 3])
def test_stencil_random(golden, idx):
    case = golden["stencil"][idx]
    x = np.random.default_rng(case["seed"]).random(case["n"])
    y = oracle.stencil(x, threads=0)
    assert sha(y) == case["sha256"]
    assert sha(npo.stencil(x)) == case["sha256"]
    if "output_hex" in case:
        assert y.tobytes().hex() == case["output_hex"]


@pytest.mark.parametrize("idx", [0, 1])
def test_heat_steps(golden, idx):
    case = golden["heat"][idx]
    x = np.random.default_rng(case["seed"]).random(case["n"])
    assert sha(oracle.heat(x, case["steps"], threads=0)) == case["sha256"]
    if case["n"] <= 4096:
        assert sha(npo.heat(x, case["steps"])) == case["sha256"]


@pytest.mark.parametrize("idx", range(8))
def test_stencil2d_step(golden, idx):
    """stencil2d.k as the reference executes it: grids with odd widths, a
    1-wide grid, a partial launch (items < w*h leaves the rest zero)."""
    case = golden["stencil2d"]["step"][idx]
    w, h = case["w"], case["h"]
    x = np.random.default_rng(case["seed"]).random(w * h)
    y = oracle.stencil2d(x, w, h, items=case["items"], threads=0)
    assert sha(y) == case["sha256"]
    if case["items"] is None:
        assert sha(npo.stencil2d(x, w, h)) == case["sha256"]
    if "output" in case:
        assert x.tolist() == case["input"] and y.tolist() == case["output"]


@pytest.mark.parametrize("idx", [0, 1])
def test_heat2d_steps(golden, idx):
    case = golden["stencil2d"]["heat"][idx]
    w, h = case["w"], case["h"]
    x = np.random.default_rng(case["seed"]).random(w * h)
    assert sha(oracle.heat2d(x, w, h, case["steps"], threads=0)) == case["sha256"]


def test_sum_known_answers(golden):
    for case in golden["sum"]:
        if "values" in case:
            v = np.array(case["values"], dtype=np.uint32)
        else:
            v = np.random.default_rng(case["seed"]).integers(
                0, 2**32, size=case["n"], dtype=np.uint32
            )
        assert oracle.sum_u32(v, threads=0) == case["result"]
        assert oracle.sum_u32(v, threads=1) == case["result"]
        assert npo.sum_u32(v) == case["result"]
    assert golden["sum"][0]["result"] == 4
    assert golden["sum"][1]["result"] == 1000


@pytest.mark.parametrize("idx", range(6))
def test_mandelbrot_small(golden, idx):
    case = golden["mandelbrot"][idx]
    w, h, it = case["width"], case["height"], case["max_iter"]
    counts = oracle.mandelbrot(w, h, tuple(case["viewport"]), case["esc"], it, threads=0)
    assert sha(counts) == case["sha256"]
    if "counts" in case:
        assert counts.tolist() == case["counts"]
    if w * h <= 4096:
        assert npo.mandelbrot(w, h, tuple(case["viewport"]), it).tolist() == case["counts"]


def test_mandelbrot_hand_pixels(golden):
    # c = 1+0i escapes at count 3 (reference test_kernel_lang.py:348-359)
    assert golden["mandelbrot"][4]["counts"][4] == 3 == npo.mandelbrot_pixel(1.0, 0.0, 64)
    # c = 0 never escapes (test_bench.py:316-323)
    assert golden["mandelbrot"][5]["counts"][4] == 50


def test_mandelbrot_960x540_2000(golden):
    case = golden["mandelbrot"][6]
    counts = oracle.mandelbrot(960, 540, max_iter=2000, threads=0)
    assert sha(counts) == case["sha256"]
    assert int(counts.astype(np.uint64).sum()) == case["sum"]


def test_mandelbrot_full_config3(golden):
    """BASELINE config 3 at full size: 7680x4320, max_iter 2000."""
    case = golden["mandelbrot"][7]
    assert case["width"] == 7680 and case["max_iter"] == 2000
    counts = oracle.mandelbrot(7680, 4320, max_iter=2000, threads=0)
    assert sha(counts) == case["sha256"]
    assert int(counts.astype(np.uint64).sum()) == case["sum"] == 11_291_094_557


def test_mandelbrot_cyclic_rows_compose():
    """Multi-GPU split: rows r mod G on device G; the union is the image."""
    full = oracle.mandelbrot(64, 48, max_iter=300, threads=0)
    parts = np.zeros_like(full)
    for g in range(3):
        oracle.mandelbrot(64, 48, max_iter=300, row_first=g, row_step=3, out=parts, threads=2)
    assert np.array_equal(full, parts)


def test_partition(golden):
    for case in golden["partition"]:
        out = oracle.partition(case["offset"], case["count"], threads=0)
        assert np.abs(out - 1.0).max() <= 1e-12
        if "output_hex" in case:
            ref = np.frombuffer(bytes.fromhex(case["output_hex"]), np.float64)
            assert np.abs(out - ref).max() <= 1e-12
            small = npo.partition(case["offset"], min(case["count"], 256))
            assert np.abs(small - ref[: small.size]).max() <= 1e-12


def test_stream_ops(golden):
    rng = np.random.default_rng(401)
    n = 1 << 20
    b, c = rng.random(n), rng.random(n)
    for case in golden["stream"]:
        op, s = case["op"], case["scalar"]
        a = oracle.stream(op, b, c, s, threads=0)
        assert sha(a) == case["sha256"], op
        assert sha(npo.stream(op, b, c, s)) == case["sha256"], op


def test_dot_oracles_agree():
    rng = np.random.default_rng(5)
    a = rng.random(300_001, dtype=np.float32)
    b = rng.random(300_001, dtype=np.float32)
    x = oracle.dot_f32(a, b, threads=0)
    assert x == oracle.dot_f32(a, b, threads=1)  # fixed chunking: thread-count independent
    assert abs(x - npo.dot_f32(a, b)) <= 1e-12 * abs(x)  # numpy sums pairwise
    exact = float(np.dot(a.astype(np.float64), b.astype(np.float64)))
    assert abs(x - exact) <= 1e-12 * abs(exact)


# -- golden_long.json: the reference itself on config 2 / config 4 work ---------------

def _long():
    import json
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", "golden_long.json")) as fh:
        return json.load(fh)


def test_dot_seq_oracle_matches_reference_bit_for_bit():
    """The reference executor's dot (dot_seq in make_golden.py: f64 buffers
    holding fp32 values, index order) reproduced exactly by oracle.dot_f32_seq;
    the chunked oracle the GPU tests use stays within 1e-12 of it."""
    for case in _long()["dot"]:
        rng = np.random.default_rng(case["seed"])
        a = rng.random(case["n"], dtype=np.float32)
        b = rng.random(case["n"], dtype=np.float32)
        assert oracle.dot_f32_seq(a, b) == case["result"] == float.fromhex(case["result_hex"])
        assert abs(oracle.dot_f32(a, b, threads=0) - case["result"]) <= 1e-12 * case["result"]


def test_heat_1000_steps_oracle_matches_reference():
    """2^20 cells x 1000 steps of the reference's stencil.k, ping-pong, run
    by the reference executor (golden_long.json) == oracle.heat."""
    for case in _long()["heat"]:
        if case["n"] > 1 << 20:
            continue  # 2^28 x 1000: GPU test only (tests/test_gpu_pinned.py)
        x = np.random.default_rng(case["seed"]).random(case["n"])
        assert sha(oracle.heat(x, case["steps"], threads=0)) == case["sha256"]
