"""Kernels with no hand-written binding run through the NVRTC path
(kernel/cuda_codegen.py + csrc/ofl_jit.cu).  Expected outputs and errors are
the reference executor's (tests/golden/golden.json "lang", produced by
running the reference on the same programs and inputs); the cases mirror the
reference's test_kernel_lang.py semantics tests (u32 wrap and floor
division, division by zero, OOB index reporting incl. the wrapped -1 index,
builtins linearisation, short-circuit, scoped locals, loop rebinding, u32()
casts)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1810_11482_b200 import InternalError, OobAccessError

pytestmark = pytest.mark.gpu

_ERR = {"InternalError": InternalError, "OobAccessError": OobAccessError}


def _uses_libm(src: str) -> bool:
    return "sin(" in src or "cos(" in src


@pytest.mark.parametrize("idx", range(15))
def test_lang_case_matches_reference(dev, golden, idx):
    case = golden["lang"][idx]
    prog = dev.create_program_with_source(case["source"]).get()
    prog.build(case["kernel"]).get(timeout=120)
    handles = []
    for (kind, n), init in zip(case["buffers"], case["inputs_hex"]):
        h = dev.create_buffer(len(bytes.fromhex(init))).get()
        h.enqueue_write(0, bytes.fromhex(init))
        handles.append(h)
    tok = prog.run(handles + case["scalars"], case["kernel"], tuple(case["grid"]), tuple(case["block"]))
    if case["error"]:
        cls, msg = case["error"]
        with pytest.raises(_ERR[cls]) as info:
            tok.get(timeout=60)
        assert str(info.value) == msg
    else:
        tok.get(timeout=60)
    for (kind, n), h, want in zip(case["buffers"], handles, case["outputs_hex"]):
        got = h.enqueue_read_sync(0, h.size_bytes)
        if kind == "f64" and _uses_libm(case["source"]):
            g = np.frombuffer(got, np.float64)
            w = np.frombuffer(bytes.fromhex(want), np.float64)
            assert np.allclose(g, w, rtol=1e-12, atol=1e-12)
        else:
            assert got.hex() == want


def test_jit_kernel_cached_and_reusable(dev):
    src = "kernel sq(x : buffer_f64, n : scalar_u32) { if (gtid < n) { x[gtid] = x[gtid] * x[gtid]; } }"
    p1 = dev.create_program_with_source(src).get()
    p1.build("sq").get(timeout=120)
    p2 = dev.create_program_with_source(src).get()
    p2.build("sq").get(timeout=5)  # cached module
    n = 100_000
    x = np.random.default_rng(0).random(n)
    X = dev.create_buffer(n * 8).get()
    X.enqueue_write(0, x)
    for p in (p1, p2):
        p.run([X, n], "sq", ((n + 255) // 256, 1, 1), (256, 1, 1))
    got = np.frombuffer(X.enqueue_read_sync(0, n * 8), np.float64)
    assert got.tobytes() == ((x * x) * (x * x)).tobytes()


def test_jit_smallest_failing_gtid_reported(dev):
    src = "kernel o(out : buffer_f64, n : scalar_u32) { out[gtid * 3] = 1.0; }"
    p = dev.create_program_with_source(src).get()
    p.build("o").get(timeout=120)
    buf = dev.create_buffer(100 * 8).get()
    with pytest.raises(OobAccessError, match="kernel buffer index 102 out of range"):
        p.run([buf, 0], "o", (4, 1, 1), (256, 1, 1)).get()


def test_fuzzed_kernels_match_reference(dev, golden):
    """150 random well-typed kernels from the reference's own generator
    (tests/golden/make_golden.py --only-fuzz), one work item each: the
    NVRTC-compiled kernel reproduces the reference executor's final buffer
    states bit for bit, and its abort (OOB index, division by zero, cast
    range) with the same error type and message."""
    failures = []
    for i, case in enumerate(golden["fuzz"]):
        prog = dev.create_program_with_source(case["source"]).get()
        prog.build("fuzzed").get(timeout=120)
        handles, args = [], []
        for tag, kind, value in case["args"]:
            if tag == "buf":
                h = dev.create_buffer(len(bytes.fromhex(value))).get()
                h.enqueue_write(0, bytes.fromhex(value))
                handles.append(h)
                args.append(h)
            else:
                args.append(value)
        tok = prog.run(args, "fuzzed", (1, 1, 1), (1, 1, 1))
        err = None
        try:
            tok.get(timeout=60)
        except (InternalError, OobAccessError) as exc:
            err = [type(exc).__name__, str(exc)]
        outs = [h.enqueue_read_sync(0, h.size_bytes).hex() for h in handles]
        if err != case["error"] or outs != case["outputs_hex"]:
            failures.append((i, err, case["error"], case["source"]))
    assert not failures, f"{len(failures)} of {len(golden['fuzz'])} differ; first: {failures[0]}"


def test_jit_abort_fails_when_all_and_then(dev):
    """An NVRTC kernel's abort is found by its token's finish step (the error
    record read back); when_all and then() over the aggregate must run it and
    fail with the same error (reference futures.py:189-216)."""
    import threading

    from paper_1810_11482_b200 import when_all

    src = "kernel o(out : buffer_f64, n : scalar_u32) { out[gtid * 3] = 1.0; }"
    p = dev.create_program_with_source(src).get()
    p.build("o").get(timeout=120)
    buf = dev.create_buffer(100 * 8).get()
    msg = "kernel buffer index 102 out of range"
    with pytest.raises(OobAccessError, match=msg):
        when_all([buf.enqueue_write(0, b"\0" * 8), p.run([buf, 0], "o", (4, 1, 1), (256, 1, 1))]).get()
    with pytest.raises(OobAccessError, match=msg):
        when_all([when_all([p.run([buf, 0], "o", (4, 1, 1), (256, 1, 1))])]).get(timeout=30)
    seen, fired = [], threading.Event()
    agg = when_all([p.run([buf, 0], "o", (4, 1, 1), (256, 1, 1))])
    agg.then(lambda _: seen.append("ran")).then(lambda _: None)._on_done(
        lambda t: (seen.append(str(t.error())), fired.set()))
    assert fired.wait(30)
    assert seen and msg in seen[-1] and "ran" not in seen
    tok = p.run([buf, 0], "o", (4, 1, 1), (256, 1, 1))
    while not when_all([tok]).done():
        pass
    assert when_all([tok]).is_failed() and msg in str(tok.error())
