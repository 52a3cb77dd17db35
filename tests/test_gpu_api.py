"""API semantics of the CUDA runtime, mirroring the reference's buffer,
program, device and futures tests (pkg/tests/test_buffer.py,
test_program.py, test_device.py) on the B200 backend."""

from __future__ import annotations

import math
import random
import threading
import time

import numpy as np
import pytest

from paper_1810_11482_b200 import (
    BadArgsError,
    CompileError,
    InternalError,
    LaunchConfigError,
    NotBuiltError,
    OobAccessError,
    Runtime,
    UnknownGidError,
    copy,
    pinned_empty,
    when_all,
)
from paper_1810_11482_b200.bindings import kernel_source

pytestmark = pytest.mark.gpu


# -- discovery ------------------------------------------------------------------


def test_device_info(rt, dev):
    info = dev.device_info().get()
    assert info == dev.info
    assert info.name == "cuda0"
    assert info.capability == (10, 0)
    assert info.compute_units == 148
    assert info.memory_bytes > 170 * 10**9
    assert [d.info.name for d in rt.get_all_devices(10, 0).get()] == ["cuda0"]
    assert rt.get_all_devices(10, 1).get() == []


def test_stream_numbering():
    with Runtime(devices=[0]) as r:
        d = r.get_all_devices().get()[0]
        assert d.create_stream() == 1
        assert d.create_stream() == 2


def test_unknown_backend_rejected():
    with pytest.raises(BadArgsError):
        Runtime(backend="host")


def test_stale_gid_fails_token(rt, dev):
    buf = dev.create_buffer(8).get()
    rt.registry.unregister(buf.gid)
    with pytest.raises(Exception):
        buf.enqueue_read(0, 8).get(timeout=5)


# -- buffers --------------------------------------------------------------------------


def test_new_buffer_reads_zero(dev):
    buf = dev.create_buffer(4000).get()
    assert buf.enqueue_read_sync(0, 4000) == bytes(4000)


def test_out_of_memory_fails_the_token(dev):
    """A request beyond the 180 GB of HBM fails the create_buffer token with
    OutOfMemoryError (reference: the device's capacity check fails the
    token, device.py:217-228); the device stays usable."""
    from paper_1810_11482_b200 import OutOfMemoryError

    tok = dev.create_buffer(1 << 40)  # 1 TiB
    with pytest.raises(OutOfMemoryError):
        tok.get(timeout=60)
    assert dev.create_buffer(64).get().size_bytes == 64


def test_create_size_zero_rejected(dev):
    with pytest.raises(BadArgsError):
        dev.create_buffer(0)


def test_write_read_roundtrip_and_bounds(dev):
    buf = dev.create_buffer(16).get()
    buf.enqueue_write(0, b"\x01\x02\x03")
    assert buf.enqueue_read_sync(0, 3) == b"\x01\x02\x03"
    with pytest.raises(OobAccessError):
        buf.enqueue_write(15, b"ab")
    with pytest.raises(OobAccessError):
        buf.enqueue_read(1, 16)
    with pytest.raises(BadArgsError):
        buf.enqueue_read(-1, 2)
    assert buf.enqueue_read_sync(0, 0) == b""


def test_write_accepts_buffer_protocol(dev):
    buf = dev.create_buffer(64).get()
    buf.enqueue_write(0, np.arange(8, dtype=np.float64))
    buf.enqueue_write(0, bytearray(b"ab"))
    buf.enqueue_write(2, memoryview(b"cd"))
    buf.enqueue_write(4, [1, 2, 3])
    got = buf.enqueue_read_sync(0, 64)
    exp = bytearray(np.arange(8, dtype=np.float64).tobytes())
    exp[0:7] = b"abcd\x01\x02\x03"
    assert got == bytes(exp)


def test_random_offsets_bulk(dev):
    rng = random.Random(1234)
    size = 4096
    buf = dev.create_buffer(size).get()
    shadow = bytearray(size)
    for _ in range(2000):
        off = rng.randrange(size)
        ln = rng.randrange(size - off + 1)
        if rng.random() < 0.5:
            blob = rng.randbytes(ln)
            buf.enqueue_write(off, blob)
            shadow[off : off + ln] = blob
        else:
            assert buf.enqueue_read_sync(off, ln) == bytes(shadow[off : off + ln])
    assert buf.enqueue_read_sync(0, size) == bytes(shadow)


def test_stream_ordered_visibility_prefix(dev):
    buf = dev.create_buffer(4).get()
    reads = []
    for value in range(1, 65):
        buf.enqueue_write(0, bytes([value] * 4))
        reads.append((value, buf.enqueue_read(0, 4)))
    for value, tok in reads:
        assert tok.get(timeout=10) == bytes([value] * 4)


def test_disjoint_writes_two_streams_then_synchronize(dev):
    buf = dev.create_buffer(8).get()
    s1, s2 = dev.create_stream(), dev.create_stream()
    buf.enqueue_write(0, b"YYYY", s1)
    buf.enqueue_write(4, b"ZZZZ", s2)
    dev.synchronize().get(timeout=5)
    assert buf.enqueue_read_sync(0, 8) == b"YYYYZZZZ"


def test_large_pageable_write_is_staged_and_source_reusable(dev):
    n = 8 << 20
    data = bytearray(np.random.default_rng(1).integers(0, 256, n, dtype=np.uint8).tobytes())
    buf = dev.create_buffer(n).get()
    tok = buf.enqueue_write(0, data)
    expected = bytes(data)
    data[:] = bytes(n)  # the runtime owns a copy once the call returned
    tok.get()
    assert buf.enqueue_read_sync(0, n) == expected


def test_pinned_zero_copy_roundtrip(dev):
    n = 1 << 20
    src = pinned_empty(n * 8, np.float64)
    src[:] = np.random.default_rng(2).random(n)
    dst = pinned_empty(n * 8, np.float64)
    buf = dev.create_buffer(n * 8).get()
    buf.enqueue_write(0, src)
    tok = buf.enqueue_read_into(0, dst)
    assert tok.get() is dst
    assert np.array_equal(src, dst)


def test_read_rows_into_strided_pinned(dev):
    """Packed device rows land at a stride in a pinned host array (one DMA);
    misuse raises synchronously."""
    from paper_1810_11482_b200 import BadArgsError, OobAccessError, pinned_empty

    rows, w = 7, 40
    src = np.arange(rows * w, dtype=np.uint32)
    buf = dev.create_buffer(src.nbytes).get()
    buf.enqueue_write(0, src.tobytes())
    img = pinned_empty(3 * rows * w * 4, np.uint32)
    img[:] = 0xFFFFFFFF
    buf.enqueue_read_rows_into(0, img, w * 4, rows, dst_offset=w * 4, dst_pitch=3 * w * 4).get()
    exp = np.full((3 * rows, w), 0xFFFFFFFF, np.uint32)
    exp[1::3] = src.reshape(rows, w)
    assert np.array_equal(img.reshape(-1, w), exp)
    with pytest.raises(OobAccessError):
        buf.enqueue_read_rows_into(0, img, w * 4, rows + 1)
    with pytest.raises(BadArgsError):
        buf.enqueue_read_rows_into(0, img, w * 4, rows, dst_offset=0, dst_pitch=w * 4 - 4)
    with pytest.raises(BadArgsError):
        buf.enqueue_read_rows_into(0, np.empty(3 * rows * w, np.uint32), w * 4, rows)


def test_read_into_pageable(dev):
    buf = dev.create_buffer(1024).get()
    buf.enqueue_write(0, bytes(range(256)) * 4)
    out = bytearray(512)
    buf.enqueue_read_into(256, out).get()
    assert bytes(out) == (bytes(range(256)) * 2)


def test_copy_within_and_across_devices(rt, rt2, dev):
    src = dev.create_buffer(64).get()
    dst = dev.create_buffer(64).get()
    blob = bytes(range(64))
    src.enqueue_write(0, blob)
    src.copy_to(dst).get(timeout=5)
    assert dst.enqueue_read_sync(0, 64) == blob
    copy(src, 4, dst, 8, 8).get(timeout=5)
    assert dst.enqueue_read_sync(8, 8) == blob[4:12]
    with pytest.raises(OobAccessError):
        copy(src, 60, dst, 0, 8)
    d0, d1 = rt2.get_all_devices().get()
    a = d0.create_buffer(32).get()
    b = d1.create_buffer(32).get()
    a.enqueue_write(0, b"q" * 32)
    copy(a, 0, b, 0, 32).get(timeout=5)
    assert b.enqueue_read_sync(0, 32) == b"q" * 32


def test_copy_is_ordered_on_both_default_streams(dev):
    src = dev.create_buffer(1 << 20).get()
    dst = dev.create_buffer(1 << 20).get()
    for k in range(20):
        src.enqueue_write(0, bytes([k]) * (1 << 20))
        copy(src, 0, dst, 0, 1 << 20)
        tok = dst.enqueue_read(0, 16)
        assert tok.get() == bytes([k]) * 16


# -- programs --------------------------------------------------------------------------


def _sum_prog(dev):
    p = dev.create_program_with_source(kernel_source("sum")).get()
    return p


def test_create_program_defers_validation(dev):
    p = dev.create_program_with_source("kernel { this is garbage").get()
    with pytest.raises(CompileError):
        p.build("anything").get(timeout=5)


def test_build_errors(dev):
    p = _sum_prog(dev)
    with pytest.raises(CompileError, match="kernel not found"):
        p.build("nope").get(timeout=5)
    q = dev.create_program_with_source("kernel k(x : buffer_f64) { x[0] = mystery; }").get()
    with pytest.raises(CompileError, match="mystery"):
        q.build("k").get(timeout=5)


def test_run_before_build_and_arity_kind(dev):
    buf = dev.create_buffer(8).get()
    p = _sum_prog(dev)
    with pytest.raises(NotBuiltError):
        p.run([buf, buf, 1], "sum", (1, 1, 1), (1, 1, 1)).get(timeout=5)
    p.build("sum").get(timeout=5)
    with pytest.raises(BadArgsError):
        p.run([buf], "sum", (1, 1, 1), (1, 1, 1)).get(timeout=5)
    with pytest.raises(BadArgsError):
        p.run([buf, 3, buf], "sum", (1, 1, 1), (1, 1, 1)).get(timeout=5)
    with pytest.raises(BadArgsError):
        p.run([buf, buf, 2**32], "sum", (1, 1, 1), (1, 1, 1))
    with pytest.raises(BadArgsError):
        p.run([buf, buf, True], "sum", (1, 1, 1), (1, 1, 1))


def test_launch_config_rejected(dev):
    buf = dev.create_buffer(8).get()
    p = _sum_prog(dev)
    p.build("sum").get()
    with pytest.raises(LaunchConfigError):
        p.run([buf, buf, 1], "sum", (0, 1, 1), (1, 1, 1))
    with pytest.raises(LaunchConfigError):
        p.run([buf, buf, 1], "sum", (2**20, 1, 1), (2**13, 1, 1))


def test_buffer_on_other_device_rejected(rt2):
    d0, d1 = rt2.get_all_devices().get()
    here = d0.create_buffer(8).get()
    there = d1.create_buffer(8).get()
    p = d0.create_program_with_source(kernel_source("sum")).get()
    p.build("sum").get()
    with pytest.raises(BadArgsError):
        p.run([there, here, 1], "sum", (1, 1, 1), (1, 1, 1))


def test_kernel_oob_fails_token_with_index(dev):
    # stencil over n cells with buffers one cell short: first bad index n-1
    n = 100
    x = dev.create_buffer((n - 1) * 8).get()
    y = dev.create_buffer(n * 8).get()
    p = dev.create_program_with_source(kernel_source("stencil")).get()
    p.build("stencil").get()
    with pytest.raises(OobAccessError, match="99"):
        p.run([x, y, n], "stencil", (4, 1, 1), (32, 1, 1)).get(timeout=5)
    # sum reading past its input
    i = dev.create_buffer(40).get()
    r = dev.create_buffer(4).get()
    s = _sum_prog(dev)
    s.build("sum").get()
    with pytest.raises(OobAccessError, match="10"):
        s.run([i, r, 11], "sum", (1, 1, 1), (1, 1, 1)).get(timeout=5)


def test_unbound_kernel_goes_through_nvrtc(dev, monkeypatch):
    src = "kernel w(out : buffer_u32, a : scalar_u32) { out[0] = a * a; }"
    p = dev.create_program_with_source(src).get()
    p.build("w").get(timeout=120)
    out = dev.create_buffer(4).get()
    p.run([out, 4_000_000_000], "w", (1, 1, 1), (1, 1, 1)).get()
    assert np.frombuffer(out.enqueue_read_sync(0, 4), np.uint32)[0] == (4_000_000_000**2) % 2**32
    monkeypatch.setenv("OFL_NO_JIT", "1")
    q = dev.create_program_with_source(src).get()
    with pytest.raises(CompileError, match="sm_100a"):
        q.build("w").get()


def test_renamed_kernel_still_binds(dev):
    src = kernel_source("stencil").replace("kernel stencil(", "kernel heat_step(")
    p = dev.create_program_with_source(src).get()
    p.build("heat_step").get()
    x = dev.create_buffer(32).get()
    y = dev.create_buffer(32).get()
    x.enqueue_write(0, np.array([1.0, 2.0, 3.0, 4.0]).tobytes())
    p.run([x, y, 4], "heat_step", (1, 1, 1), (32, 1, 1))
    assert np.frombuffer(y.enqueue_read_sync(0, 32), np.float64).tolist() == [1.0, 4.0, 6.0, 4.0]


def test_int_coerces_to_f64_scalar(dev):
    n = 16
    A, B, C = (dev.create_buffer(n * 8).get() for _ in range(3))
    B.enqueue_write(0, np.ones(n).tobytes())
    C.enqueue_write(0, np.ones(n).tobytes())
    p = dev.create_program_with_source(kernel_source("stream")).get()
    p.build("triad").get()
    p.run([A, B, C, 3, n], "triad", (1, 1, 1), (32, 1, 1))
    assert np.frombuffer(A.enqueue_read_sync(0, n * 8), np.float64).tolist() == [4.0] * n


# -- futures over device operations -------------------------------------------------------


def test_then_runs_after_device_completion(dev):
    buf = dev.create_buffer(1 << 24).get()
    big = np.random.default_rng(0).integers(0, 256, 1 << 24, dtype=np.uint8).tobytes()
    seen = []
    done = threading.Event()
    tok = buf.enqueue_write(0, big)
    t2 = tok.then(lambda _: seen.append(threading.current_thread().name) or 7)
    t2.then(lambda _: done.set())
    assert done.wait(10)
    assert t2.get() == 7
    assert seen  # ran on the completion thread or inline


def test_done_polls_without_blocking(dev):
    buf = dev.create_buffer(1 << 26).get()
    tok = buf.enqueue_write(0, bytes(1 << 26))
    t0 = time.perf_counter()
    while not tok.done():
        assert time.perf_counter() - t0 < 10
    assert tok.is_ready()


def test_when_all_chain_device_tokens(dev):
    from paper_1810_11482_b200 import make_ready

    n = 1024
    A, B, C, D = (dev.create_buffer(n * 8).get() for _ in range(4))
    p = dev.create_program_with_source(kernel_source("stream")).get()
    p.build("triad").get()
    s1 = dev.create_stream()
    prev = make_ready(None)
    payload = pinned_empty(8)
    for k in range(5000):
        w = D.enqueue_write(0, payload, s1 if k % 2 else 0)
        r = p.run([A, B, C, 3.0, n], "triad", (4, 1, 1), (256, 1, 1))
        prev = when_all([prev, w, r])
    prev.get()
    assert prev.is_ready()
    fired = threading.Event()
    prev.then(lambda _: fired.set())
    assert fired.wait(5)


def test_when_all_armed_chain_fires(dev):
    from paper_1810_11482_b200 import make_ready

    buf = dev.create_buffer(1 << 22).get()
    prev = make_ready(None)
    for _ in range(2000):
        prev = when_all([prev, buf.enqueue_write(0, b"x" * 64)])
    fired = threading.Event()
    prev.then(lambda _: fired.set())
    assert fired.wait(10)


def test_when_all_first_error_wins(dev):
    buf = dev.create_buffer(8).get()
    p = _sum_prog(dev)
    bad = p.run([buf, buf, 1], "sum", (1, 1, 1), (1, 1, 1))  # not built
    good = buf.enqueue_write(0, b"12345678")
    with pytest.raises(NotBuiltError):
        when_all([good, bad]).get(timeout=5)


def test_synchronize_covers_all_streams(dev):
    buf = dev.create_buffer(1 << 24).get()
    streams = [dev.create_stream() for _ in range(4)]
    toks = [buf.enqueue_write(0, bytes(1 << 24), s) for s in streams]
    dev.synchronize().get(timeout=10)
    assert all(t.done() for t in toks)


def test_many_threads_enqueue_concurrently(dev):
    buf = dev.create_buffer(64 * 8).get()
    errors = []

    def worker(k):
        try:
            s = dev.create_stream()
            for i in range(200):
                buf.enqueue_write(k * 8, np.array([k * 1000 + i], np.float64), s).get()
        except Exception as exc:  # noqa: BLE001
            errors.append(exc)

    ts = [threading.Thread(target=worker, args=(k,)) for k in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors
    got = np.frombuffer(buf.enqueue_read_sync(0, 64), np.float64)
    assert got.tolist() == [k * 1000 + 199 for k in range(8)]


# -- multi-device on one GPU ------------------------------------------------------------------


def test_mandelbrot_cyclic_rows_two_devices(rt2):
    """Cyclic row split across devices, assembled on the host: identical to
    the single-device image (bit-exact)."""
    from paper_1810_11482_b200.bench.harness import mandelbrot_multi

    import oracle

    devices = rt2.get_all_devices().get()
    exp = oracle.mandelbrot(640, 360, max_iter=1000, threads=0).tobytes()
    for chunks in (1, 3, 8, 500):
        for interleave in (True, False):
            counts = mandelbrot_multi(devices, 640, 360, 1000, chunks=chunks,
                                      interleave=interleave)
            assert counts.tobytes() == exp, (chunks, interleave)


@pytest.mark.parametrize("w,h,bands", [(643, 357, 5), (640, 360, 1), (17, 9, 7), (1000, 3, 2),
                                       (333, 101, 200)])
def test_mandelbrot_chunked_ragged(dev, w, h, bands):
    """Chunked (interleaved and banded) Mandelbrot into the pinned image on
    ragged shapes (partial tiles, more chunks than rows): the image equals
    the oracle's, and a second frame through the same streams is identical."""
    from paper_1810_11482_b200.bench.harness import MandelbrotTiles

    import oracle

    exp = oracle.mandelbrot(w, h, max_iter=300, threads=0).tobytes()
    for interleave in (True, False):
        tiles = MandelbrotTiles([dev], w, h, 300, chunks=bands, interleave=interleave)
        for _ in range(2):
            tiles.image[:] = 0xFFFFFFFF
            assert tiles().tobytes() == exp, interleave


@pytest.mark.parametrize("chunks,interleave", [(8, True), (8, False), (16, True), (7, True)])
def test_mandelbrot_chunked_single_device_config3(dev, golden, chunks, interleave):
    """Config 3 on one device in chunks on two streams (read of chunk c
    overlapping chunk c+1), interleaved or banded rows: the reference's sha256."""
    import hashlib

    from paper_1810_11482_b200.bench.harness import mandelbrot_multi

    counts = mandelbrot_multi([dev], 7680, 4320, 2000, chunks=chunks, interleave=interleave)
    assert hashlib.sha256(counts.tobytes()).hexdigest() == golden["mandelbrot"][7]["sha256"]


def test_heat_multi_device_halo(rt2):
    from paper_1810_11482_b200.bench.harness import heat_multi

    import oracle

    devices = rt2.get_all_devices().get()
    x = np.random.default_rng(77).random(100_003)
    got = heat_multi(devices, x, 37)
    assert got.tobytes() == oracle.heat(x, 37, threads=0).tobytes()


def test_nccl_allreduce_single_rank(dev, rt):
    from paper_1810_11482_b200.collectives import Communicator

    comm = Communicator.single_process(rt, [dev])
    buf = dev.create_buffer(8).get()
    buf.enqueue_write(0, np.array([2.5]).tobytes())
    comm.allreduce([buf], count=1, dtype="f64").get()
    assert np.frombuffer(buf.enqueue_read_sync(0, 8), np.float64)[0] == 2.5


def test_when_all_runs_read_landing(dev):
    """A pageable enqueue_read_into lands through a staging block in its
    token's finish step: gating on when_all(...).get() / then() / done() must
    make the bytes visible (reference futures.py:189-216)."""
    n = 3 << 20
    payload = np.random.default_rng(5).integers(0, 256, n, dtype=np.uint8)
    buf = dev.create_buffer(n).get()
    buf.enqueue_write(0, payload)
    out = bytearray(n)
    assert when_all([buf.enqueue_read_into(0, out)]).get(timeout=30) is None
    assert bytes(out) == payload.tobytes()
    out2 = bytearray(n)
    seen, fired = [], threading.Event()
    when_all([buf.enqueue_read_into(0, out2), buf.enqueue_write(0, payload)]).then(
        lambda _: (seen.append(bytes(out2) == payload.tobytes()), fired.set()))
    assert fired.wait(30) and seen == [True]
    out3 = np.zeros(n, np.uint8)
    agg = when_all([buf.enqueue_read_into(0, out3)])
    t0 = time.time()
    while not agg.done():
        assert time.time() - t0 < 30
    assert out3.tobytes() == payload.tobytes()


def test_launch_and_write_plans_track_arguments(rt, dev):
    """The handles' launch / pinned-write plans (handles.py) reuse a resolved
    call only for the same argument objects: a changed scalar, a new pinned
    payload, another stream or an unregistered buffer take the full path."""
    n = 4096
    prog = dev.create_program_with_source(kernel_source("stream")).get()
    prog.build("triad").get()
    A, B, C = (dev.create_buffer(n * 8).get() for _ in range(3))
    b = pinned_empty(n * 8, np.float64)
    c = pinned_empty(n * 8, np.float64)
    b[:] = np.arange(n)
    c[:] = 1.0
    B.enqueue_write(0, b)
    C.enqueue_write(0, c)
    args = [A, B, C, 3.0, n]
    grid, block = (n // 256, 1, 1), (256, 1, 1)
    for s in (3.0, 3.0, 5.0, 5.0, 0.5):
        args[3] = s
        prog.run(args, "triad", grid, block)
        got = np.frombuffer(A.enqueue_read(0, n * 8).get(), np.float64)
        assert np.array_equal(got, np.arange(n) + s), s
    s1 = dev.create_stream()
    c[:] = 2.0
    C.enqueue_write(0, c)  # same array again, new contents
    prog.run(args, "triad", grid, block, s1).get()
    got = np.frombuffer(A.enqueue_read(0, n * 8).get(), np.float64)
    assert np.array_equal(got, np.arange(n) + 0.5 * 2.0)
    rt.registry.unregister(C.gid)
    with pytest.raises(UnknownGidError):
        prog.run(args, "triad", grid, block).get()


@pytest.mark.gpu
def test_pci_bus_id_and_local_cpus():
    """The GPU's PCI address names its sysfs node; its CPU list (if the
    platform reports one) intersects the CPUs this process may use."""
    import os

    from paper_1810_11482_b200 import device

    bus = device.pci_bus_id(0)
    assert len(bus) == 12 and bus == bus.lower() and bus[4] == ":" and bus[10] == "."
    cpus = device.local_cpus(0)
    if os.path.isdir(os.path.join("/sys/bus/pci/devices", bus)) and cpus is not None:
        assert cpus & os.sched_getaffinity(0)
