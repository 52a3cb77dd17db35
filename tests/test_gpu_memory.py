"""Stream-ordered device memory (csrc/ofl_runtime.cu: ofl_malloc / ofl_free
on the device's memory pool): dropping a buffer neither stalls nor waits for
other streams' in-flight work, and the memory is not reused before the work
enqueued ahead of the free has finished."""

from __future__ import annotations

import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _warm(rt, dev):
    """First use of each allocation path (driver entry points, the reaper
    thread, pool setup) outside the measured part, and one released buffer
    of each size the tests allocate: a first-time physical allocation may
    wait behind queued work inside the driver; steady-state allocations
    reuse released memory and make no driver call.  The memory earlier
    tests released is handed back first (Runtime.trim_memory), so these
    allocations find room without a reclaim that would empty the caches."""
    dev.synchronize().get()
    rt.trim_memory()
    for size in (32 << 20, 4 << 20, 4 << 20, 1 << 20, 1 << 10):
        b = dev.create_buffer(size).get()
        rt.registry.unregister(b.gid)
        del b
    dev.synchronize().get()
    time.sleep(0.2)  # the reaper has passed their (already complete) fences


def _long_heat(dev, stream: int, n: int = 1 << 27, steps: int = 6000):
    """A kernel chain of ~90 ms on `stream` (heat builtin, passes of ~1.4 ms)."""
    X, Y = dev.create_buffer(n * 8).get(), dev.create_buffer(n * 8).get()
    X.enqueue_write(0, np.full(n, 0.5), stream).get()
    prog = dev.create_builtin_program().get()
    prog.build("heat").get()
    tok = prog.run([X, Y, n, steps], "heat", (n // 256, 1, 1), (256, 1, 1), stream)
    return tok, (X, Y)


def test_free_does_not_stall_other_streams(rt, dev):
    _warm(rt, dev)
    s1 = dev.create_stream()
    tok, keep = _long_heat(dev, s1)
    times = []
    for size in (4 << 20, 4 << 20, 1 << 10, 1 << 10):  # a VMM mapping and a pool buffer, twice
        t0 = time.perf_counter()
        tmp = dev.create_buffer(size).get()      # allocate + zero fill on the internal stream
        t1 = time.perf_counter()
        rt.registry.unregister(tmp.gid)          # last reference: ofl_free (stream-ordered)
        del tmp
        times.append((round((t1 - t0) * 1e3, 2), round((time.perf_counter() - t1) * 1e3, 2)))
    # the frees are enqueued behind the heat chain, not waited for (a
    # cudaFree would have synchronised the device: ~90 ms, the chain done);
    # an allocation's zero fill runs on the high-priority internal stream at
    # the chain's next pass boundary
    assert all(drop < 10.0 for _, drop in times), times
    assert not tok.done(), f"dropping buffers waited for another stream's kernel: {times}"
    tok.get()


def test_freed_memory_not_reused_before_prior_work(rt, dev):
    """A buffer dropped while a kernel still writes it: a new allocation of
    the same size must not see (or be clobbered by) that kernel's writes."""
    s1, s2 = dev.create_stream(), dev.create_stream()
    n = 1 << 26
    for _ in range(3):
        tok, (X, Y) = _long_heat(dev, s1, n=n, steps=400)
        rt.registry.unregister(X.gid)
        rt.registry.unregister(Y.gid)
        del X, Y
        Z = dev.create_buffer(n * 8).get()       # zero-filled, maybe the same pool memory
        pattern = np.arange(n, dtype=np.float64)
        Z.enqueue_write(0, pattern, s2).get()
        tok.get()                                 # the heat chain has finished writing
        got = np.frombuffer(Z.enqueue_read(0, n * 8, s2).get(), np.float64)
        assert np.array_equal(got, pattern)


def test_trim_memory_returns_released_memory(rt, dev):
    """Runtime.trim_memory: released buffers' memory (cached VMM mappings,
    pool blocks) goes back to the device."""
    import torch

    dev.synchronize().get()
    rt.trim_memory()
    free0, _ = torch.cuda.mem_get_info(0)
    bufs = [dev.create_buffer(1 << 30).get() for _ in range(4)] + [dev.create_buffer(1 << 12).get()]
    for b in bufs:
        rt.registry.unregister(b.gid)
    del bufs, b
    dev.synchronize().get()
    time.sleep(0.2)
    held, _ = torch.cuda.mem_get_info(0)
    assert held <= free0 - (4 << 30) + (64 << 20)   # cached for reuse, not yet returned
    rt.trim_memory()
    free1, _ = torch.cuda.mem_get_info(0)
    assert free1 >= free0 - (64 << 20)


def test_allocation_after_free_does_not_wait(rt, dev):
    """Allocations go to their own stream: they never queue behind a free's
    fence waits."""
    _warm(rt, dev)
    s1 = dev.create_stream()
    tok, keep = _long_heat(dev, s1)
    tmp = dev.create_buffer(1 << 20).get()
    rt.registry.unregister(tmp.gid)
    del tmp
    t0 = time.perf_counter()
    fresh = dev.create_buffer(32 << 20).get()
    dt = time.perf_counter() - t0
    assert not tok.done()
    assert fresh.enqueue_read(0, 16).get() == bytes(16)
    tok.get()
    assert dt < 0.05, dt


def test_released_memory_is_reclaimed_for_other_sizes(rt, dev):
    """Released VMM mappings are kept for reuse by same-size allocations;
    an allocation of another size that does not fit otherwise gets them
    back (ofl_runtime.cu reclaim: pool trim + cached mappings unmapped)."""
    import torch

    free0, total = torch.cuda.mem_get_info(0)
    piece = 8 << 30
    count = int(free0 * 0.7) // piece
    held = [dev.create_buffer(piece).get() for _ in range(count)]
    for b in held:
        rt.registry.unregister(b.gid)
    del held, b
    dev.synchronize().get()
    time.sleep(0.2)
    # larger than what is free unless the released mappings are unmapped
    big = int(free0 * 0.8)
    b = dev.create_buffer(big).get()
    assert b.enqueue_read(big - 16, 16).get() == bytes(16)
    rt.registry.unregister(b.gid)
    del b
    small = dev.create_buffer(1 << 10).get()
    assert small.enqueue_read(0, 16).get() == bytes(16)

