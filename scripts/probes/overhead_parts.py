"""Probe: host cost of each call in a futurized step (config 5), issue only,
on the B200 box: enqueue_write (8 B pinned), program.run (triad N=1024),
when_all over (prev, w, r), get() on a finished aggregate; and the raw C
chain synchronised every step for comparison.  Measured (round 2):
enqueue_write 2.1 us, program.run 4.7 us (of which ~3.3 us inside
ofl_stream_op: the driver's launch), when_all 0.6 us, get 0.04 us; a step
synchronised every time 13.8 us vs 10.5 us raw."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

from paper_1810_11482_b200 import Runtime, make_ready, pinned_empty, when_all  # noqa: E402
from paper_1810_11482_b200.bindings import kernel_source  # noqa: E402

K = 300  # below the launch queue depth: host issue cost, not GPU throughput
with Runtime(devices=[0]) as rt:
    dev = rt.get_all_devices().get()[0]
    n = 1024
    A, B, C, D = (dev.create_buffer(n * 8).get() for _ in range(4))
    prog = dev.create_program_with_source(kernel_source("stream")).get()
    prog.build("triad").get()
    payload = pinned_empty(8)
    payload[:] = 1
    args = [A, B, C, 3.0, n]
    grid, block = ((n + 255) // 256, 1, 1), (256, 1, 1)

    def timed(fn, k=K):
        dev.synchronize().get()
        t0 = time.perf_counter()
        fn(k)
        t1 = time.perf_counter()
        dev.synchronize().get()
        return (t1 - t0) / k * 1e6

    def writes(k):
        for _ in range(k):
            D.enqueue_write(0, payload)

    def runs(k):
        for _ in range(k):
            prog.run(args, "triad", grid, block)

    w = D.enqueue_write(0, payload)
    r = prog.run(args, "triad", grid, block)
    dev.synchronize().get()

    def alls(k):
        prev = make_ready(None)
        for _ in range(k):
            prev = when_all([prev, w, r])

    done = when_all([w, r])
    done.get()

    def gets(k):
        for _ in range(k):
            done.get()

    def step_sync(k):
        for _ in range(k):
            D.enqueue_write(0, payload)
            prog.run(args, "triad", grid, block).get()

    for name, fn in (("enqueue_write", writes), ("program.run", runs), ("when_all", alls),
                     ("get (done)", gets)):
        timed(fn, 300)
        print(f"{name:16s} " + " ".join(f"K={k}: {timed(fn, k):.3f}" for k in (20, 100, 300))
              + " us/call (issue only)")
    import cProfile
    import pstats
    cProfile.run("runs(300)", "/tmp/runs.prof")
    pstats.Stats("/tmp/runs.prof").sort_stats("tottime").print_stats(8)
    print(f"{'write+run.get':16s} {timed(step_sync, 2000):.3f} us/step (sync each step)")
    from paper_1810_11482_b200 import _native
    lib = _native.load()
    st = rt.device_objects()[0].stream(0)
    secs = ctypes.c_double()
    ptrs = [rt.local._buffer(x.gid).ptr for x in (A, B, C)]
    dptr = rt.local._buffer(D.gid).ptr
    for mode, label in ((2, "raw sync each"),):
        lib.ofl_bench_raw_chain(st.ptr, dptr, payload.ctypes.data, 8, *ptrs, n, 5000, mode, ctypes.byref(secs))
        print(f"{label:16s} {secs.value / 5000 * 1e6:.3f} us/step")
