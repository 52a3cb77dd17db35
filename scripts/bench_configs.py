#!/usr/bin/env python
"""All BASELINE.json configurations on one B200, through the public API.

    python scripts/bench_configs.py [--only stream,heat,mandel,dot,overhead,partition]
                                    [--out profiles/rNN_configs.json]

Device times are CUDA events on the launching stream (libofl.so events);
every result is checked against the CPU oracle (oracle/) or the reference's
golden vectors (tests/golden/golden.json) before it is reported.
"""

from __future__ import annotations

import argparse
import ctypes
import hashlib
import json
import math
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

import oracle  # noqa: E402  (checker only)
from paper_1810_11482_b200 import Runtime, _native, make_ready, pinned_empty, when_all  # noqa: E402
from paper_1810_11482_b200.bench.harness import (  # noqa: E402
    PartitionConfig,
    prepare_partitions,
    enqueue_partition_round,
)
from paper_1810_11482_b200.bindings import kernel_source  # noqa: E402

LIB = _native.load()


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except Exception:  # noqa: BLE001
        return {"hbm_gbs": 6650.0}


class Timer:
    """CUDA events on one stream."""

    def __init__(self, stream, ordinal=0):
        self.stream = stream
        self.a, self.b = ctypes.c_void_p(), ctypes.c_void_p()
        LIB.ofl_event_create(ordinal, ctypes.byref(self.a))
        LIB.ofl_event_create(ordinal, ctypes.byref(self.b))

    def start(self):
        LIB.ofl_event_record(self.a, self.stream.ptr)

    def stop(self) -> float:
        LIB.ofl_event_record(self.b, self.stream.ptr)
        ms = ctypes.c_float()
        _native.check(LIB.ofl_event_elapsed_ms(self.a, self.b, ctypes.byref(ms)), "elapsed")
        return ms.value


def sha(b) -> str:
    return hashlib.sha256(bytes(b)).hexdigest()


def stream_cfg(rt, dev, out):
    st = rt.device_objects()[0].stream(0)
    n = 1 << 25
    rng = np.random.default_rng(1)
    b, c = rng.random(n), rng.random(n)
    A, B, C = (dev.create_buffer(n * 8).get() for _ in range(3))
    B.enqueue_write(0, b)
    C.enqueue_write(0, c)
    prog = dev.create_program_with_source(kernel_source("stream")).get()
    res = {}
    for op, nbytes in (("copy", 16), ("scale", 16), ("add", 24), ("triad", 24)):
        prog.build(op).get()
        args = {"copy": [A, B, n], "scale": [A, B, 3.0, n], "add": [A, B, C, n],
                "triad": [A, B, C, 3.0, n]}[op]
        grid = ((n + 255) // 256, 1, 1)
        for _ in range(10):
            prog.run(args, op, grid, (256, 1, 1))
        t = Timer(st)
        K = 500
        t.start()
        for _ in range(K):
            prog.run(args, op, grid, (256, 1, 1))
        ms = t.stop() / K
        got = np.frombuffer(A.enqueue_read(0, n * 8).get(), np.float64)
        ok = got.tobytes() == oracle.stream(op, b, c, 3.0, threads=0).tobytes()
        gbs = nbytes * n / (ms * 1e-3) / 1e9
        res[op] = {"n": n, "us": round(ms * 1e3, 2), "gbs": round(gbs, 1),
                   "frac_measured_hbm": round(gbs / peaks()["hbm_gbs"], 4),
                   "frac_8tbs_spec": round(gbs / 8000.0, 4), "bitexact": ok}
    # size sweep: N = 2^22 .. 2^30, triad, back-to-back launches;
    # 3 x 8 x N bytes <= L2 (126 MB) only at 2^22 — those launches run from L2
    sweep = {}
    l2 = rt.device_objects()[0].physical.l2_bytes
    prog.build("triad").get()
    for lg in range(22, 31):
        m = 1 << lg
        As, Bs, Cs = (dev.create_buffer(m * 8).get() for _ in range(3))
        Bs.enqueue_write(0, np.full(m, 0.5))
        Cs.enqueue_write(0, np.full(m, 0.25))
        args = [As, Bs, Cs, 3.0, m]
        grid = ((m + 255) // 256, 1, 1)
        for _ in range(5):
            prog.run(args, "triad", grid, (256, 1, 1))
        K = max(10, min(1000, (1 << 32) // (24 * m) * 10))
        t = Timer(st)
        t.start()
        for _ in range(K):
            prog.run(args, "triad", grid, (256, 1, 1))
        ms = t.stop() / K
        gbs = 24.0 * m / (ms * 1e-3) / 1e9
        ok = bool(np.all(np.frombuffer(As.enqueue_read(0, 8 * min(m, 1 << 16)).get(),
                                       np.float64) == 0.5 + 3.0 * 0.25))
        sweep[f"2^{lg}"] = {"us": round(ms * 1e3, 2), "gbs": round(gbs, 1),
                            "frac_measured_hbm": round(gbs / peaks()["hbm_gbs"], 4),
                            "working_set_mb": round(24 * m / 1e6, 1), "check": ok}
        del As, Bs, Cs
    res["triad_size_sweep"] = sweep
    res["l2_bytes"] = l2
    out["config1_stream"] = res


def heat_cfg(rt, dev, out, steps=1000, n=1 << 28):
    st = rt.device_objects()[0].stream(0)
    res = {}
    # parity at N=2^20, T=1000 against the oracle (bit-exact), per schedule
    xs = np.random.default_rng(3).random(1 << 20)
    expect = oracle.heat(xs, 1000, threads=0).tobytes()
    prog = dev.create_builtin_program().get()
    prog.build("heat").get()
    X = dev.create_buffer(n * 8).get()
    Y = dev.create_buffer(n * 8).get()
    x = np.random.default_rng(20180214).random(n)
    finals = {}
    for tb in (1, 8, 16, 32, 64, 72):  # 72 = the default cap
        os.environ["OFL_HEAT_TB"] = str(tb)
        Xs = dev.create_buffer(xs.nbytes).get()
        Ys = dev.create_buffer(xs.nbytes).get()
        Xs.enqueue_write(0, xs)
        prog.run([Xs, Ys, xs.size, 1000], "heat", (xs.size // 256, 1, 1), (256, 1, 1))
        small_ok = Xs.enqueue_read(0, xs.nbytes).get() == expect
        X.enqueue_write(0, x)
        dev.synchronize().get()
        t = Timer(st)
        t.start()
        prog.run([X, Y, n, steps], "heat", (n // 256, 1, 1), (256, 1, 1))
        ms = t.stop()
        final = X if steps % 2 == 0 else Y
        digest = sha(final.enqueue_read(0, 1 << 20).get())  # leading 1 MiB fingerprint
        finals[tb] = digest
        alg = 16.0 * n * steps
        res[f"tb{tb}"] = {"ms_total": round(ms, 2), "us_per_step": round(ms * 1e3 / steps, 2),
                          "effective_gbs": round(alg / (ms * 1e-3) / 1e9, 1),
                          "frac_measured_hbm_effective": round(alg / (ms * 1e-3) / 1e9 / peaks()["hbm_gbs"], 4),
                          "parity_2^20_T1000_bitexact": small_ok}
    res["schedules_agree_bitexact"] = len(set(finals.values())) == 1
    # end to end through the API: x from pinned host memory, 1000 steps, the
    # final field back into pinned host memory (wall clock, best of 3)
    xin = pinned_empty(n * 8, np.float64)
    xin[:] = x
    xout = pinned_empty(n * 8, np.float64)
    final = X if steps % 2 == 0 else Y
    e2e = []
    for _ in range(3):
        dev.synchronize().get()
        t0 = time.perf_counter()
        X.enqueue_write(0, xin)
        prog.run([X, Y, n, steps], "heat", (n // 256, 1, 1), (256, 1, 1))
        final.enqueue_read_into(0, xout).get()
        e2e.append((time.perf_counter() - t0) * 1e3)
    res["e2e_ms_pinned_host"] = round(min(e2e), 2)
    res["e2e_fingerprint_matches"] = sha(xout[: 1 << 17]) == finals[72]
    del xin, xout
    res["n"], res["steps"] = n, steps
    res["note"] = ("effective GB/s counts the algorithmic 16 B/cell/step; with temporal "
                   "blocking (tb>1) the HBM traffic is ~16 B/cell per tb steps, so this "
                   "can exceed the HBM roofline")
    os.environ.pop("OFL_HEAT_TB", None)
    out["config2_heat"] = res


def mandel_cfg(rt, dev, out, golden):
    st = rt.device_objects()[0].stream(0)
    w, h, it = 7680, 4320, 2000
    O = dev.create_buffer(w * h * 4).get()
    prog = dev.create_program_with_source(kernel_source("mandelbrot")).get()
    prog.build("mandelbrot").get()
    args = [O, w, h, -2.0, 1.0, -1.5, 1.5, 4.0, it]
    grid = ((w * h + 255) // 256, 1, 1)
    for _ in range(3):
        prog.run(args, "mandelbrot", grid, (256, 1, 1))
    t = Timer(st)
    K = 20
    t.start()
    for _ in range(K):
        prog.run(args, "mandelbrot", grid, (256, 1, 1))
    ms = t.stop() / K
    host = pinned_empty(w * h * 4, np.uint32)
    O.enqueue_read_into(0, host).get()
    ok = sha(host) == golden["mandelbrot"][7]["sha256"]
    total_iters = int(host.astype(np.uint64).sum())
    # algorithmic FP64 ops (the reference's evaluation): per counted iteration
    # 4 mul + 4 add/sub, + 3 for the final escape test.  The fused kernel
    # executes 7 per iteration (zi = fma(2, zr*zi, cim)) + 1 for the final
    # test — for the iterations it runs: with exact cycle detection (default)
    # bounded pixels stop once their orbit provably repeats, so the
    # reference-op rate below is an equivalent rate, not a hardware rate; the
    # FP64 roofline is reported on the plain kernel (OFL_MANDEL_PERIOD=0,
    # measured in a subprocess because the switch is read once per process).
    escaped = int((host < it).sum())
    dp_ops = 8 * total_iters + 3 * escaped
    dp_ops_exec = 7 * total_iters + escaped
    plain_ms = None
    if os.environ.get("OFL_MANDEL_PERIOD", "1") != "0":
        import subprocess

        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--only", "mandel"],
                           env=dict(os.environ, OFL_MANDEL_PERIOD="0"), capture_output=True,
                           text=True)
        try:
            plain_ms = json.loads(r.stdout)["config3_mandelbrot"]["kernel_ms"]
        except Exception:  # noqa: BLE001
            plain_ms = None
    fp64 = fp64_peak(rt)
    e2e_host = pinned_empty(w * h * 4, np.uint32)
    t0 = time.perf_counter()
    for _ in range(5):
        prog.run(args, "mandelbrot", grid, (256, 1, 1))
        O.enqueue_read_into(0, e2e_host).get()
    e2e_ms = (time.perf_counter() - t0) / 5 * 1e3
    # overlapped: 8 chunks alternating over two streams, each chunk read by
    # one DMA straight into the pinned image while the next chunk computes
    from paper_1810_11482_b200 import when_all
    from paper_1810_11482_b200.bench.harness import MandelbrotTiles

    tiles = MandelbrotTiles([dev], w, h, it, chunks=8)
    when_all(tiles.enqueue()).get()
    t0 = time.perf_counter()
    for _ in range(5):
        when_all(tiles.enqueue()).get()
    e2e_overlap_ms = (time.perf_counter() - t0) / 5 * 1e3
    image = tiles.image
    ok_overlap = sha(image) == golden["mandelbrot"][7]["sha256"]
    out["config3_mandelbrot"] = {
        "width": w, "height": h, "max_iter": it, "kernel_ms": round(ms, 3),
        "e2e_ms_with_d2h": round(e2e_ms, 3), "sha256_matches_reference": ok,
        "e2e_ms_overlapped_8_chunks": round(e2e_overlap_ms, 3),
        "overlapped_sha256_matches_reference": ok_overlap,
        "total_iterations": total_iters, "dp_ops": dp_ops,
        "achieved_dp_tops": round(dp_ops / (ms * 1e-3) / 1e12, 3),
        "fp64_peak_measured_tops": fp64,
        "cycle_detection": os.environ.get("OFL_MANDEL_PERIOD", "1") != "0",
        "reference_op_rate_over_fp64_peak": round(dp_ops / (ms * 1e-3) / 1e12 / fp64, 4)
        if fp64 else None,
        "plain_kernel_ms": plain_ms if plain_ms is not None else round(ms, 3),
        "plain_frac_fp64": round(dp_ops / ((plain_ms or ms) * 1e-3) / 1e12 / fp64, 4)
        if fp64 else None,
        "plain_frac_fp64_executed_ops": round(dp_ops_exec / ((plain_ms or ms) * 1e-3) / 1e12 / fp64, 4)
        if fp64 else None,
    }


def fp64_peak(rt) -> float:
    fn = getattr(LIB, "ofl_bench_fp64_peak", None)
    if fn is None:
        return None
    fn.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)]
    fn.restype = ctypes.c_int
    st = rt.device_objects()[0].stream(0)
    v = ctypes.c_double()
    if fn(st.ptr, ctypes.byref(v)):
        return None
    return round(v.value / 1e12, 3)


def dot_cfg(rt, dev, out, n=1 << 31):
    st = rt.device_objects()[0].stream(0)
    A = dev.create_buffer(n * 4).get()
    B = dev.create_buffer(n * 4).get()
    R = dev.create_buffer(8).get()
    rng = np.random.default_rng(20180214)
    chunk = 1 << 27
    a_all = np.empty(n, np.float32)
    b_all = np.empty(n, np.float32)
    for lo in range(0, n, chunk):
        a_all[lo : lo + chunk] = rng.random(min(chunk, n - lo), dtype=np.float32)
        b_all[lo : lo + chunk] = rng.random(min(chunk, n - lo), dtype=np.float32)
    for lo in range(0, n, chunk):
        A.enqueue_write(lo * 4, a_all[lo : lo + chunk])
        B.enqueue_write(lo * 4, b_all[lo : lo + chunk])
    prog = dev.create_builtin_program().get()
    prog.build("dot_f32").get()
    grid = (n // 256, 1, 1)
    for _ in range(3):
        prog.run([A, B, R, n], "dot_f32", grid, (256, 1, 1))
    t = Timer(st)
    K = 20
    t.start()
    for _ in range(K):
        prog.run([A, B, R, n], "dot_f32", grid, (256, 1, 1))
    ms = t.stop() / K
    got = float(np.frombuffer(R.enqueue_read(0, 8).get(), np.float64)[0])
    exp = oracle.dot_f32(a_all, b_all, threads=0)
    # end to end through the API from the pageable numpy inputs (16 GiB over
    # the host link via libofl's pipelined staging), wall clock
    dev.synchronize().get()
    t0 = time.perf_counter()
    A.enqueue_write(0, a_all)
    B.enqueue_write(0, b_all)
    prog.run([A, B, R, n], "dot_f32", grid, (256, 1, 1))
    got_e2e = float(np.frombuffer(R.enqueue_read(0, 8).get(), np.float64)[0])
    e2e_ms = (time.perf_counter() - t0) * 1e3
    gbs = 8.0 * n / (ms * 1e-3) / 1e9
    out["config4_dot"] = {"n": n, "kernel_ms": round(ms, 3), "gbs": round(gbs, 1),
                          "frac_measured_hbm": round(gbs / peaks()["hbm_gbs"], 4),
                          "result": got, "oracle": exp, "rel_err": abs(got - exp) / abs(exp),
                          "within_1e-5": abs(got - exp) <= 1e-5 * abs(exp),
                          "e2e_ms_pageable_host": round(e2e_ms, 1),
                          "e2e_result_same": got_e2e == got}


def overhead_cfg(rt, dev, out):
    from bench import OverheadBench  # noqa: E402

    out["config5_overhead"] = {
        "8B_payload": OverheadBench(dev, rt).sweep(),
        "4KiB_payload": OverheadBench(dev, rt, payload_bytes=4096).sweep((1, 100, 10000)),
    }


def stencil2d_cfg(rt, dev, out, w=16384, h=16384):
    """One stencil2d.k Jacobi step over a 16384^2 f64 grid (2 GiB per
    buffer): 16 B/cell algorithmic, HBM-bound; K launches ping-ponging."""
    st = rt.device_objects()[0].stream(0)
    n = w * h
    x = np.random.default_rng(20180214).random(n)
    X, Y = dev.create_buffer(n * 8).get(), dev.create_buffer(n * 8).get()
    X.enqueue_write(0, x)
    Y.enqueue_write(0, x)
    prog = dev.create_program_with_source(kernel_source("stencil2d")).get()
    prog.build("stencil2d").get()
    grid = (math.ceil(n / 256), 1, 1)
    prog.run([X, Y, w, h], "stencil2d", grid, (256, 1, 1))
    got = Y.enqueue_read(0, n * 8).get()
    ok = got == oracle.stencil2d(x, w, h, out=x.copy(), threads=0).tobytes()
    for _ in range(3):
        prog.run([X, Y, w, h], "stencil2d", grid, (256, 1, 1))
    t = Timer(st)
    K = 20
    t.start()
    for k in range(K):
        a, b = (X, Y) if k % 2 == 0 else (Y, X)
        prog.run([a, b, w, h], "stencil2d", grid, (256, 1, 1))
    ms = t.stop() / K
    gbs = 16.0 * n / (ms * 1e-3) / 1e9
    out["stencil2d"] = {"w": w, "h": h, "kernel_ms": round(ms, 3), "gbs": round(gbs, 1),
                        "frac_measured_hbm": round(gbs / peaks()["hbm_gbs"], 4),
                        "bitexact_one_step": ok}


def cpu_cfg(rt, dev, out):
    """The CPU restatement of the reference path (oracle/, C, no FMA) timed
    on this box's host cores for every config, 1 thread (the reference runs
    each launch on one core, codegen.py:118-123) and all threads, on bounded
    samples scaled to the full config (stated per entry)."""
    import os as _os

    T = oracle.max_threads()
    res = {"threads_all": T, "cpu_count": _os.cpu_count()}

    def timed(fn):
        t0 = time.perf_counter()
        fn()
        return time.perf_counter() - t0

    n = 1 << 25
    b, c = np.random.default_rng(1).random(n), np.random.default_rng(2).random(n)
    a = np.empty(n)
    oracle.stream("triad", b, c, 3.0, out=a, threads=T)
    for th in (1, T):
        sec = min(timed(lambda: oracle.stream("triad", b, c, 3.0, out=a, threads=th))
                  for _ in range(3))
        res[f"triad_2^25_t{th}"] = {"ms": round(sec * 1e3, 2), "gbs": round(24 * n / sec / 1e9, 2)}
    x = np.random.default_rng(3).random(1 << 28)
    for th in (1, T):
        sec = timed(lambda: oracle.heat(x, 2, threads=th))
        res[f"heat_2^28_t{th}"] = {"sample": "2 steps", "ms_per_step": round(sec / 2 * 1e3, 1),
                                   "extrapolated_1000_steps_s": round(sec / 2 * 1000, 1)}
    del x
    w, h, it = 7680, 4320, 2000
    rows = 96  # 1/45 of the image, cyclic rows so the sample is representative
    for th in (1, T):
        sec = timed(lambda: oracle.mandelbrot(w, h, max_iter=it, row_first=0, row_step=h // rows,
                                              threads=th))
        res[f"mandelbrot_t{th}"] = {"sample": f"{rows} of {h} rows (cyclic)",
                                    "extrapolated_s": round(sec * h / rows, 1)}
    m = 1 << 28
    fa = np.random.default_rng(4).random(m, dtype=np.float32)
    fb = np.random.default_rng(5).random(m, dtype=np.float32)
    for th in (1, T):
        sec = timed(lambda: oracle.dot_f32(fa, fb, threads=th))
        res[f"dot_f32_t{th}"] = {"sample": "2^28 elements", "extrapolated_2^31_ms":
                                 round(sec * 8 * 1e3, 1), "gbs": round(8 * m / sec / 1e9, 2)}
    out["cpu_reference_port"] = res


def sum_cfg(rt, dev, out):
    """u32 wrap-around sum (sum.k) at 2^28 elements: 4 B/elem, HBM-bound."""
    st = rt.device_objects()[0].stream(0)
    n = 1 << 28
    v = np.random.default_rng(5).integers(0, 2**32, n, dtype=np.uint32)
    I = dev.create_buffer(n * 4).get()
    R = dev.create_buffer(4).get()
    I.enqueue_write(0, v)
    prog = dev.create_program_with_source(kernel_source("sum")).get()
    prog.build("sum").get()
    for _ in range(3):
        prog.run([I, R, n], "sum", (1, 1, 1), (32, 1, 1))
    t = Timer(st)
    K = 50
    t.start()
    for _ in range(K):
        prog.run([I, R, n], "sum", (1, 1, 1), (32, 1, 1))
    ms = t.stop() / K
    got = int(np.frombuffer(R.enqueue_read(0, 4).get(), np.uint32)[0])
    gbs = 4.0 * n / (ms * 1e-3) / 1e9
    out["sum_u32"] = {"n": n, "kernel_ms": round(ms, 4), "gbs": round(gbs, 1),
                      "frac_measured_hbm": round(gbs / peaks()["hbm_gbs"], 4),
                      "bitexact": got == oracle.sum_u32(v, threads=0)}


def transfer_cfg(rt, dev, out):
    """Host<->device copy rates through the API (enqueue_write/read)."""
    n = 1 << 28  # 256 MiB
    buf = dev.create_buffer(n).get()
    buf2 = dev.create_buffer(n).get()
    pin = pinned_empty(n)
    pin2 = pinned_empty(n)
    pin[:] = 7
    page = np.full(n, 5, np.uint8)
    res = {}

    def rate(fn, reps=5):
        fn()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        return round(n * reps / (time.perf_counter() - t0) / 1e9, 2)

    res["h2d_pinned_gbs"] = rate(lambda: buf.enqueue_write(0, pin).get())
    res["d2h_pinned_gbs"] = rate(lambda: buf.enqueue_read_into(0, pin2).get())
    s1 = dev.create_stream()
    res["bidir_pinned_gbs_total"] = round(2 * rate(
        lambda: when_all([buf.enqueue_write(0, pin), buf2.enqueue_read_into(0, pin2, s1)]).get()), 2)
    res["h2d_pageable_numpy_gbs"] = rate(lambda: buf.enqueue_write(0, page).get())
    res["d2h_to_bytes_gbs"] = rate(lambda: buf.enqueue_read(0, n).get(), reps=3)
    ok = buf.enqueue_read(0, 4096).get() == bytes([5]) * 4096
    res["pageable_roundtrip_ok"] = ok
    out["transfers_256MiB"] = res


def partition_cfg(rt, dev, out):
    res = {}
    for m in (1, 2, 3, 6):
        cfg = PartitionConfig(m=m, partitions=4)
        n, parts = prepare_partitions(cfg, [dev])
        outs = [pinned_empty(p.count * 8, np.float64) for p in parts]
        for _ in range(2):
            for t in enqueue_partition_round(parts, outs):
                t.get()
        samples = []
        for _ in range(11):
            t0 = time.perf_counter()
            for t in enqueue_partition_round(parts, outs):
                t.get()
            samples.append(time.perf_counter() - t0)
        mean_ms = sum(samples[1:]) / 10 * 1e3
        dev_max = float(max(np.abs(o - 1.0).max() for o in outs))
        res[f"m{m}"] = {"n": n, "mean_ms": round(mean_ms, 3), "max_abs_dev": dev_max,
                        "h2d_d2h_gbs": round(16.0 * n / (mean_ms * 1e-3) / 1e9, 2)}
    out["alg1_partition"] = res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only",
                    default="stream,heat,mandel,dot,sum,stencil2d,overhead,partition,transfer,cpu")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    with open(os.path.join(REPO, "tests", "golden", "golden.json")) as fh:
        golden = json.load(fh)
    out = {"device": None}
    with Runtime(devices=[0]) as rt:
        dev = rt.get_all_devices().get()[0]
        out["device"] = rt.device_objects()[0].physical.product
        for name in args.only.split(","):
            t0 = time.time()
            {"stream": lambda: stream_cfg(rt, dev, out),
             "heat": lambda: heat_cfg(rt, dev, out),
             "mandel": lambda: mandel_cfg(rt, dev, out, golden),
             "dot": lambda: dot_cfg(rt, dev, out),
             "overhead": lambda: overhead_cfg(rt, dev, out),
             "partition": lambda: partition_cfg(rt, dev, out),
             "transfer": lambda: transfer_cfg(rt, dev, out),
             "sum": lambda: sum_cfg(rt, dev, out),
             "stencil2d": lambda: stencil2d_cfg(rt, dev, out),
             "cpu": lambda: cpu_cfg(rt, dev, out)}[name]()
            print(f"[{name}] {time.time() - t0:.1f}s", file=sys.stderr, flush=True)
    text = json.dumps(out, indent=1)
    print(text)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(text)


if __name__ == "__main__":
    main()
