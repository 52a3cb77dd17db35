#!/usr/bin/env python
"""Headline benchmark: STREAM triad GB/s on B200 through the futurized
device/buffer/program API, plus the per-future launch overhead.

Metric (BASELINE.json): "STREAM triad GB/s (frac of HBM peak) @1/2/4/8 B200;
per-future launch overhead µs".  Workload: BASELINE config 1 — triad
a = b + 3.0*c over N = 2^25 fp64 elements per GPU (24 B/elem algorithmic),
issued as `program.run(...)` on a program built from the kernel language
(paper_1810_11482_b200/kernels/stream.k), each run returning a future.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 is launched by torchrun, one process per GPU; each rank runs its own
replica (the triad shards with no exchange: weak scaling, no collective),
ranks meet at a barrier around the timed region and the slowest rank's
CUDA-event time is the job time.  `--impl reference` times the CPU
restatement of the reference path (oracle/, all host threads) on the same
config; only rank 0 runs it.

Timed region (value): K launches back to back on the device, inputs resident
in HBM, 805 MB per step per GPU (> 126 MB L2, so every step streams HBM).
e2e: the same metric through the public API with host buffers: per step two
enqueue_write from pinned memory, the run, and an enqueue_read_into pinned
memory, `.get()` on the read — wall clock, copies included.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "STREAM triad GB/s (frac of HBM peak) @1/2/4/8 B200; per-future launch overhead µs"
FALLBACK_HBM_GBS = 6650.0
SPEC_HBM_GBS = 8000.0  # B200 HBM3e datasheet; the measured copy peak above is a torch copy_


def env_int(name: str, default: int) -> int:
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def hbm_peak() -> tuple[float, str]:
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic() -> dict:
    path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except Exception:  # noqa: BLE001
        return {}


class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) during the timed region."""

    def __init__(self, index: int, period: float = 0.002):
        self.samples: list = []
        self.reasons: set = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self._nv = None
        self.period = period

    _REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    }

    def _sample(self):
        nv = self._nv
        try:
            self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
            mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            for bit, name in self._REASONS.items():
                if mask & bit and name != "gpu_idle":
                    self.reasons.add(name)
        except Exception:  # noqa: BLE001
            pass

    def _run(self):
        while not self._stop.wait(self.period):
            self._sample()

    def start(self):
        if self._nv is not None:
            self._sample()  # at least one sample inside even a short region
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()

    def stop(self) -> dict:
        self._stop.set()
        if self._thread is not None:
            self._thread.join()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        s = sorted(self.samples)
        return {
            "sm_mhz": s[len(s) // 2],
            "sm_max_mhz": self.max_mhz,
            "reasons": sorted(self.reasons),
            "samples": len(s),
        }


class Dist:
    """torch.distributed plumbing (barrier, max over ranks); no-op at N=1.
    The triad shards with no data-path collective, so the plumbing only
    moves two scalars per run; it uses gloo (host) so it never competes with
    the measured device work and also works with more ranks than GPUs."""

    def __init__(self, world: int, local_rank: int):
        self.world = world
        self.dist = None
        if world > 1:
            import torch
            import torch.distributed as dist

            dist.init_process_group("gloo")
            self.dist = dist
            self.torch = torch

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if self.dist is None:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.dist is None:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64)
        self.dist.all_reduce(t)
        return float(t.item())

    def gather(self, obj) -> list:
        if self.dist is None:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def close(self):
        if self.dist is not None:
            self.dist.destroy_process_group()


def cpu_triad_rate(n: int, seconds: float, threads: int) -> dict:
    """The oracle (C restatement of the reference path) timed on host cores."""
    import numpy as np

    import oracle

    rng = np.random.default_rng(20180214)
    b = rng.random(n)
    c = rng.random(n)
    a = np.empty(n)
    oracle.stream("triad", b, c, 3.0, out=a, threads=threads)  # warm-up / page-in
    reps = 0
    t0 = time.perf_counter()
    while True:
        oracle.stream("triad", b, c, 3.0, out=a, threads=threads)
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return {"gbs": 24.0 * n * reps / el / 1e9, "reps": reps, "seconds": el}


def run_reference(args) -> None:
    """--impl reference: the CPU restatement of the reference path, all
    host threads, same config/metric; rank 0 only."""
    if env_int("RANK", 0) != 0:
        return
    import numpy as np

    import oracle

    threads = oracle.max_threads()
    n = args.n
    rng = np.random.default_rng(20180214)
    b, c = rng.random(n), rng.random(n)
    a = np.empty(n)
    # W untimed + K timed steps; one step = one triad sweep over a bounded
    # sample of the N-element workload (the first m elements), m chosen from
    # the warm-up rate so the K timed steps take about --ref-seconds.
    oracle.stream("triad", b, c, 3.0, out=a, threads=threads)  # page-in, full size
    t0 = time.perf_counter()
    oracle.stream("triad", b, c, 3.0, out=a, threads=threads)
    full_s = max(time.perf_counter() - t0, 1e-6)
    budget = max(1.0, float(args.ref_seconds))
    m = n if full_s * args.steps <= budget else max(1 << 16, int(n * budget / (full_s * args.steps)))
    m = min(n, m)
    for _ in range(args.warmup):
        oracle.stream("triad", b[:m], c[:m], 3.0, out=a[:m], threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.stream("triad", b[:m], c[:m], 3.0, out=a[:m], threads=threads)
    el = time.perf_counter() - t0
    gbs = 24.0 * m * args.steps / el / 1e9
    r = {"gbs": gbs}
    world = max(1, env_int("WORLD_SIZE", 1))
    sample = (f"{args.steps} timed triad sweeps (after {args.warmup} warm-up) over the first "
              f"{m} of N={n} fp64 elements ({el:.1f} s), C restatement in oracle/ on "
              f"{threads} host threads")
    if world > 1:
        sample += (f"; the whole job is {world} x N elements, all in the one host memory, so "
                   "this bandwidth is the CPU path's rate for it")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(r["gbs"], 3),
        "unit": "GB/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(el / args.steps * 1e3 * n / m, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(n, world),
        "cpu_baseline": {
            "value": round(r["gbs"], 3), "unit": "GB/s", "cores": threads, "kind": "port",
            "sample": sample,
        },
        "e2e": {"value": round(r["gbs"], 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(n: int, world: int) -> dict:
    return {
        "workload": "STREAM triad a=b+3.0*c, N=2^25 fp64 per GPU, futurized program.run "
        "(BASELINE config 1)",
        "n_per_gpu": n,
        "bytes_per_step_per_gpu": 24 * n,
        "l2_policy": "inputs larger than L2 (3 x 256 MiB per GPU vs 126 MB L2)",
        "parallelism": f"{world} independent replicas (weak scaling, no collective)",
    }


class OverheadBench:
    """Per-future overhead vs raw CUDA streams (BASELINE config 5).

    One step = an 8-byte H2D write + the STREAM triad over N=1024 (the
    product kernel and launch), chained K deep.  Futurized: every step is
    ``w = enqueue_write; r = run; prev = when_all([prev, w, r])`` and the
    chain ends with ``prev.get()``.  Raw (csrc/ofl_bench.cu, a C loop on the
    CUDA runtime): the same cudaMemcpyAsync + launch per step, mode 0 =
    stream order only, mode 1 = an event recorded after each step and waited
    on by the next (explicit dependency chaining); cudaStreamSynchronize at
    the end.  BASELINE.md §3: overhead per future = (t_futurized - t_raw)/K,
    one future per step (the step's when_all), no other division.  Each K
    is timed as the min over 3 batches of the mean time per chain, a batch
    holding enough chains to last >= ~20 ms.  Sync-each-step: ``run().get()``
    every step vs raw mode 2 (cudaStreamSynchronize per step)."""

    def __init__(self, dev, rt, payload_bytes: int = 8):
        import numpy as np

        from paper_1810_11482_b200 import _native, pinned_empty
        from paper_1810_11482_b200.bindings import kernel_source

        self.lib = _native.load()
        self._native = _native
        self.dev = dev
        self.n = n = 1024
        self.A, self.B, self.C, self.D = (dev.create_buffer(n * 8).get() for _ in range(4))
        self.prog = dev.create_program_with_source(kernel_source("stream")).get()
        self.prog.build("triad").get()
        self.payload_bytes = payload_bytes
        self.payload = pinned_empty(payload_bytes)
        self.payload[:] = 1
        self.args = [self.A, self.B, self.C, 3.0, n]
        self.grid, self.block = ((n + 255) // 256, 1, 1), (256, 1, 1)
        self.stream = rt.device_objects()[0].stream(0)
        self.dptr = rt.local._buffer(self.D.gid).ptr
        self.ptrs = [rt.local._buffer(x.gid).ptr for x in (self.A, self.B, self.C)]
        del np

    def raw(self, steps: int, mode: int) -> float:
        secs = ctypes.c_double()
        a, b, c = self.ptrs
        self._native.check(
            self.lib.ofl_bench_raw_chain(self.stream.ptr, self.dptr, self.payload.ctypes.data,
                                         self.payload_bytes, a, b, c, self.n, steps, mode,
                                         ctypes.byref(secs)),
            "raw chain")
        return secs.value

    def futurized(self, steps: int) -> float:
        from paper_1810_11482_b200 import make_ready, when_all

        D, prog, args, grid, block, payload = (self.D, self.prog, self.args, self.grid,
                                               self.block, self.payload)
        t0 = time.perf_counter()
        prev = make_ready(None)
        for _ in range(steps):
            w = D.enqueue_write(0, payload)
            r = prog.run(args, "triad", grid, block)
            prev = when_all([prev, w, r])
        prev.get()
        return time.perf_counter() - t0

    def synced(self, steps: int) -> float:
        D, prog, args, grid, block, payload = (self.D, self.prog, self.args, self.grid,
                                               self.block, self.payload)
        t0 = time.perf_counter()
        for _ in range(steps):
            D.enqueue_write(0, payload)
            prog.run(args, "triad", grid, block).get()
        return time.perf_counter() - t0

    @staticmethod
    def per_chain(fn, k: int) -> float:
        """min over 3 batches of the mean seconds per K-step chain."""
        reps = max(1, 2000 // k)
        best = float("inf")
        for _ in range(3):
            t = sum(fn(k) for _ in range(reps)) / reps
            best = min(best, t)
        return best

    def point(self, k: int) -> dict:
        self.dev.synchronize().get()
        raw0 = self.per_chain(lambda s: self.raw(s, 0), k)
        raw1 = self.per_chain(lambda s: self.raw(s, 1), k)
        fut = self.per_chain(self.futurized, k)
        us = 1e6 / k
        return {
            "K": k,
            "raw_stream_order_us_per_step": round(raw0 * us, 3),
            "raw_event_chained_us_per_step": round(raw1 * us, 3),
            "futurized_us_per_step": round(fut * us, 3),
            "overhead_us_per_future": round((fut - raw0) * us, 3),
            "overhead_us_per_future_vs_event_chained": round((fut - raw1) * us, 3),
        }

    def sync_point(self, k: int) -> dict:
        self.dev.synchronize().get()
        raw2 = self.per_chain(lambda s: self.raw(s, 2), k)
        fut = self.per_chain(self.synced, k)
        us = 1e6 / k
        return {"K": k, "raw_sync_each_step_us": round(raw2 * us, 3),
                "futurized_get_each_step_us": round(fut * us, 3),
                "overhead_us_per_future": round((fut - raw2) * us, 3)}

    def sweep(self, ks=(1, 10, 100, 1000, 10000, 100000), sync_k: int = 1000) -> dict:
        # warm both paths (first launches, pinned-range lookups, JIT-free)
        self.raw(200, 0)
        self.raw(200, 1)
        self.futurized(200)
        self.synced(50)
        points = [self.point(k) for k in ks]
        head = next((p for p in points if p["K"] == 10000), points[-1])
        return {
            "formula": "(t_futurized - t_raw) / K per K-step chain, one future per step "
                       "(BASELINE.md §3); raw = same cudaMemcpyAsync + launch from C",
            "step": f"H2D {self.payload_bytes} B + triad N={self.n}, prev = when_all([prev, w, r])",
            "overhead_us_per_future": head["overhead_us_per_future"],
            "overhead_us_per_future_vs_event_chained":
                head["overhead_us_per_future_vs_event_chained"],
            "at_K": head["K"],
            "max_over_K_us": max(p["overhead_us_per_future"] for p in points),
            "sweep": points,
            "sync_each_step": self.sync_point(sync_k),
            "target_us": 5.0,
        }


class EventTimer:
    """CUDA events on one stream (libofl events): device time of what is
    enqueued between start() and stop()."""

    def __init__(self, lib, stream, ordinal: int):
        from paper_1810_11482_b200 import _native

        self.lib, self.stream, self._native = lib, stream, _native
        self.a, self.b = ctypes.c_void_p(), ctypes.c_void_p()
        _native.check(lib.ofl_event_create(ordinal, ctypes.byref(self.a)), "event")
        _native.check(lib.ofl_event_create(ordinal, ctypes.byref(self.b)), "event")

    def start(self):
        self.lib.ofl_event_record(self.a, self.stream.ptr)

    def stop(self) -> float:
        self.lib.ofl_event_record(self.b, self.stream.ptr)
        ms = ctypes.c_float()
        self._native.check(self.lib.ofl_event_elapsed_ms(self.a, self.b, ctypes.byref(ms)),
                           "elapsed")
        return ms.value


def _golden(name: str) -> dict:
    try:
        with open(os.path.join(REPO, "tests", "golden", name)) as fh:
            return json.load(fh)
    except Exception:  # noqa: BLE001
        return {}


def _sha(buf) -> str:
    import hashlib

    return hashlib.sha256(memoryview(buf).cast("B")).hexdigest()


def fp64_peak_ops(lib, stream) -> float:
    """Measured FP64 DMUL/DADD issue rate (ops/s), csrc/ofl_bench.cu."""
    v = ctypes.c_double()
    if lib.ofl_bench_fp64_peak(stream.ptr, ctypes.byref(v)):
        return 0.0
    return v.value


def config_heat(rt, dev, lib, fp64: float, n: int = 1 << 28, steps: int = 1000) -> dict:
    """Config 2 on one GPU: 2^28 cells x 1000 steps of stencil.k through the
    `heat` builtin; parity = sha256 of the final field equals the REFERENCE's
    (tests/golden/golden_long.json, offloadrt host backend, ~13 min)."""
    import numpy as np

    from paper_1810_11482_b200 import pinned_empty

    st = rt.device_objects()[0].stream(0)
    x = pinned_empty(n * 8, np.float64)
    x[:] = np.random.default_rng(20180214).random(n)
    xout = pinned_empty(n * 8, np.float64)
    X, Y = dev.create_buffer(n * 8).get(), dev.create_buffer(n * 8).get()
    prog = dev.create_builtin_program().get()
    prog.build("heat").get()
    final = X if steps % 2 == 0 else Y
    grid, block = (n // 256, 1, 1), (256, 1, 1)
    mono = []
    for _ in range(3):  # end to end in sequence: pinned x in, 1000 steps, field back out
        dev.synchronize().get()
        t0 = time.perf_counter()
        X.enqueue_write(0, x)
        prog.run([X, Y, n, steps], "heat", grid, block)
        final.enqueue_read_into(0, xout).get()
        mono.append(time.perf_counter() - t0)
    ref = next((c for c in _golden("golden_long.json").get("heat", [])
                if c["n"] == n and c["steps"] == steps), None)
    digest = _sha(xout)
    # end to end with the transfers overlapped with the steps: independent
    # halo-extended pieces on rotating streams (bench.HeatChunks)
    from paper_1810_11482_b200 import when_all
    from paper_1810_11482_b200.bench import HeatChunks

    chunked = HeatChunks(dev, n, steps)
    e2e = []
    for _ in range(3):
        xout[:1] = 0
        dev.synchronize().get()
        t0 = time.perf_counter()
        when_all(chunked.enqueue(x, xout)).get()
        e2e.append(time.perf_counter() - t0)
    digest_chunked = _sha(xout)
    del chunked
    # the host-link floor of that schedule: the same pieces written and read
    # with zero steps (HeatChunks with steps=0: no halo, no kernel work)
    copies = HeatChunks(dev, n, 0)
    floor = []
    for _ in range(3):
        dev.synchronize().get()
        t0 = time.perf_counter()
        when_all(copies.enqueue(x, xout)).get()
        floor.append(time.perf_counter() - t0)
    del copies
    kernel = []
    for _ in range(3):  # device time of the steps alone (input re-written, untimed)
        X.enqueue_write(0, x)
        t = EventTimer(lib, st, dev_ordinal(rt))
        t.start()
        prog.run([X, Y, n, steps], "heat", grid, block)
        kernel.append(t.stop())
    ms = min(kernel)
    useful = 2.0 * n * steps  # 2 FP64 ops per cell-step (the fused update; reference: 2 mul + 2 add)
    alg_bytes = 16.0 * n * steps
    return {
        "workload": "heat 2^28 fp64 x 1000 steps (BASELINE config 2), builtin `heat`, 1 GPU",
        "kernel_ms": round(ms, 3),
        "effective_gbs": round(alg_bytes / (ms * 1e-3) / 1e9, 1),
        "useful_fp64_ops_per_s": round(useful / (ms * 1e-3), 1),
        "fp64_peak_ops_per_s": round(fp64, 1),
        "frac_fp64": round(useful / (ms * 1e-3) / fp64, 4) if fp64 else None,
        "e2e_ms_pinned_host": round(min(e2e) * 1e3, 2),
        "e2e_link_floor_ms": round(min(floor) * 1e3, 2),
        "e2e_frac_of_link_floor": round(min(floor) / min(e2e), 4),
        "e2e_schedule": "bench.HeatChunks: 64 halo-extended pieces over 12 buffer pairs / streams, "
                        "write / 1000 steps / read of successive pieces overlapped",
        "e2e_ms_sequential": round(min(mono) * 1e3, 2),
        "e2e_h2d_bytes": n * 8, "e2e_d2h_bytes": n * 8,
        "sha256": digest,
        "parity": ("bit-exact vs reference (golden_long.json), kernel and both e2e schedules"
                   if ref and digest == ref["sha256"] == digest_chunked
                   else "MISMATCH vs reference" if ref else "reference sha unavailable"),
        "note": "effective_gbs counts 16 B/cell/step; temporal blocking keeps tb steps "
                "in registers, so it exceeds the HBM roofline and FP64 issue is the bound",
    }


def config_mandelbrot(rt, dev, lib, fp64: float) -> dict:
    """Config 3: 7680x4320, max_iter 2000, the reference's mandelbrot.k;
    parity = sha256 of the counts equals the reference's (golden.json)."""
    import numpy as np

    from paper_1810_11482_b200 import pinned_empty, when_all
    from paper_1810_11482_b200.bench.harness import MandelbrotTiles
    from paper_1810_11482_b200.bindings import kernel_source

    w, h, it = 7680, 4320, 2000
    st = rt.device_objects()[0].stream(0)
    O = dev.create_buffer(w * h * 4).get()
    prog = dev.create_program_with_source(kernel_source("mandelbrot")).get()
    prog.build("mandelbrot").get()
    args = [O, w, h, -2.0, 1.0, -1.5, 1.5, 4.0, it]
    grid = ((w * h + 255) // 256, 1, 1)
    for _ in range(3):
        prog.run(args, "mandelbrot", grid, (256, 1, 1))
    t = EventTimer(lib, st, dev_ordinal(rt))
    K = 10
    t.start()
    for _ in range(K):
        prog.run(args, "mandelbrot", grid, (256, 1, 1))
    ms = t.stop() / K
    host = pinned_empty(w * h * 4, np.uint32)
    O.enqueue_read_into(0, host).get()
    ref = next((c for c in _golden("golden.json").get("mandelbrot", [])
                if c["width"] == w and c["height"] == h and c["max_iter"] == it), None)
    ok = ref is not None and _sha(host) == ref["sha256"]
    total = int(host.astype(np.uint64).sum())
    escaped = int((host < it).sum())
    dp_ops = 8 * total + 3 * escaped  # the reference's evaluation, per counted iteration
    tiles = MandelbrotTiles([dev], w, h, it, chunks=8)
    when_all(tiles.enqueue()).get()
    e2e = []
    for _ in range(5):
        t0 = time.perf_counter()
        when_all(tiles.enqueue()).get()
        e2e.append(time.perf_counter() - t0)
    ok_e2e = ref is not None and _sha(tiles.image) == ref["sha256"]
    floor = []  # the image read alone (one D2H into pinned memory): the link floor
    for _ in range(5):
        t0 = time.perf_counter()
        O.enqueue_read_into(0, host).get()
        floor.append(time.perf_counter() - t0)
    return {
        "workload": "Mandelbrot 7680x4320 max_iter 2000 (BASELINE config 3), 1 GPU",
        "kernel_ms": round(ms, 3),
        "e2e_ms_overlapped_into_pinned_image": round(min(e2e) * 1e3, 3),
        "e2e_d2h_bytes": w * h * 4,
        "e2e_link_floor_ms": round(min(floor) * 1e3, 3),
        "e2e_frac_of_link_floor": round(min(floor) / min(e2e), 4),
        "reference_dp_ops": dp_ops,
        "reference_op_rate_over_fp64_peak": round(dp_ops / (ms * 1e-3) / fp64, 4) if fp64 else None,
        "note": "exact shortcuts (cycle detection; pixels provably inside the main cardioid "
                "or the period-2 bulb) skip iterations of never-escaping pixels, so the "
                "reference-op rate is an equivalent rate and exceeds 1; the FP64 roofline of "
                "the plain kernel is in profiles/r02_configs.json",
        "parity": "bit-exact vs reference sha256 (kernel and overlapped e2e)" if ok and ok_e2e
                  else "MISMATCH vs reference",
    }


def config_dot(rt, dev, lib, n: int = 1 << 31) -> dict:
    """Config 4 on one GPU: fp32 dot over 2^31 elements, fp64 accumulation;
    parity = relative error vs the fp64 oracle (tolerance 1e-5)."""
    import numpy as np

    import oracle

    st = rt.device_objects()[0].stream(0)
    rng = np.random.default_rng(20180214)
    a = rng.random(n, dtype=np.float32)
    b = rng.random(n, dtype=np.float32)
    A, B, R = dev.create_buffer(n * 4).get(), dev.create_buffer(n * 4).get(), dev.create_buffer(8).get()
    prog = dev.create_builtin_program().get()
    prog.build("dot_f32").get()
    grid = (n // 256, 1, 1)
    e2e = []
    for _ in range(2):  # end to end from the pageable numpy arrays
        dev.synchronize().get()
        t0 = time.perf_counter()
        A.enqueue_write(0, a)
        B.enqueue_write(0, b)
        prog.run([A, B, R, n], "dot_f32", grid, (256, 1, 1))
        got = float(np.frombuffer(R.enqueue_read(0, 8).get(), np.float64)[0])
        e2e.append(time.perf_counter() - t0)
    t = EventTimer(lib, st, dev_ordinal(rt))
    K = 10
    batches = []
    for _ in range(3):  # best of 3 batches of K back-to-back launches
        t.start()
        for _ in range(K):
            prog.run([A, B, R, n], "dot_f32", grid, (256, 1, 1))
        batches.append(t.stop() / K)
    ms = min(batches)
    exp = oracle.dot_f32(a, b, threads=0)
    rel = abs(got - exp) / abs(exp)
    gbs = 8.0 * n / (ms * 1e-3) / 1e9
    peak, _ = hbm_peak()
    return {
        "workload": "dot fp32 N=2^31, fp64 accumulation (BASELINE config 4), 1 GPU",
        "kernel_ms": round(ms, 3), "gbs": round(gbs, 1), "frac_hbm": round(gbs / peak, 4),
        "e2e_ms_pageable_numpy": round(min(e2e) * 1e3, 1), "e2e_h2d_bytes": 8 * n,
        "rel_err_vs_oracle": rel,
        "parity": "within 1e-12 (tolerance 1e-5) of the fp64 oracle" if rel <= 1e-12
                  else ("within 1e-5" if rel <= 1e-5 else "MISMATCH"),
    }


def dev_ordinal(rt) -> int:
    return rt.device_objects()[0].ordinal


def multi_heat(rt, dev, lib, D, rank: int, world: int) -> dict:
    """Config 2 across the ranks (strong scaling): 2^28 cells x 1000 steps
    in slabs, one process per GPU, the halo exchange fused into each pass
    as peer stores through CUDA IPC (bench.ProcessHeatSlabs).  Each rank
    generates only its slab of the reference input (PCG64 advanced to the
    slab's first cell).  Parity: rank 0 hashes the owned cells of every rank
    in order and compares with the reference's sha256."""
    import hashlib

    import numpy as np

    from paper_1810_11482_b200.bench import decomp
    from paper_1810_11482_b200.bench.harness import ProcessHeatSlabs

    n, steps, halo = 1 << 28, 1000, 96
    sl = decomp.slabs(n, world, halo)[rank]
    bg = np.random.PCG64(20180214)
    bg.advance(sl.start)
    x_local = np.random.Generator(bg).random(sl.length)
    slabs = ProcessHeatSlabs(rt, dev, x_local, halo=halo, n=n)
    st = rt.device_objects()[0].stream(0)
    t = EventTimer(lib, st, dev_ordinal(rt))

    def one(k: int) -> float:
        slabs.reset(x_local)
        D.barrier()
        t.start()
        slabs.run(k).get(timeout=300)
        ms = t.stop()
        D.barrier()
        return D.max(ms)

    one(halo)  # warm-up: IPC mappings, first launches
    times = [one(steps) for _ in range(2)]
    mine = slabs.owned()
    digest = None
    dd, torch = D.dist, D.torch
    if rank == 0:
        h = hashlib.sha256(mine)
        for r in range(1, world):
            size = torch.zeros(1, dtype=torch.int64)
            dd.recv(size, src=r)
            buf = torch.empty(int(size.item()), dtype=torch.uint8)
            dd.recv(buf, src=r)
            h.update(buf.numpy().tobytes())
        digest = h.hexdigest()
    else:
        dd.send(torch.tensor([len(mine)], dtype=torch.int64), dst=0)
        dd.send(torch.frombuffer(bytearray(mine), dtype=torch.uint8), dst=0)
    slabs.close()
    ref = next((c for c in _golden("golden_long.json").get("heat", [])
                if c["n"] == n and c["steps"] == steps), None)
    ms = min(times)
    useful = 2.0 * n * steps
    fp64 = fp64_peak_ops(lib, st)
    return {
        "workload": f"heat 2^28 fp64 x 1000 steps (BASELINE config 2) over {world} GPUs, one "
                    "process each, slabs with the halo exchange fused into the pass (peer stores "
                    "via CUDA IPC, halo 96)",
        "scaling": "strong", "n_gpus": world, "kernel_ms_max_over_ranks": round(ms, 3),
        "frac_fp64_per_gpu": round(useful / (ms * 1e-3) / (fp64 * world), 4) if fp64 else None,
        "parity": None if rank else ("bit-exact vs reference (golden_long.json)"
                                     if ref and digest == ref["sha256"] else "MISMATCH vs reference"),
    }


def multi_dot(rt, dev, lib, D, rank: int, world: int) -> dict:
    """Config 4 across the ranks (strong scaling): 2^31 fp32 elements in
    contiguous shards, the cross-GPU sum fused into the reduction kernel over
    CUDA-IPC-mapped peer memory (collectives.ProcessPeerGroup)."""
    import numpy as np

    import oracle
    from paper_1810_11482_b200.bench import decomp
    from paper_1810_11482_b200.collectives import ProcessPeerGroup

    n = 1 << 31
    lo, hi = decomp.shard_bounds(n, world)[rank:rank + 2]
    m = hi - lo
    rng = np.random.default_rng(20180214 + rank)
    a = rng.random(m, dtype=np.float32)
    b = rng.random(m, dtype=np.float32)
    A, B, R = dev.create_buffer(m * 4).get(), dev.create_buffer(m * 4).get(), dev.create_buffer(8).get()
    A.enqueue_write(0, a)
    B.enqueue_write(0, b).get()
    part = oracle.dot_f32(a, b, threads=0)
    del a, b
    grp = ProcessPeerGroup(rt, dev)
    st = rt.device_objects()[0].stream(0)
    for _ in range(3):
        grp.dot_f32(A, B, R, m)
    dev.synchronize().get()
    t = EventTimer(lib, st, dev_ordinal(rt))
    K = 10
    D.barrier()
    t.start()
    for _ in range(K):
        grp.dot_f32(A, B, R, m)
    ms = D.max(t.stop() / K)
    got = float(np.frombuffer(R.enqueue_read(0, 8).get(), np.float64)[0])
    total = D.sum(part)
    D.barrier()
    grp.close()
    rel = abs(got - total) / abs(total)
    peak, _ = hbm_peak()
    gbs = 8.0 * n / (ms * 1e-3) / 1e9
    out = {
        "workload": f"dot fp32 N=2^31 (BASELINE config 4) over {world} GPUs, one process each, "
                    "partials exchanged inside the reduction kernel over peer memory",
        "scaling": "strong", "n_gpus": world, "kernel_ms_max_over_ranks": round(ms, 4),
        "gbs_whole_job": round(gbs, 1), "frac_hbm_per_gpu": round(gbs / (peak * world), 4),
        "rel_err_vs_oracle": rel,
        "parity": "within 1e-12 (tolerance 1e-5)" if rel <= 1e-12 else
                  ("within 1e-5" if rel <= 1e-5 else "MISMATCH"),
    }
    # the same step with the library collective instead: the dot_f32 builtin
    # into R, then one ncclAllReduce of the 8-byte partial on the same stream
    try:
        from paper_1810_11482_b200.collectives import Communicator

        comm = Communicator.from_process_group(rt, dev)
        prog = dev.create_builtin_program().get()
        prog.build("dot_f32").get()
        grid = (max(1, m // 256), 1, 1)

        def step() -> None:
            prog.run([A, B, R, m], "dot_f32", grid, (256, 1, 1))
            comm.allreduce([R], count=1, dtype="f64")

        for _ in range(3):
            step()
        dev.synchronize().get()
        D.barrier()
        t.start()
        for _ in range(K):
            step()
        ms_nccl = D.max(t.stop() / K)
        got = float(np.frombuffer(R.enqueue_read(0, 8).get(), np.float64)[0])
        comm.close()
        rel_nccl = abs(got - total) / abs(total)
        out["nccl_allreduce"] = {
            "kernel_ms_max_over_ranks": round(ms_nccl, 4),
            "gbs_whole_job": round(8.0 * n / (ms_nccl * 1e-3) / 1e9, 1),
            "rel_err_vs_oracle": rel_nccl,
            "parity": "within 1e-12 (tolerance 1e-5)" if rel_nccl <= 1e-12 else
                      ("within 1e-5" if rel_nccl <= 1e-5 else "MISMATCH"),
        }
    except Exception as exc:  # noqa: BLE001 - reported beside the fused result
        out["nccl_allreduce"] = {"error": f"{type(exc).__name__}: {exc}"}
    return out


def multi_mandelbrot(rt, dev, lib, D, rank: int, world: int) -> dict:
    """Config 3 across the ranks: cyclic rows (row r -> rank r mod world),
    8 chunks per rank read straight into a pinned image; the images are
    summed to rank 0 (disjoint rows) and hashed against the reference's."""
    import hashlib

    from paper_1810_11482_b200 import when_all
    from paper_1810_11482_b200.bench.harness import MandelbrotTiles

    w, h, it = 7680, 4320, 2000
    tiles = MandelbrotTiles([dev], w, h, it, chunks=8, shard=(rank, world))
    tiles.image[:] = 0
    when_all(tiles.enqueue()).get()
    wall = []
    for _ in range(5):
        D.barrier()
        t0 = time.perf_counter()
        when_all(tiles.enqueue()).get()
        wall.append(D.max(time.perf_counter() - t0))
    dd, torch = D.dist, D.torch
    img = torch.from_numpy(tiles.image.view("int32").copy())
    dd.reduce(img, dst=0, op=dd.ReduceOp.SUM)
    ref = next((c for c in _golden("golden.json").get("mandelbrot", [])
                if c["width"] == w and c["height"] == h and c["max_iter"] == it), None)
    ok = rank == 0 and ref is not None and \
        hashlib.sha256(img.numpy().tobytes()).hexdigest() == ref["sha256"]
    return {
        "workload": f"Mandelbrot 7680x4320 @2000 (BASELINE config 3) over {world} GPUs, one "
                    "process each, cyclic rows into each rank's pinned image",
        "scaling": "strong", "n_gpus": world,
        "e2e_ms_max_over_ranks": round(min(wall) * 1e3, 3),
        "parity": None if rank else ("bit-exact vs reference sha256" if ok else "MISMATCH"),
    }


def run_multi_configs(rt, dev, lib, D, rank: int, world: int, names, out: dict) -> dict:
    for name in names:
        t0 = time.time()
        fn = {"heat": multi_heat, "dot": multi_dot, "mandelbrot": multi_mandelbrot}[name]
        try:
            out[name] = fn(rt, dev, lib, D, rank, world)
        except Exception as exc:  # noqa: BLE001 - reported; the headline still prints
            out[name] = {"error": f"{type(exc).__name__}: {exc}"}
        out[name]["wall_s"] = round(time.time() - t0, 1)
        dev.synchronize().get()
    return out


def run_configs(rt, dev, lib, names, out: dict) -> dict:
    st = rt.device_objects()[0].stream(0)
    fp64 = fp64_peak_ops(lib, st)
    for name in names:
        t0 = time.time()
        fn = {"heat": lambda: config_heat(rt, dev, lib, fp64),
              "mandelbrot": lambda: config_mandelbrot(rt, dev, lib, fp64),
              "dot": lambda: config_dot(rt, dev, lib)}[name]
        try:
            out[name] = fn()
        except Exception as exc:  # noqa: BLE001 - reported, the headline still prints
            out[name] = {"error": f"{type(exc).__name__}: {exc}"}
        out[name]["wall_s"] = round(time.time() - t0, 1)
        dev.synchronize().get()
    return out


def run_ours(args) -> None:
    import numpy as np

    from paper_1810_11482_b200 import Runtime, _native, pinned_empty
    from paper_1810_11482_b200.bindings import kernel_source

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)
    dist = Dist(world, local_rank)
    lib = _native.load()
    n = args.n
    s = 3.0

    ngpu = _native.device_count()
    ordinal = local_rank % max(1, ngpu)  # > GPUs ranks only in plumbing tests
    oversubscribed = world > ngpu
    # threads and pinned staging next to this GPU (one rank per GPU on a
    # multi-socket host); nothing to do on a single NUMA node
    from paper_1810_11482_b200.device import bind_host_to_device

    host_binding = None if oversubscribed else bind_host_to_device(ordinal)
    rt = Runtime(devices=[ordinal])
    dev = rt.get_all_devices().get()[0]
    A, B, C = (dev.create_buffer(n * 8).get() for _ in range(3))
    rng = np.random.default_rng(20180214 + rank)
    b_host = pinned_empty(n * 8, np.float64)
    c_host = pinned_empty(n * 8, np.float64)
    a_host = pinned_empty(n * 8, np.float64)
    b_host[:] = rng.random(n)
    c_host[:] = rng.random(n)
    prog = dev.create_program_with_source(kernel_source("stream")).get()
    B.enqueue_write(0, b_host)
    C.enqueue_write(0, c_host)
    prog.build("triad").get()
    targs = [A, B, C, s, n]
    grid, block = ((n + 255) // 256, 1, 1), (256, 1, 1)

    # parity before timing: bit-exact against the CPU oracle
    prog.run(targs, "triad", grid, block)
    A.enqueue_read_into(0, a_host).get()
    import oracle

    expect = oracle.stream("triad", b_host, c_host, s, threads=0)
    if not np.array_equal(a_host.view(np.uint64), expect.view(np.uint64)):
        raise SystemExit("triad parity FAILED: device result differs from the CPU oracle")

    for _ in range(args.warmup):
        prog.run(targs, "triad", grid, block)
    dev.synchronize().get()

    stream = rt.device_objects()[0].stream(0)
    ev0, ev1 = ctypes.c_void_p(), ctypes.c_void_p()
    _native.check(lib.ofl_event_create(ordinal, ctypes.byref(ev0)), "event")
    _native.check(lib.ofl_event_create(ordinal, ctypes.byref(ev1)), "event")
    sampler = ClockSampler(ordinal)
    dist.barrier()
    launches0 = lib.ofl_kernel_launches()
    sampler.start()
    lib.ofl_event_record(ev0, stream.ptr)
    for _ in range(args.steps):
        prog.run(targs, "triad", grid, block)
    lib.ofl_event_record(ev1, stream.ptr)
    ms = ctypes.c_float()
    _native.check(lib.ofl_event_elapsed_ms(ev0, ev1, ctypes.byref(ms)), "elapsed")
    clocks = sampler.stop()
    launches = lib.ofl_kernel_launches() - launches0
    total_ms = ms.value
    dist.barrier()
    job_ms = dist.max(total_ms)
    clocks_per_rank = dist.gather(dict(clocks, rank=rank, ordinal=ordinal, device_ms=total_ms))
    if world > 1:
        # the job's clock summary: the slowest rank's median, all reasons seen
        meds = [c["sm_mhz"] for c in clocks_per_rank if c.get("sm_mhz")]
        clocks = dict(clocks, sm_mhz=min(meds) if meds else clocks.get("sm_mhz"),
                      reasons=sorted({r for c in clocks_per_rank for r in c.get("reasons", [])}))

    step_bytes = 24 * n
    value = world * step_bytes * args.steps / (job_ms * 1e-3) / 1e9
    avg_launch_ms = total_ms / args.steps  # this rank's kernel, back to back
    achieved = step_bytes / (avg_launch_ms * 1e-3) / 1e9
    peak, peak_src = hbm_peak()

    # end-to-end through the public API with host buffers: per step two
    # pinned H2D writes, the run, a D2H read into pinned memory; steps
    # alternate between two streams and two device buffer sets (Alg. 1
    # style) so step k's read overlaps step k+1's writes on the full-duplex
    # link; every step's copies are inside the timed region.
    nsets = max(2, args.e2e_sets)
    sets = [(A, B, C, 0)] + [tuple(dev.create_buffer(n * 8).get() for _ in range(3))
                             + (dev.create_stream(),) for _ in range(nsets - 1)]
    outs = [a_host] + [pinned_empty(n * 8, np.float64) for _ in range(nsets - 1)]

    def e2e(steps: int, compute: bool = True) -> None:
        pending = []
        for k in range(steps):
            Ak, Bk, Ck, sk = sets[k % nsets]
            if len(pending) == nsets:
                pending.pop(0).get()
            Bk.enqueue_write(0, b_host, sk)
            Ck.enqueue_write(0, c_host, sk)
            if compute:
                prog.run([Ak, Bk, Ck, s, n], "triad", grid, block, sk)
            pending.append(Ak.enqueue_read_into(0, outs[k % nsets], sk))
        for t in pending:
            t.get()

    def timed_e2e(compute: bool) -> float:
        e2e(4, compute)
        dist.barrier()
        t0 = time.perf_counter()
        e2e(args.e2e_steps, compute)
        return dist.max(time.perf_counter() - t0)

    # the same copies with no kernel: the host link's floor for this schedule
    link_s = timed_e2e(False)
    e2e_s = timed_e2e(True)
    e2e_value = world * step_bytes * args.e2e_steps / e2e_s / 1e9
    for o in outs:
        if not np.array_equal(o.view(np.uint64), expect.view(np.uint64)):
            raise SystemExit("triad e2e parity FAILED")

    overhead = None
    if rank == 0 and not args.no_overhead:
        ks = tuple(int(k) for k in args.overhead_ks.split(",") if k)
        overhead = OverheadBench(dev, rt).sweep(ks)

    cpu = None
    if rank == 0 and world == 1 and args.cpu_seconds > 0:
        r = cpu_triad_rate(n, args.cpu_seconds, 1)
        cpu = {
            "value": round(r["gbs"], 3), "unit": "GB/s", "cores": 1, "kind": "port",
            "sample": f"{r['reps']} single-thread triad sweeps of N={n} fp64 "
            f"({r['seconds']:.1f} s) with the C restatement in oracle/ (the reference "
            "executes each launch sequentially on one core)",
        }

    traffic = ncu_traffic().get("triad")
    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(job_ms / args.steps, 5),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": workload_config(n, world),
        "roofline": {
            "bound": "hbm",
            "achieved": round(achieved, 2),
            "peak": peak,
            "unit": "GB/s",
            "frac": round(achieved / peak, 4),
            "frac_of_spec": round(achieved / SPEC_HBM_GBS, 4),
            "traffic": traffic,
            "peak_source": peak_src,
            "kernel": "k_stream_tile<TRIAD,512,1,PDL> (csrc/k_stream.cu; programmatic dependent launch)",
            "algorithmic_bytes_per_launch": step_bytes,
            "avg_launch_us": round(avg_launch_ms * 1e3, 3),
        },
        "e2e": {
            "value": round(e2e_value, 3),
            "unit": "GB/s",
            "h2d_bytes_per_step": 2 * n * 8,
            "d2h_bytes_per_step": n * 8,
            "steps": args.e2e_steps,
            "ms_per_step": round(e2e_s / args.e2e_steps * 1e3, 3),
            "link_floor_ms_per_step": round(link_s / args.e2e_steps * 1e3, 3),
            "frac_of_link_floor": round(link_s / e2e_s, 4),
            "schedule": "write b, write c (pinned), run, read_into a (pinned) per step; "
            f"steps rotate over {nsets} streams x {nsets} device buffer sets; wall clock; "
            "link floor = the same writes and reads with no kernel",
        },
        "cpu_baseline": cpu,
        "host_binding": host_binding or "unchanged (the GPU's local CPUs are all allowed, or unknown)",
        "gpu_launches": int(launches),
        "clocks": clocks,
        "clocks_per_rank": clocks_per_rank if world > 1 else None,
        "future_overhead_us": overhead,
        "configs": None,
        "parity": "bit-exact vs CPU oracle (oracle/ofl_oracle.c)",
        "oversubscribed": oversubscribed,
    }

    # configs 2-4 after the headline.  A watchdog bounds them: if they have
    # not finished within --configs-budget seconds (a hung peer exchange on
    # some rank, say), every rank leaves and rank 0 still prints the headline
    # with the configs that did finish.
    names = [c for c in args.configs.split(",") if c]
    multi = world > 1 and names and (not oversubscribed or args.force_multi)
    if (rank == 0 and world == 1 and names) or multi:
        configs: dict = {}
        line["configs"] = configs
        finished = threading.Event()

        def watchdog() -> None:
            if finished.wait(args.configs_budget):
                return
            if rank == 0:
                done = dict(configs)  # one C-level copy: the main thread may still insert
                for name in names:
                    done.setdefault(name, {"error": f"not finished within --configs-budget "
                                                    f"{args.configs_budget:g} s"})
                done["overhead"] = overhead
                print(json.dumps(dict(line, configs=done)), flush=True)
            os._exit(0)

        threading.Thread(target=watchdog, daemon=True).start()
        if multi:
            # configs 2-4 across the ranks (every rank takes part; rank 0 reports)
            run_multi_configs(rt, dev, lib, dist, rank, world, names, configs)
        else:
            run_configs(rt, dev, lib, names, configs)
        configs["overhead"] = overhead
        finished.set()

    if rank == 0:
        print(json.dumps(line), flush=True)
    rt.close()
    dist.close()


# Switches that change what runs (heat pass schedule, Mandelbrot without
# cycle detection, a substitute library, no NVRTC): a headline number must
# come from the shipped defaults.
VARIANT_SWITCHES = ("OFL_HEAT_TB", "OFL_MANDEL_PERIOD", "OFL_LIB", "OFL_NO_JIT")


def refuse_variant_switches(args) -> None:
    set_ = [k for k in VARIANT_SWITCHES if k in os.environ]
    if set_ and not args.allow_variants:
        raise SystemExit(f"bench.py: refusing to run with run-changing switches set: {set_} "
                         "(unset them, or pass --allow-variants for a sweep)")


def spawn_ranks(n: int, argv: list) -> None:
    """--gpus N without torchrun: run N ranks (one per GPU) under
    torch.distributed.run on 127.0.0.1 and pass through rank 0's line."""
    import socket
    import subprocess

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    # torchrun would read "--n" as an abbreviation of its own options
    argv = ["--elements" if a == "--n" else
            ("--elements=" + a[4:] if a.startswith("--n=") else a) for a in argv]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]
    r = subprocess.run(cmd)
    if r.returncode:
        raise SystemExit(r.returncode)


def main(argv=None) -> None:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--elements", "--n", dest="n", type=int, default=1 << 25,
                    help="triad elements per GPU (default 2^25, BASELINE config 1)")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--e2e-sets", type=int, default=2,
                    help="device buffer sets / streams the e2e steps rotate over")
    ap.add_argument("--overhead-ks", default="1,10,100,1000,10000,100000",
                    help="chain lengths K of the per-future overhead sweep (config 5)")
    ap.add_argument("--no-overhead", action="store_true")
    ap.add_argument("--force-multi", action="store_true",
                    help="run the multi-GPU configs even with more ranks than GPUs (testing)")
    ap.add_argument("--allow-variants", action="store_true",
                    help="permit OFL_* run-changing switches (sweeps only, never a headline)")
    ap.add_argument("--configs", default="heat,mandelbrot,dot",
                    help="BASELINE configs 2-4 measured after the headline (N=1 only); '' = none")
    ap.add_argument("--configs-budget", type=float, default=600.0,
                    help="seconds the configs may take before the headline is printed without them")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-seconds", type=float, default=60.0,
                    help="--impl reference: approximate length of the K timed steps")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    refuse_variant_switches(args)
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        # one process per GPU: launch ourselves under torchrun (same command
        # line), exactly as the driver does for N>1
        spawn_ranks(args.gpus, sys.argv[1:] if argv is None else list(argv))
        return
    if world is not None and int(world) != args.gpus and args.impl == "ours":
        ap.error(f"--gpus {args.gpus} but WORLD_SIZE={world}: one rank per GPU expected")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
