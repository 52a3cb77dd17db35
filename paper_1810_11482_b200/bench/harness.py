"""The reference's benchmark workloads on the CUDA runtime, plus the B200
configurations of BASELINE.json.

Mirrors /root/reference/pkg/src/offloadrt/bench/harness.py (configs,
validators, run_stencil / run_partition / run_mandelbrot(_series) / run_sum,
CSV rows) so callers of the reference harness switch over unchanged, and
adds the multi-device compositions the reference never runs:

* ``heat_multi``       — 1-D slab decomposition, halo exchange between
                         devices every `halo` steps (config 2);
* ``mandelbrot_multi`` — cyclic row split across devices, host-side image
                         assembly overlapped with the remaining devices'
                         compute (config 3);
* ``dot_multi``        — partitioned fp32 dot product + one NCCL allreduce
                         (config 4);
* ``run_stream``       — STREAM copy/scale/add/triad (config 1).

Every run validates its output before a time is reported, like the
reference (harness.py:1-7); validators are vectorised numpy restatements of
the kernels (the reference's own validator functions, harness.py:123-158).
"""

from __future__ import annotations

import csv
import math
import os
import time
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from ..bindings import kernel_source
from ..errors import BadArgsError, ValidationFailedError
from ..futures import task_pool, when_all
from ..handles import BufferHandle, DeviceHandle, ProgramHandle, copy
from ..hostmem import pinned_empty
from . import decomp
from .image import write_image
from .timing import TimingProtocol, measure

DEFAULT_SEED = 20180214
VIEWPORT = (-2.0, 1.0, -1.5, 1.5)


# -- configs (reference harness.py:45-95) -------------------------------------


@dataclass(frozen=True)
class StencilConfig:
    n: int
    block_x: int = 32

    def __post_init__(self):
        if self.n < 3:
            raise BadArgsError("stencil needs n >= 3")


@dataclass(frozen=True)
class PartitionConfig:
    m: int
    partitions: int
    block_size: int = 256

    def __post_init__(self):
        if not 1 <= self.m <= 8:
            raise BadArgsError("partition m must be in 1..8")
        if self.partitions < 1:
            raise BadArgsError("partition count must be positive")

    def vector_length(self, num_devices: int) -> int:
        n = (2**self.m) * 1024 * self.block_size
        return n * self.partitions if num_devices == 1 else n


@dataclass(frozen=True)
class MandelbrotConfig:
    width: int
    height: int
    max_iter: int = 256
    escape_radius: float = 2.0
    viewport: tuple = VIEWPORT
    async_write: bool = False

    def __post_init__(self):
        if self.width * self.height < 1:
            raise BadArgsError("image must have at least one pixel")


@dataclass(frozen=True)
class BenchReport:
    benchmark: str
    backend: str
    devices: int
    partitions: int
    n_or_pixels: int
    mean_ms: float
    validated: bool
    config: dict = field(default_factory=dict, compare=False)


CSV_FIELDS = ["benchmark", "backend", "devices", "partitions", "n_or_pixels", "mean_ms", "validated"]


def append_csv(path, report: BenchReport) -> None:
    fresh = not os.path.exists(path) or os.path.getsize(path) == 0
    with open(path, "a", newline="") as fh:
        w = csv.writer(fh)
        if fresh:
            w.writerow(CSV_FIELDS)
        w.writerow([report.benchmark, report.backend, report.devices, report.partitions,
                    report.n_or_pixels, f"{report.mean_ms:.6f}", "1" if report.validated else "0"])


# -- validators (reference harness.py:123-158) ----------------------------------


def stencil_oracle(x: np.ndarray) -> np.ndarray:
    y = x.copy()
    y[1:-1] = 0.5 * x[:-2] + x[1:-1] + 0.5 * x[2:]
    return y


def sum_oracle(values: np.ndarray) -> int:
    return int(values.astype(np.uint64).sum()) & 0xFFFFFFFF


def mandelbrot_oracle(cfg: MandelbrotConfig) -> np.ndarray:
    w, h = cfg.width, cfg.height
    re0, re1, im0, im1 = cfg.viewport
    idx = np.arange(w * h, dtype=np.int64)
    cre = re0 + ((idx % w).astype(np.float64) + 0.5) * (re1 - re0) / float(w)
    cim = im0 + ((idx // w).astype(np.float64) + 0.5) * (im1 - im0) / float(h)
    zr = np.zeros(idx.size)
    zi = np.zeros(idx.size)
    count = np.zeros(idx.size, dtype=np.uint32)
    live = np.ones(idx.size, dtype=bool)
    limit = cfg.escape_radius * cfg.escape_radius
    for _ in range(cfg.max_iter):
        live &= ~(zr * zr + zi * zi > limit)
        if not live.any():
            break
        a, b = zr[live], zi[live]
        t = a * a - b * b + cre[live]
        zi[live] = 2.0 * a * b + cim[live]
        zr[live] = t
        count[live] += 1
    return count


def _expect_equal(actual: np.ndarray, expected: np.ndarray, what: str) -> None:
    if actual.shape != expected.shape or not np.array_equal(actual, expected):
        bad = np.flatnonzero(actual != expected) if actual.shape == expected.shape else [0]
        i = int(bad[0]) if len(bad) else 0
        raise ValidationFailedError(
            f"{what}: first mismatch at index {i}: device={actual.flat[i]!r} "
            f"oracle={expected.flat[i] if expected.size > i else None!r}"
        )


def _build(device: DeviceHandle, name: str, source: Optional[str] = None) -> ProgramHandle:
    prog = device.create_program_with_source(source or kernel_source(name)).get()
    prog.build(name).get()
    return prog


def _builtin(device: DeviceHandle, name: str) -> ProgramHandle:
    prog = device.create_builtin_program().get()
    prog.build(name).get()
    return prog


# -- stencil (reference harness.py:199-230) ---------------------------------------


def run_stencil(cfg: StencilConfig, device: DeviceHandle,
                protocol: TimingProtocol = TimingProtocol(), seed: int = DEFAULT_SEED) -> BenchReport:
    x = np.random.default_rng(seed).random(cfg.n)
    payload = x.tobytes()
    xb = device.create_buffer(cfg.n * 8).get()
    yb = device.create_buffer(cfg.n * 8).get()
    prog = _build(device, "stencil")
    grid, block = (math.ceil(cfg.n / cfg.block_x), 1, 1), (cfg.block_x, 1, 1)
    result: dict = {}

    def iteration():
        xb.enqueue_write(0, payload)
        prog.run([xb, yb, cfg.n], "stencil", grid, block)
        result["out"] = yb.enqueue_read(0, cfg.n * 8).get()

    mean_ms = measure(iteration, protocol)
    _expect_equal(np.frombuffer(result["out"], np.float64), stencil_oracle(x), "stencil")
    return BenchReport("stencil", "cuda", 1, 1, cfg.n, mean_ms, True,
                       {"n": cfg.n, "block_x": cfg.block_x})


# -- partition: the paper's Alg. 1 (reference harness.py:236-335) ---------------


@dataclass
class PartitionPart:
    buffer: BufferHandle
    program: ProgramHandle
    stream: int
    offset: int
    count: int
    payload: object
    block_size: int


def prepare_partitions(cfg: PartitionConfig, devices: Sequence[DeviceHandle],
                       seed: int = DEFAULT_SEED, pinned: bool = True):
    """One buffer + stream per partition, partition i on device i mod k; the
    kernel is built once per device.  Payloads are staged in pinned memory
    (zero-copy DMA) unless pinned=False."""
    if not devices:
        raise BadArgsError("partition needs at least one device")
    n = cfg.vector_length(len(devices))
    x = np.random.default_rng(seed).random(n)
    programs = [_build(d, "partition") for d in devices]
    base, extra = divmod(n, cfg.partitions)
    parts, offset = [], 0
    for i in range(cfg.partitions):
        count = base + (1 if i < extra else 0)
        dev = devices[i % len(devices)]
        if pinned:
            payload = pinned_empty(count * 8, np.float64)
            payload[:] = x[offset : offset + count]
        else:
            payload = x[offset : offset + count].tobytes()
        parts.append(PartitionPart(dev.create_buffer(count * 8).get(), programs[i % len(devices)],
                                   dev.create_stream(), offset, count, payload, cfg.block_size))
        offset += count
    return n, parts


def enqueue_partition_round(parts: Sequence[PartitionPart], into: Optional[list] = None) -> list:
    """Alg. 1: three rounds of asynchronous enqueues — all writes, all runs,
    all reads — ordered only by each partition's stream."""
    for p in parts:
        p.buffer.enqueue_write(0, p.payload, p.stream)
    for p in parts:
        p.program.run([p.buffer, p.offset, p.count], "partition",
                      (math.ceil(p.count / p.block_size), 1, 1), (p.block_size, 1, 1), p.stream)
    if into is not None:
        return [p.buffer.enqueue_read_into(0, out, p.stream) for p, out in zip(parts, into)]
    return [p.buffer.enqueue_read(0, p.count * 8, p.stream) for p in parts]


def run_partition(cfg: PartitionConfig, devices: Sequence[DeviceHandle],
                  protocol: TimingProtocol = TimingProtocol(), seed: int = DEFAULT_SEED,
                  tolerance: float = 1e-12) -> BenchReport:
    n, parts = prepare_partitions(cfg, devices, seed)
    outs = [pinned_empty(p.count * 8, np.float64) for p in parts]

    def iteration():
        for t in enqueue_partition_round(parts, outs):
            t.get()

    mean_ms = measure(iteration, protocol)
    out = np.concatenate(outs)
    if out.size != n:
        raise ValidationFailedError(f"partition returned {out.size} of {n} elements")
    dev = np.abs(out - 1.0)
    if dev.size and dev.max() > tolerance:
        i = int(np.argmax(dev > tolerance))
        raise ValidationFailedError(f"partition: element {i} is {out[i]!r}, expected 1.0 within {tolerance}")
    return BenchReport("partition", "cuda", len(devices), cfg.partitions, n, mean_ms, True,
                       {"m": cfg.m, "block_size": cfg.block_size})


# -- mandelbrot (reference harness.py:341-437) --------------------------------------


def compute_mandelbrot(cfg: MandelbrotConfig, device: DeviceHandle, protocol, validate=True):
    pixels = cfg.width * cfg.height
    out = device.create_buffer(pixels * 4).get()
    prog = _build(device, "mandelbrot")
    re0, re1, im0, im1 = cfg.viewport
    esc = cfg.escape_radius * cfg.escape_radius
    args = [out, cfg.width, cfg.height, re0, re1, im0, im1, esc, cfg.max_iter]
    host = pinned_empty(pixels * 4, np.uint32)

    def iteration():
        prog.run(args, "mandelbrot", (math.ceil(pixels / 256), 1, 1), (256, 1, 1))
        out.enqueue_read_into(0, host).get()

    mean_ms = measure(iteration, protocol)
    counts = np.array(host)
    if validate:
        _expect_equal(counts, mandelbrot_oracle(cfg), "mandelbrot")
    return counts, mean_ms


def run_mandelbrot(cfg: MandelbrotConfig, device: DeviceHandle,
                   protocol: TimingProtocol = TimingProtocol(), image_path=None) -> BenchReport:
    counts, mean_ms = compute_mandelbrot(cfg, device, protocol)
    if image_path is not None:
        write_image(counts, cfg.width, cfg.height, image_path, cfg.max_iter)
    return BenchReport("mandelbrot", "cuda", 1, 1, cfg.width * cfg.height, mean_ms, True,
                       {"width": cfg.width, "height": cfg.height, "max_iter": cfg.max_iter})


@dataclass(frozen=True)
class SeriesEvent:
    kind: str
    index: int
    start: float
    end: float


def run_mandelbrot_series(sizes: Sequence[int], device: DeviceHandle,
                          protocol: TimingProtocol = TimingProtocol(), async_write: bool = False,
                          out_dir=None, write_fn: Optional[Callable] = None):
    """Increasing square images; each is written to disk after it validates.
    With async_write the write of image i runs on the task pool while image
    i+1 computes (reference harness.py:393-437)."""
    write_fn = write_fn or write_image
    reports, events, writers = [], [], []

    def emit(counts, cfg, index):
        t0 = time.perf_counter()
        if out_dir is not None:
            path = os.path.join(out_dir, f"mandelbrot_{cfg.width}x{cfg.height}.ppm")
            write_fn(counts, cfg.width, cfg.height, path, cfg.max_iter)
        events.append(SeriesEvent("write", index, t0, time.perf_counter()))

    for index, size in enumerate(sizes):
        cfg = MandelbrotConfig(width=size, height=size, async_write=async_write)
        t0 = time.perf_counter()
        counts, mean_ms = compute_mandelbrot(cfg, device, protocol)
        events.append(SeriesEvent("compute", index, t0, time.perf_counter()))
        reports.append(BenchReport("mandelbrot", "cuda", 1, 1, size * size, mean_ms, True,
                                   {"width": size, "height": size, "async_write": async_write}))
        if async_write:
            writers.append(task_pool().submit(emit, counts, cfg, index))
        else:
            emit(counts, cfg, index)
    for w in writers:
        w.result()
    events.sort(key=lambda e: e.start)
    return reports, events


class MandelbrotTiles:
    """Config 3 on several devices: rows r with r mod G == g go to device g
    (cyclic split — contiguous bands leave devices idle); each
    device computes its rows packed densely.  A device's rows are computed in
    ``chunks`` launches alternating over two compute streams (the tail of
    one chunk overlaps the next); each chunk is read on a copy stream (which
    waits, on the device, for that chunk's launch only) with one strided DMA straight to its rows of the pinned host image
    (``enqueue_read_rows_into``), so the reads overlap the computation of the
    later chunks and no host-side scatter copy is needed.

    By default chunks are contiguous bands, each read by one linear DMA:
    with the interior test and cycle detection the kernel (1.3 ms for config
    3) is faster than the 132.7 MB read (2.4 ms), so the reads set the pace
    and linear copies beat strided ones (8 bands: 2.52 ms end to end, 8
    interleaved chunks 3.06, profiles/r02_mandel_chunks.txt).  With
    ``interleave`` chunk i of a device takes every chunks-th of its rows
    starting at its i-th, so every chunk samples the whole image and costs the
    same — the better split when the kernel, not the read, is the bound."""

    def __init__(self, devices: Sequence[DeviceHandle], width: int, height: int, max_iter: int,
                 viewport=VIEWPORT, esc: float = 4.0, stream: int = 0, chunks: int = 1,
                 interleave: bool = False, shard: Optional[tuple] = None):
        """``shard=(index, count)``: one process per GPU — the (single) device
        computes the rows of part `index` of `count` into its image; the
        other parts' rows are left untouched (another process owns them)."""
        self.devices = list(devices)
        self.width, self.height, self.max_iter = width, height, max_iter
        self.viewport, self.esc = viewport, esc
        if shard is not None:
            if len(self.devices) != 1 or not 0 <= shard[0] < shard[1]:
                raise BadArgsError("a shard is one device's part index < part count")
            self._total, self._index = shard[1], [shard[0]]
        else:
            self._total, self._index = len(self.devices), list(range(len(self.devices)))
        G = len(self.devices)
        self.rows = [len(decomp.cyclic_rows(height, self._total, self._index[g])) for g in range(G)]
        self.progs = [_builtin(d, "mandelbrot_rows") for d in self.devices]
        self.streams, self.parts = [], []
        self._reads = {}  # (device, chunk) -> ticket of the chunk's last read
        for g, d in enumerate(self.devices):
            r = self.rows[g]
            c = max(1, min(chunks, r))
            # chunked: kernels alternate over two compute streams (the tail
            # of one chunk overlaps the next), reads go on a third
            self.streams.append([stream] if c == 1 else
                                [d.create_stream(), d.create_stream(), d.create_stream()])
            if interleave:
                # (first device row, device-row step, rows)
                spans = [(i, c, (r - i + c - 1) // c) for i in range(c)]
            else:
                bounds = [r * i // c for i in range(c + 1)]
                spans = [(k0, 1, k1 - k0) for k0, k1 in zip(bounds, bounds[1:])]
            self.parts.append([(k0, step, cnt, d.create_buffer(max(4, cnt * width * 4)).get())
                               for k0, step, cnt in spans if cnt > 0])
        self.image = pinned_empty(width * height * 4, np.uint32)

    def enqueue(self) -> list:
        """Launch every chunk and its read into ``self.image``; returns the
        read tokens."""
        from .. import _native
        from ..completion import DeviceToken

        G = len(self.devices)
        P = self._total  # parts of the cyclic row split
        re0, re1, im0, im1 = self.viewport
        w = self.width
        toks = []
        for g in range(G):
            part = self._index[g]
            sids = self.streams[g]
            copy = sids[-1]
            split = len(sids) > 1
            if split:
                head = self.parts[g][0][3]
                dev_obj = head._runtime.local._buffer(head.gid).device
                s_copy = dev_obj.stream(copy)
            for i, (k0, step, cnt, buf) in enumerate(self.parts[g]):
                compute = sids[i % 2] if split else copy
                if split:
                    s_compute = dev_obj.stream(compute)
                    prev = self._reads.get((g, i))
                    if prev:  # WAR: the last read of this chunk's buffer
                        _native.check(s_compute.lib.ofl_stream_wait(s_compute.ptr, s_copy.ptr,
                                                                    prev), "chunk ordering")
                first = part + k0 * P  # image row of the chunk's first row
                items = (first + (cnt - 1) * step * P + 1) * w  # through its last row
                run = self.progs[g].run([buf, w, self.height, re0, re1, im0, im1, self.esc,
                                         self.max_iter, first, step * P], "mandelbrot_rows",
                                        (items // w, 1, 1), (w, 1, 1), compute)  # exactly items
                if split:
                    if type(run) is not DeviceToken:
                        run.get()  # a failed launch raises here
                    # the copy stream waits for this chunk only (device-side)
                    _native.check(s_copy.lib.ofl_stream_wait(s_copy.ptr, s_compute.ptr,
                                                             run._ticket), "chunk ordering")
                read = buf.enqueue_read_rows_into(0, self.image, w * 4, cnt, first * w * 4,
                                                  step * P * w * 4, copy)
                if split and type(read) is DeviceToken:
                    self._reads[(g, i)] = read._ticket
                toks.append(read)
        return toks

    def __call__(self, image: Optional[np.ndarray] = None) -> np.ndarray:
        when_all(self.enqueue()).get()
        if image is None:
            return np.array(self.image)
        image[:] = self.image
        return image


def mandelbrot_multi(devices: Sequence[DeviceHandle], width: int, height: int, max_iter: int,
                     viewport=VIEWPORT, esc: float = 4.0, chunks: int = 1,
                     interleave: bool = False) -> np.ndarray:
    return MandelbrotTiles(devices, width, height, max_iter, viewport, esc, chunks=chunks,
                           interleave=interleave)()


# -- heat equation across devices (config 2) ---------------------------------------


def _drive_slabs(a_handles: list, b_handles: list, layout: list, unit: int, rounds: list,
                 launch: Callable, what: str):
    """Run slab passes with the halo exchange fused into the kernels.

    Round r launches, on every device g (default stream), one pass from its
    current buffer into the other one; the pass writes its owned cells and
    peer-stores its first / last boundary strip into the neighbours' ghost
    cells of *their* next buffer (``unit`` bytes per cell or row).  Each
    device's pass first waits for its two neighbours' previous pass (RAW on
    the ghosts it reads, WAR on the ghosts it stores).  Returns the buffers
    swapped to (current, other) and a token for the last round."""
    import ctypes

    from .. import _native

    def objs(handles):
        return [h._runtime.local._buffer(h.gid) for h in handles]

    cur_h, nxt_h = list(a_handles), list(b_handles)
    cur, nxt = objs(cur_h), objs(nxt_h)
    G = len(layout)
    streams = [o.device.stream(0) for o in cur]
    ords = [o.device.ordinal for o in cur]
    lib = streams[0].lib
    prev = [0] * G
    ticket = ctypes.c_uint64()
    for arg in rounds:
        now = []
        for g in range(G):
            st = streams[g]
            for nb in (g - 1, g + 1):
                if 0 <= nb < G and prev[nb]:
                    _native.check(lib.ofl_stream_wait(st.ptr, streams[nb].ptr, prev[nb]),
                                  "halo ordering")
            up = (nxt[g - 1].ptr + (layout[g - 1].left + layout[g - 1].owned) * unit) if g else None
            down = nxt[g + 1].ptr if g + 1 < G else None
            _native.check(launch(lib, st, cur[g], nxt[g], layout[g], up, ords[g - 1] if g else -1,
                                 down, ords[g + 1] if g + 1 < G else -1, arg,
                                 ctypes.byref(ticket)), what)
            now.append(ticket.value)
        prev = now
        cur, nxt, cur_h, nxt_h = nxt, cur, nxt_h, cur_h
    tok = when_all([streams[g].token(prev[g]) for g in range(G)]) if rounds else None
    return cur_h, nxt_h, tok


class HeatSlabs:
    """1-D slab decomposition of the heat equation over several devices.

    Device g owns cells [lo_g, hi_g) and keeps `halo` ghost cells on each
    inner side.  Every `halo` steps it advances its slab by one temporal-
    blocked pass (the ghosts absorb the shrinking valid region) and the
    owned boundary strips must reach the neighbours' ghosts.  Global
    endpoints stay fixed because a slab's outer end is either the true
    endpoint or a ghost that is overwritten before use.

    Exchange (``fused``, default when halo <= 128 and all devices are in this
    process): the pass kernel itself stores its first / last `halo` owned
    cells into the neighbours' ghost cells through peer pointers (NVLink
    stores, ``ofl_heat_slab``), and each device's next pass waits on its two
    neighbours' previous pass (cross-device events) — no copy operations and
    no host round trip.  ``fused=False``: the pass runs through the public
    ``heat`` builtin and the strips move by device-side ``copy()``
    (``cudaMemcpyPeerAsync``) on the default streams of both ends."""

    def __init__(self, devices: Sequence[DeviceHandle], x: np.ndarray, halo: int = 1,
                 fused: Optional[bool] = None):
        G = len(devices)
        n = x.size
        if halo < 1:
            raise BadArgsError("halo must be >= 1")
        self.devices = list(devices)
        self.n, self.halo = n, halo
        try:
            self.layout = decomp.slabs(n, G, halo)
        except ValueError as exc:
            raise BadArgsError(str(exc)) from None
        self.bounds = decomp.shard_bounds(n, G)
        self.left = [s.left for s in self.layout]
        self.right = [s.right for s in self.layout]
        self.length = [s.length for s in self.layout]
        self.a, self.b = [], []
        for g, d in enumerate(self.devices):
            lo = self.layout[g].start
            local = np.ascontiguousarray(x[lo : lo + self.length[g]])
            A = d.create_buffer(self.length[g] * 8).get()
            B = d.create_buffer(self.length[g] * 8).get()
            A.enqueue_write(0, local.tobytes())
            self.a.append(A)
            self.b.append(B)
        self.fused = (halo <= 128) if fused is None else bool(fused)
        if self.fused and halo > 128:
            raise BadArgsError("the fused exchange needs halo <= 128 (one pass per exchange)")
        self.progs = None if self.fused else [_builtin(d, "heat") for d in self.devices]

    def _exchange(self, cur: list) -> list:
        return [copy(cur[sg], s_cell * 8, cur[dg], d_cell * 8, cells * 8)
                for sg, s_cell, dg, d_cell, cells in decomp.halo_exchanges(self.layout, self.halo)]

    def run(self, steps: int):
        if self.fused:
            return self._run_fused(steps)
        cur, nxt = self.a, self.b
        left = steps
        toks = []
        while left > 0:
            k = min(self.halo, left)
            for g, p in enumerate(self.progs):
                L = self.length[g]
                p.run([cur[g], nxt[g], L, k], "heat", (math.ceil(L / 256), 1, 1), (256, 1, 1))
            if k % 2:
                cur, nxt = nxt, cur
            left -= k
            if left > 0:
                toks = self._exchange(cur)
        self.a, self.b = cur, nxt
        return when_all(toks) if toks else None

    def _run_fused(self, steps: int):
        h = self.halo
        ks = [min(h, steps - done) for done in range(0, steps, h)]

        def launch(lib, st, cur, nxt, sl, up, up_dev, down, down_dev, k, ticket):
            return lib.ofl_heat_slab(st.ptr, cur.ptr, nxt.ptr, sl.length, k, sl.left,
                                     sl.left + sl.owned, up, up_dev, down, down_dev, h, ticket)

        self.a, self.b, tok = _drive_slabs(self.a, self.b, self.layout, 8, ks, launch,
                                           "heat slab pass")
        return tok

    def gather(self) -> np.ndarray:
        out = np.empty(self.n)
        reads = []
        for g in range(len(self.devices)):
            owned = self.bounds[g + 1] - self.bounds[g]
            reads.append((g, self.a[g].enqueue_read(self.left[g] * 8, owned * 8)))
        for g, t in reads:
            out[self.bounds[g] : self.bounds[g + 1]] = np.frombuffer(t.get(), np.float64)
        return out


class ProcessHeatSlabs:
    """Config 2 with one process per GPU (torchrun): rank g owns slab g of
    the 1-D heat equation.  The slabs' buffers and a per-rank completion
    counter are shared through CUDA IPC once at construction; each pass is
    (1) a one-thread gate kernel that waits on the device until both
    neighbours' counters show the previous pass done, (2) the slab pass with
    its boundary strips stored straight into the neighbours' ghost cells
    (ofl_heat_slab over the IPC mappings), (3) a one-thread kernel that
    publishes this rank's counter — no host synchronisation per exchange."""

    def __init__(self, rt, device: DeviceHandle, x: np.ndarray, halo: int = 64, group=None,
                 n: Optional[int] = None):
        """x: the whole vector, or (with ``n`` = the global length) only this
        rank's slab — its ``decomp.slabs(n, world, halo)[rank]`` cells, ghosts
        included — so no rank has to hold the whole field."""
        import ctypes

        import torch.distributed as dist

        from .. import _native

        if not 1 <= halo <= 128:
            raise BadArgsError("halo must be 1..128")
        lib = _native.load()
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        total = x.size if n is None else int(n)
        self.group, self.halo, self.n = group, halo, total
        try:
            self.layout = decomp.slabs(total, self.world, halo)
        except ValueError as exc:
            raise BadArgsError(str(exc)) from None
        self.bounds = decomp.shard_bounds(total, self.world)
        sl = self.layout[self.rank]
        if n is None:
            local = np.ascontiguousarray(np.asarray(x, dtype=np.float64)[sl.start : sl.start + sl.length])
        else:
            local = np.ascontiguousarray(x, dtype=np.float64)
            if local.size != sl.length:
                raise BadArgsError(f"rank {self.rank}'s slab has {sl.length} cells, got {local.size}")
        self.bufs = [device.create_buffer(local.nbytes, shareable=True).get() for _ in range(2)]
        self.bufs[0].enqueue_write(0, local.tobytes())
        self.block = device.create_buffer(64, shareable=True).get()  # [0] counter, [8] status
        objs = [rt.local._buffer(b.gid) for b in (*self.bufs, self.block)]
        self.ordinal = objs[0].device.ordinal
        self.stream = objs[0].device.stream(0)
        self._ptrs = [o.ptr for o in objs]
        mine = []
        for o in objs:
            h = ctypes.create_string_buffer(64)
            _native.check(lib.ofl_ipc_handle(o.ptr, h), "ipc handle")
            mine.append(h.raw)
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        self._opened = []
        self.peer = {}  # rank -> (bufA, bufB, block) device pointers in this process
        for r in (self.rank - 1, self.rank + 1):
            if 0 <= r < self.world:
                ptrs = []
                for h in allh[r]:
                    p = ctypes.c_void_p()
                    _native.check(lib.ofl_ipc_open(self.ordinal, h, ctypes.byref(p)), "ipc open")
                    self._opened.append(p.value)
                    ptrs.append(p.value)
                self.peer[r] = ptrs
        counters = [self.peer[r][2] for r in sorted(self.peer)]
        self.gate = device.create_buffer(8 * max(1, len(counters))).get()
        if counters:
            self.gate.enqueue_write(0, np.array(counters, dtype=np.uint64).tobytes()).get()
        self._gate_ptr = rt.local._buffer(self.gate.gid).ptr
        self._ncounters = len(counters)
        self.passes = 0
        self.cur = 0  # index of the buffer holding the current state
        dist.barrier(group=group)  # every mapping exists before anyone stores

    def run(self, steps: int):
        import ctypes

        from .. import _native

        lib = self.stream.lib
        st, h = self.stream, self.halo
        sl, g = self.layout[self.rank], self.rank
        ticket = ctypes.c_uint64()
        done = 0
        while done < steps:
            k = min(h, steps - done)
            nxt = 1 - self.cur
            _native.check(lib.ofl_gate_wait(st.ptr, self._gate_ptr, self._ncounters, self.passes,
                                            self._ptrs[2] + 8, ctypes.byref(ticket)), "gate wait")
            up = down = None
            if g - 1 in self.peer:
                left = self.layout[g - 1]
                up = self.peer[g - 1][nxt] + (left.left + left.owned) * 8
            if g + 1 in self.peer:
                down = self.peer[g + 1][nxt]
            _native.check(lib.ofl_heat_slab(
                st.ptr, self._ptrs[self.cur], self._ptrs[nxt], sl.length, k, sl.left,
                sl.left + sl.owned, up, self.ordinal, down, self.ordinal, h,
                ctypes.byref(ticket)), "heat slab pass")
            self.passes += 1
            _native.check(lib.ofl_gate_signal(st.ptr, self._ptrs[2], self.passes,
                                              ctypes.byref(ticket)), "gate signal")
            self.cur = nxt
            done += k
        return st.token(ticket.value) if steps else None

    def reset(self, local: np.ndarray) -> None:
        """Restart from `local` (this rank's slab cells, ghosts included).
        Call between runs, when no rank has a pass in flight (e.g. after a
        barrier): it rewrites the buffer the next pass reads."""
        self.bufs[0].enqueue_write(0, np.ascontiguousarray(local, dtype=np.float64))
        self.cur = 0

    def owned(self) -> bytes:
        """This rank's owned cells of the current state (raises if a gate
        timed out waiting for a neighbour)."""
        sl = self.layout[self.rank]
        mine = self.bufs[self.cur].enqueue_read(sl.left * 8, sl.owned * 8).get()
        status = np.frombuffer(self.block.enqueue_read(8, 8).get(), np.uint64)[0]
        if status:
            raise RuntimeError("heat slab gate timed out waiting for a neighbour")
        return mine

    def gather(self) -> np.ndarray:
        """The whole vector on every rank (host all-gather of the owned cells)."""
        import torch.distributed as dist

        sl = self.layout[self.rank]
        mine = np.frombuffer(self.bufs[self.cur].enqueue_read(sl.left * 8, sl.owned * 8).get(),
                             np.float64)
        status = np.frombuffer(self.block.enqueue_read(8, 8).get(), np.uint64)[0]
        if status:
            raise RuntimeError("heat slab gate timed out waiting for a neighbour")
        parts = [None] * self.world
        dist.all_gather_object(parts, mine, group=self.group)
        return np.concatenate(parts)

    def close(self) -> None:
        import torch.distributed as dist

        from .. import _native

        dist.barrier(group=self.group)  # nobody stores into mappings being closed
        lib = _native.load()
        for p in self._opened:
            lib.ofl_ipc_close(self.ordinal, p)
        self._opened = []


class Heat2DSlabs:
    """Row-slab decomposition of the 2-D heat equation (kernels/stencil2d.k)
    over several devices in this process.  Slab g holds its owned rows plus
    one ghost row on each inner side; each step is one ``ofl_stencil2d_slab``
    launch per device that writes the owned rows and stores its first / last
    owned row straight into the neighbours' ghost rows (NVLink peer stores),
    ordered after the neighbours' previous step by cross-device events —
    the same fused exchange as the 1-D ``HeatSlabs``."""

    def __init__(self, devices: Sequence[DeviceHandle], x: np.ndarray, w: int, h: int):
        G = len(devices)
        x = np.asarray(x, dtype=np.float64).reshape(h, w)
        try:
            self.layout = decomp.slabs(h, G, 1)
        except ValueError as exc:
            raise BadArgsError(str(exc)) from None
        self.devices, self.w, self.h = list(devices), w, h
        self.bounds = decomp.shard_bounds(h, G)
        self.a, self.b = [], []
        for g, d in enumerate(self.devices):
            sl = self.layout[g]
            local = np.ascontiguousarray(x[sl.start : sl.start + sl.length])
            A = d.create_buffer(local.nbytes).get()
            B = d.create_buffer(local.nbytes).get()
            A.enqueue_write(0, local.tobytes())
            B.enqueue_write(0, local.tobytes())
            self.a.append(A)
            self.b.append(B)

    def run(self, steps: int):
        w = self.w

        def launch(lib, st, cur, nxt, sl, up, up_dev, down, down_dev, _arg, ticket):
            return lib.ofl_stencil2d_slab(st.ptr, cur.ptr, nxt.ptr, w, sl.length, sl.left,
                                          sl.left + sl.owned, up, up_dev, down, down_dev, ticket)

        self.a, self.b, tok = _drive_slabs(self.a, self.b, self.layout, w * 8, [None] * steps,
                                           launch, "stencil2d slab step")
        return tok

    def gather(self) -> np.ndarray:
        out = np.empty((self.h, self.w))
        reads = []
        for g, sl in enumerate(self.layout):
            reads.append((g, self.a[g].enqueue_read(sl.left * self.w * 8, sl.owned * self.w * 8)))
        for g, t in reads:
            out[self.bounds[g] : self.bounds[g + 1]] = np.frombuffer(t.get(), np.float64).reshape(
                -1, self.w)
        return out.ravel()


def heat2d_multi(devices: Sequence[DeviceHandle], x: np.ndarray, w: int, h: int,
                 steps: int) -> np.ndarray:
    slabs = Heat2DSlabs(devices, x, w, h)
    slabs.run(steps)
    return slabs.gather()


def heat_multi(devices: Sequence[DeviceHandle], x: np.ndarray, steps: int, halo: int = 1,
               fused: Optional[bool] = None) -> np.ndarray:
    slabs = HeatSlabs(devices, np.asarray(x, dtype=np.float64), halo, fused)
    slabs.run(steps)
    return slabs.gather()


class HeatChunks:
    """Config 2 end to end from host memory, with the transfers overlapped
    with the steps (the reference's run_stencil, harness.py:199-230, moves
    the whole field in, steps, and reads it back in sequence).

    After T steps a cell depends only on the cells within T of it, so the
    field is cut into ``chunks`` contiguous pieces and piece k is computed
    on its own: its input range extended by ``steps`` cells on each inner
    side is written to a device buffer pair, the ``heat`` builtin advances
    that sub-field T steps — its ends held fixed, which is exact at the
    field's real ends and wrong only within T cells of an inner cut, outside
    the piece's own cells — and the piece's own cells are read back.  The
    result is bit-identical to stepping the whole field (every cell sees the
    same operations on the same values).  Pieces rotate over ``sets``
    buffer pairs, each on its own stream, so the write of piece k+1, the
    steps of piece k and the read of piece k-1 run at once: the host link
    (2 x n x 8 bytes, both directions busy) rather than the sum of copy and
    compute sets the pace.  Redundant work: 2 x steps cells per inner cut.
    Config 2 on one B200: 108.6 ms written, stepped and read in sequence,
    54-56 ms with 16-32 pieces over 6-8 pairs (profiles/r02_heat_e2e.txt);
    once short fields stopped paying a per-pass floor, 51-53 ms with 64
    pieces over 12 pairs, against ~45 ms for the same copies with no steps
    (profiles/r02_heat_small_fields.txt).  The pieces' steps must run
    concurrently: one compute stream running them in order (a write / step
    / read stream each) took 70 ms, small fields alone leave SMs idle.

    ``x`` and ``out`` are pinned float64 arrays of n cells (``pinned_empty``),
    read and written by DMA in place."""

    def __init__(self, device: DeviceHandle, n: int, steps: int, chunks: int = 64, sets: int = 12):
        if n < 3 or steps < 0 or chunks < 1 or sets < 1:
            raise BadArgsError("heat chunks: n >= 3, steps >= 0, chunks >= 1, sets >= 1")
        chunks = max(1, min(chunks, n // max(1, 2 * steps) or 1, n))
        self.device, self.n, self.steps = device, n, steps
        bounds = [n * i // chunks for i in range(chunks + 1)]
        # (own lo, own hi, extended lo, extended hi)
        self.pieces = [(lo, hi, max(0, lo - steps), min(n, hi + steps))
                       for lo, hi in zip(bounds, bounds[1:])]
        longest = max(ehi - elo for _, _, elo, ehi in self.pieces)
        self.prog = _builtin(device, "heat")
        self.sets = [(device.create_buffer(longest * 8).get(), device.create_buffer(longest * 8).get(),
                      device.create_stream()) for _ in range(max(1, min(sets, chunks)))]

    def enqueue(self, x: np.ndarray, out: np.ndarray) -> list:
        """Issue every piece (write, steps, read); returns the read tokens."""
        if x.dtype != np.float64 or out.dtype != np.float64 or x.size < self.n or out.size < self.n:
            raise BadArgsError("heat chunks: x and out must be float64 arrays of n cells")
        toks = []
        for k, (lo, hi, elo, ehi) in enumerate(self.pieces):
            X, Y, st = self.sets[k % len(self.sets)]
            m = ehi - elo
            X.enqueue_write(0, x[elo:ehi], st)
            self.prog.run([X, Y, m, self.steps], "heat", ((m + 255) // 256, 1, 1), (256, 1, 1), st)
            final = X if self.steps % 2 == 0 else Y
            toks.append(final.enqueue_read_into((lo - elo) * 8, out[lo:hi], st))
        return toks

    def __call__(self, x: np.ndarray, out: np.ndarray) -> np.ndarray:
        when_all(self.enqueue(x, out)).get()
        return out


# -- sum (reference harness.py:443-477) --------------------------------------------


def run_sum(n: int, device: DeviceHandle, protocol: TimingProtocol = TimingProtocol(),
            seed: int = DEFAULT_SEED, values: Optional[np.ndarray] = None) -> BenchReport:
    if n < 1:
        raise BadArgsError("sum needs n >= 1")
    if values is None:
        values = np.random.default_rng(seed).integers(0, 2**32, size=n, dtype=np.uint32)
    values = np.asarray(values, dtype=np.uint32)
    payload = values.tobytes()
    ib = device.create_buffer(n * 4).get()
    rb = device.create_buffer(4).get()
    prog = _build(device, "sum")
    result: dict = {}

    def iteration():
        ib.enqueue_write(0, payload)
        prog.run([ib, rb, n], "sum", (1, 1, 1), (32, 1, 1))
        result["out"] = rb.enqueue_read(0, 4).get()

    mean_ms = measure(iteration, protocol)
    actual = int(np.frombuffer(result["out"], np.uint32)[0])
    if actual != sum_oracle(values):
        raise ValidationFailedError(f"sum: device={actual} oracle={sum_oracle(values)}")
    return BenchReport("sum", "cuda", 1, 1, n, mean_ms, True, {"n": n})


# -- STREAM (config 1) -----------------------------------------------------------------


def run_stream(op: str, n: int, device: DeviceHandle, protocol: TimingProtocol = TimingProtocol(),
               seed: int = DEFAULT_SEED, scalar: float = 3.0) -> BenchReport:
    rng = np.random.default_rng(seed)
    b, c = rng.random(n), rng.random(n)
    A, B, C = (device.create_buffer(n * 8).get() for _ in range(3))
    B.enqueue_write(0, b.tobytes())
    C.enqueue_write(0, c.tobytes())
    prog = _build(device, op, kernel_source("stream"))
    args = {"copy": [A, B, n], "scale": [A, B, scalar, n], "add": [A, B, C, n],
            "triad": [A, B, C, scalar, n]}[op]
    grid, block = (math.ceil(n / 256), 1, 1), (256, 1, 1)

    def iteration():
        prog.run(args, op, grid, block).get()

    mean_ms = measure(iteration, protocol)
    got = np.frombuffer(A.enqueue_read(0, n * 8).get(), np.float64)
    exp = {"copy": b, "scale": scalar * b, "add": b + c, "triad": b + scalar * c}[op]
    _expect_equal(got, exp, f"stream {op}")
    nbytes = (16 if op in ("copy", "scale") else 24) * n
    return BenchReport(f"stream_{op}", "cuda", 1, 1, n, mean_ms, True,
                       {"n": n, "gbs": nbytes / (mean_ms * 1e-3) / 1e9})


# -- partitioned dot product + allreduce (config 4) ---------------------------------------


class DotShards:
    """a, b split contiguously over the devices; each device reduces its
    shard to one fp64 partial.  Combining the partials:

    * ``fused`` (default for several physical GPUs in this process, no ``comm``):
      the reduction kernel's last CTA exchanges the partials with the other
      devices over NVLink peer memory and sums them in rank order
      (``collectives.PeerGroup``) — one kernel per device, no collective call;
    * ``comm`` (a ``collectives.Communicator``): the dot_f32 builtin, then
      one NCCL allreduce on the same stream;
    * neither: partials summed on the host."""

    def __init__(self, devices: Sequence[DeviceHandle], a: np.ndarray, b: np.ndarray, comm=None,
                 fused: Optional[bool] = None):
        G = len(devices)
        n = a.size
        self.devices = list(devices)
        self.n = n
        self.bounds = decomp.shard_bounds(n, G)
        self.A, self.B, self.R = [], [], []
        for g, d in enumerate(self.devices):
            lo, hi = self.bounds[g], self.bounds[g + 1]
            A = d.create_buffer(max(4, (hi - lo) * 4)).get()
            B = d.create_buffer(max(4, (hi - lo) * 4)).get()
            if hi > lo:
                A.enqueue_write(0, np.ascontiguousarray(a[lo:hi]))
                B.enqueue_write(0, np.ascontiguousarray(b[lo:hi]))
            self.A.append(A)
            self.B.append(B)
            self.R.append(d.create_buffer(8).get())
        self.progs = [_builtin(d, "dot_f32") for d in self.devices]
        self.comm = comm
        if fused is None:  # default: distinct physical GPUs and no communicator
            ords = {d._runtime.local._device(d.gid).ordinal for d in self.devices}
            fused = comm is None and G > 1 and len(ords) == G
        self.fused = bool(fused)
        self.group = None
        if self.fused:
            from ..collectives import PeerGroup

            self.group = PeerGroup(self.devices[0]._runtime, self.devices)

    def enqueue(self):
        if self.fused:
            counts = [self.bounds[g + 1] - self.bounds[g] for g in range(len(self.devices))]
            return self.group.dot_f32(self.A, self.B, self.R, counts)
        for g, p in enumerate(self.progs):
            m = self.bounds[g + 1] - self.bounds[g]
            p.run([self.A[g], self.B[g], self.R[g], m], "dot_f32", (max(1, math.ceil(m / 256)), 1, 1),
                  (256, 1, 1))
        if self.comm is not None:
            return self.comm.allreduce(self.R, count=1, dtype="f64")
        return None

    def result(self) -> float:
        if self.comm is None and not self.fused:
            return float(sum(np.frombuffer(r.enqueue_read(0, 8).get(), np.float64)[0] for r in self.R))
        return float(np.frombuffer(self.R[0].enqueue_read(0, 8).get(), np.float64)[0])


def dot_multi(devices: Sequence[DeviceHandle], a: np.ndarray, b: np.ndarray, comm=None,
              fused: Optional[bool] = None) -> float:
    shards = DotShards(devices, a, b, comm, fused)
    shards.enqueue()
    return shards.result()
