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

    def __init__(self, index: int, period: float = 0.01):
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

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self._REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(self.period)

    def start(self):
        if self._nv is not None:
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


def overhead_sweep(dev, rt, steps_pipelined: int, steps_sync: int, payload_bytes: int = 8) -> dict:
    """Per-future overhead vs raw CUDA streams (BASELINE config 5)."""
    import numpy as np

    from paper_1810_11482_b200 import _native, make_ready, pinned_empty, when_all
    from paper_1810_11482_b200.bindings import kernel_source

    lib = _native.load()
    n = 1024
    A, B, C, D = (dev.create_buffer(n * 8).get() for _ in range(4))
    prog = dev.create_program_with_source(kernel_source("stream")).get()
    prog.build("triad").get()
    payload = pinned_empty(payload_bytes)
    payload[:] = 1
    args = [A, B, C, 3.0, n]
    grid, block = ((n + 255) // 256, 1, 1), (256, 1, 1)
    stream = rt.device_objects()[0].stream(0)
    dptr = rt.local._buffer(D.gid).ptr
    aptr, bptr, cptr = (rt.local._buffer(x.gid).ptr for x in (A, B, C))

    def raw(steps: int, mode: int) -> float:
        secs = ctypes.c_double()
        _native.check(
            lib.ofl_bench_raw_chain(
                stream.ptr, dptr, payload.ctypes.data, payload_bytes, aptr, bptr, cptr, n, steps,
                mode,
                ctypes.byref(secs),
            ),
            "raw chain",
        )
        return secs.value

    def capi(steps: int) -> float:
        # the product C-ABI (libofl tickets, same kernel launch) called from
        # Python without futures: splits the overhead into C-ABI + futures
        t = ctypes.c_uint64()
        ref = ctypes.byref(t)
        h2d, op, sp, src = lib.ofl_h2d, lib.ofl_stream_op, stream.ptr, payload.ctypes.data
        dev.synchronize().get()
        t0 = time.perf_counter()
        for _ in range(steps):
            h2d(sp, dptr, src, payload_bytes, ref)
            op(sp, 3, aptr, bptr, cptr, 3.0, n, ref)
        dev.synchronize().get()
        return time.perf_counter() - t0

    def pipelined(steps: int) -> float:
        dev.synchronize().get()
        t0 = time.perf_counter()
        prev = make_ready(None)
        for _ in range(steps):
            w = D.enqueue_write(0, payload)
            r = prog.run(args, "triad", grid, block)
            prev = when_all([prev, w, r])
        prev.get()
        return time.perf_counter() - t0

    def synced(steps: int) -> float:
        dev.synchronize().get()
        t0 = time.perf_counter()
        for _ in range(steps):
            D.enqueue_write(0, payload)
            prog.run(args, "triad", grid, block).get()
        return time.perf_counter() - t0

    # warm both paths
    raw(200, 0)
    capi(200)
    pipelined(200)
    raw(100, 2)
    synced(100)
    out = {}
    t_raw = min(raw(steps_pipelined, 0) for _ in range(3))
    t_capi = min(capi(steps_pipelined) for _ in range(3))
    t_fut = min(pipelined(steps_pipelined) for _ in range(3))
    out["pipelined_when_all"] = {
        "steps": steps_pipelined,
        "raw_us_per_step": t_raw / steps_pipelined * 1e6,
        "c_abi_us_per_step": t_capi / steps_pipelined * 1e6,
        "futurized_us_per_step": t_fut / steps_pipelined * 1e6,
        "overhead_us_per_step": (t_fut - t_raw) / steps_pipelined * 1e6,
        "overhead_us_per_future": (t_fut - t_raw) / steps_pipelined / 2 * 1e6,
    }
    t_raw = min(raw(steps_sync, 2) for _ in range(3))
    t_fut = min(synced(steps_sync) for _ in range(3))
    out["sync_each_step"] = {
        "steps": steps_sync,
        "raw_us_per_step": t_raw / steps_sync * 1e6,
        "futurized_us_per_step": t_fut / steps_sync * 1e6,
        "overhead_us_per_step": (t_fut - t_raw) / steps_sync * 1e6,
    }
    for v in out.values():
        for k in list(v):
            if isinstance(v[k], float):
                v[k] = round(v[k], 3)
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

    def e2e(steps: int) -> None:
        pending = []
        for k in range(steps):
            Ak, Bk, Ck, sk = sets[k % nsets]
            if len(pending) == nsets:
                pending.pop(0).get()
            Bk.enqueue_write(0, b_host, sk)
            Ck.enqueue_write(0, c_host, sk)
            prog.run([Ak, Bk, Ck, s, n], "triad", grid, block, sk)
            pending.append(Ak.enqueue_read_into(0, outs[k % nsets], sk))
        for t in pending:
            t.get()

    e2e(4)
    dist.barrier()
    t0 = time.perf_counter()
    e2e(args.e2e_steps)
    e2e_s = dist.max(time.perf_counter() - t0)
    e2e_value = world * step_bytes * args.e2e_steps / e2e_s / 1e9
    for o in outs:
        if not np.array_equal(o.view(np.uint64), expect.view(np.uint64)):
            raise SystemExit("triad e2e parity FAILED")

    overhead = None
    if rank == 0 and not args.no_overhead:
        overhead = overhead_sweep(dev, rt, args.overhead_steps, max(100, args.overhead_steps // 10))

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
    if rank == 0:
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
                "schedule": "write b, write c (pinned), run, read_into a (pinned) per step; "
                f"steps rotate over {nsets} streams x {nsets} device buffer sets; wall clock",
            },
            "cpu_baseline": cpu,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "future_overhead_us": overhead,
            "parity": "bit-exact vs CPU oracle (oracle/ofl_oracle.c)",
            "oversubscribed": oversubscribed,
        }
        print(json.dumps(line), flush=True)
    rt.close()
    dist.close()


def main(argv=None) -> None:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--n", type=int, default=1 << 25)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--e2e-sets", type=int, default=2,
                    help="device buffer sets / streams the e2e steps rotate over")
    ap.add_argument("--overhead-steps", type=int, default=10000)
    ap.add_argument("--no-overhead", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-seconds", type=float, default=60.0,
                    help="--impl reference: approximate length of the K timed steps")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
