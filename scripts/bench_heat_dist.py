#!/usr/bin/env python
"""BASELINE config 2 with one process per GPU: the 1-D heat equation over
2^28 f64 cells, 1000 steps, 1-D slabs across G GPUs (strong scaling), halo
exchange fused into the pass kernels as peer stores over CUDA IPC mappings,
passes ordered by device-side gate kernels (bench.ProcessHeatSlabs).

    torchrun --nproc-per-node G --master-addr 127.0.0.1 scripts/bench_heat_dist.py \
        [--cells 268435456] [--steps 1000] [--halo 64]

Job time = CUDA events around the steps on each rank's stream, max over
ranks.  Parity: bit-exact against the oracle's heat equation when
--check (at the given size; use a small --cells for that)."""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, default=1 << 28)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--halo", type=int, default=64)
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    from paper_1810_11482_b200 import Runtime, _native
    from paper_1810_11482_b200.bench.harness import ProcessHeatSlabs

    if not dist.is_initialized():
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29541")
        dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    lib = _native.load()
    x = np.random.default_rng(20180214).random(args.cells)
    with Runtime(devices=[local % max(1, _native.device_count())]) as rt:
        dev = rt.get_all_devices().get()[0]
        slabs = ProcessHeatSlabs(rt, dev, x, halo=args.halo)
        slabs.run(min(args.halo, args.steps)).get(timeout=600)  # warm-up pass
        st = slabs.stream
        e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
        lib.ofl_event_create(st.device.ordinal, ctypes.byref(e0))
        lib.ofl_event_create(st.device.ordinal, ctypes.byref(e1))
        dist.barrier()
        lib.ofl_event_record(e0, st.ptr)
        tok = slabs.run(args.steps)
        lib.ofl_event_record(e1, st.ptr)
        tok.get(timeout=600)
        ms = ctypes.c_float()
        lib.ofl_event_elapsed_ms(e0, e1, ctypes.byref(ms))
        t = torch.tensor([ms.value], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ok = None
        if args.check:
            import oracle

            got = slabs.gather()
            warm = min(args.halo, args.steps)
            ok = got.tobytes() == oracle.heat(x, warm + args.steps, threads=0).tobytes()
        slabs.close()
    if rank == 0:
        print(json.dumps({
            "config": f"heat 1-D, {args.cells} cells, {args.steps} steps, {world} GPU(s), "
                      f"one process per GPU, halo {args.halo} via IPC peer stores",
            "ms_total": round(float(t.item()), 3),
            "cell_steps_per_s": round(args.cells * args.steps / (float(t.item()) * 1e-3), 1),
            "bitexact": ok,
        }), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
