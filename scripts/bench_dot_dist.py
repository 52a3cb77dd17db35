#!/usr/bin/env python
"""BASELINE config 4: partitioned fp32 dot product, N = 2^31 total, across
1/2/4/8 GPUs (strong scaling); the per-GPU partials are combined inside the
reduction kernel over peer memory (default) or by one NCCL allreduce.

    torchrun --nproc-per-node G --master-addr 127.0.0.1 scripts/bench_dot_dist.py [--elements 2147483648] [--combine fused|nccl]

Each rank owns a contiguous shard (bench/decomp.shard_bounds), reduces it
with the dot_f32 builtin into an fp64 scalar on the device, and an
ncclAllReduce enqueued on the same stream leaves the total on every rank —
no host round trip inside the step.  Step time = CUDA events on the launch
stream, max over ranks; the result is checked against the CPU oracle
(fp64 chunked dot of the shard, summed over ranks with gloo).
"""

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
    ap.add_argument("--elements", type=int, default=1 << 31)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--combine", choices=("fused", "nccl"), default="fused",
                    help="fused: partials exchanged inside the reduction kernel over peer memory "
                         "(CUDA IPC mappings); nccl: dot_f32 then one ncclAllReduce")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    import oracle
    from paper_1810_11482_b200 import Runtime, _native
    from paper_1810_11482_b200.bench import decomp
    from paper_1810_11482_b200.collectives import Communicator, ProcessPeerGroup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    lib = _native.load()
    with Runtime(devices=[local % max(1, _native.device_count())]) as rt:
        dev = rt.get_all_devices().get()[0]
        lo, hi = decomp.shard_bounds(args.elements, world)[rank : rank + 2]
        m = hi - lo
        rng = np.random.default_rng(20180214 + rank)
        A = dev.create_buffer(max(4, m * 4)).get()
        B = dev.create_buffer(max(4, m * 4)).get()
        R = dev.create_buffer(8).get()
        part = 0.0
        chunk = 1 << 27
        for off in range(0, m, chunk):
            k = min(chunk, m - off)
            a = rng.random(k, dtype=np.float32)
            b = rng.random(k, dtype=np.float32)
            A.enqueue_write(off * 4, a)
            B.enqueue_write(off * 4, b).get()
            part += oracle.dot_f32(a, b, threads=0)
        comm = group = None
        if args.combine == "fused" and world > 1:
            group = ProcessPeerGroup(rt, dev)
        else:
            comm = (Communicator.from_process_group(rt, dev) if world > 1
                    else Communicator.single_process(rt, [dev]))
        prog = dev.create_builtin_program().get()
        prog.build("dot_f32").get()
        grid = (max(1, m // 256), 1, 1)

        def step():
            if group is not None:
                group.dot_f32(A, B, R, m)
                return
            prog.run([A, B, R, m], "dot_f32", grid, (256, 1, 1))
            if comm is not None:
                comm.allreduce([R], count=1, dtype="f64")

        for _ in range(args.warmup):
            step()
        dev.synchronize().get()
        st = rt.device_objects()[0].stream(0)
        e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
        lib.ofl_event_create(st.device.ordinal, ctypes.byref(e0))
        lib.ofl_event_create(st.device.ordinal, ctypes.byref(e1))
        if world > 1:
            dist.barrier()
        lib.ofl_event_record(e0, st.ptr)
        for _ in range(args.steps):
            step()
        lib.ofl_event_record(e1, st.ptr)
        ms = ctypes.c_float()
        lib.ofl_event_elapsed_ms(e0, e1, ctypes.byref(ms))
        t = torch.tensor([ms.value, part], dtype=torch.float64)
        if world > 1:
            mx = t[:1].clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            sm = t[1:].clone()
            dist.all_reduce(sm)
            job_ms, total = float(mx.item()), float(sm.item())
        else:
            job_ms, total = ms.value, part
        got = float(np.frombuffer(R.enqueue_read(0, 8).get(), np.float64)[0])
        if rank == 0:
            step_ms = job_ms / args.steps
            print(json.dumps({
                "config": "dot f32 N=%d across %d GPU(s), %s" % (
                    args.elements, world, "partials exchanged in-kernel over peer memory"
                    if group is not None else "NCCL allreduce"),
                "ms_per_step": round(step_ms, 4),
                "gbs_whole_job": round(8.0 * args.elements / (step_ms * 1e-3) / 1e9, 1),
                "result": got, "oracle": total, "rel_err": abs(got - total) / abs(total),
                "within_1e-5": abs(got - total) <= 1e-5 * abs(total),
            }), flush=True)
        if not abs(got - total) <= 1e-12 * abs(total):
            raise SystemExit(f"rank {rank}: dot parity FAILED ({got} vs {total})")
        if comm is not None:
            comm.close()
        if group is not None:
            dist.barrier()
            group.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
