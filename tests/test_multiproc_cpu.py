"""Multi-process (world_size 2, gloo, CPU) checks of the N>1 logic: the same
decomposition arithmetic the GPU harness uses (bench/decomp.py), with the
CPU oracle standing in for the device kernels and gloo for NCCL/NVLink:

* dot: contiguous shards + allreduce(sum) == whole-vector dot;
* heat: slabs with halo ghosts, exchange every `halo` steps == global run
  (bit-exact), for halo 1 and a temporal-blocking halo;
* Mandelbrot: cyclic rows assembled == whole image (bit-exact);
* timing: the job time is the max over ranks (bench.py's rule).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import oracle  # noqa: E402
from paper_1810_11482_b200.bench import decomp  # noqa: E402


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank: int, world: int, port: int) -> None:
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _dot_worker(rank, world, port):
    _init(rank, world, port)
    n = 1_000_003
    rng = np.random.default_rng(11)
    a = rng.random(n, dtype=np.float32)
    b = rng.random(n, dtype=np.float32)
    lo, hi = decomp.shard_bounds(n, world)[rank : rank + 2]
    part = torch.tensor([oracle.dot_f32(a[lo:hi], b[lo:hi])], dtype=torch.float64)
    dist.all_reduce(part)
    total = oracle.dot_f32(a, b)
    assert abs(part.item() - total) <= 1e-12 * abs(total)
    dist.destroy_process_group()


def _heat_worker(rank, world, port, halo, steps):
    _init(rank, world, port)
    n = 50_001
    x = np.random.default_rng(5).random(n)
    layout = decomp.slabs(n, world, halo)
    me = layout[rank]
    cur = x[me.start : me.start + me.length].copy()
    left = steps
    while left > 0:
        k = min(halo, left)
        cur = oracle.heat(cur, k)
        left -= k
        if left == 0:
            break
        reqs = []
        recv_bufs = []
        for sg, s_cell, dg, d_cell, cells in decomp.halo_exchanges(layout, halo):
            if sg == rank:
                reqs.append(dist.isend(torch.from_numpy(cur[s_cell : s_cell + cells].copy()), dst=dg))
            if dg == rank:
                buf = torch.empty(cells, dtype=torch.float64)
                reqs.append(dist.irecv(buf, src=sg))
                recv_bufs.append((d_cell, cells, buf))
        for r in reqs:
            r.wait()
        for d_cell, cells, buf in recv_bufs:
            cur[d_cell : d_cell + cells] = buf.numpy()
    owned = cur[me.left : me.left + me.owned].copy()
    gathered = [None] * world  # slab sizes differ: gather as objects
    dist.all_gather_object(gathered, owned)
    full = np.concatenate(gathered)
    assert full.tobytes() == oracle.heat(x, steps).tobytes()
    dist.destroy_process_group()


def _mandel_worker(rank, world, port):
    _init(rank, world, port)
    w, h = 97, 61
    mine = np.zeros(w * h, np.uint32)
    oracle.mandelbrot(w, h, max_iter=400, row_first=rank, row_step=world, out=mine)
    rows = list(decomp.cyclic_rows(h, world, rank))
    assert np.count_nonzero(mine.reshape(h, w)[[r for r in range(h) if r not in rows]]) == 0
    t = torch.from_numpy(mine.astype(np.int64))
    dist.all_reduce(t)  # rows are disjoint: the sum assembles the image
    assert t.numpy().astype(np.uint32).tobytes() == oracle.mandelbrot(w, h, max_iter=400).tobytes()
    dist.destroy_process_group()


def _timing_worker(rank, world, port):
    _init(rank, world, port)
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    assert t.item() == float(world)
    dist.destroy_process_group()


def _spawn(fn, *args):
    mp.spawn(fn, args=(2, _free_port()) + args, nprocs=2, join=True)


def test_dot_shards_allreduce():
    _spawn(_dot_worker)


@pytest.mark.parametrize("halo,steps", [(1, 9), (4, 13), (8, 8)])
def test_heat_slabs_halo_exchange(halo, steps):
    _spawn(_heat_worker, halo, steps)


def test_mandelbrot_cyclic_rows():
    _spawn(_mandel_worker)


def test_job_time_is_max_over_ranks():
    _spawn(_timing_worker)


def test_decomp_arithmetic():
    assert decomp.shard_bounds(10, 3) == [0, 3, 6, 10]
    lay = decomp.slabs(100, 3, 2)
    assert [(s.lo, s.hi, s.left, s.right) for s in lay] == [(0, 33, 0, 2), (33, 66, 2, 2), (66, 100, 2, 0)]
    ex = decomp.halo_exchanges(lay, 2)
    assert ex[0] == (0, 31, 1, 0, 2) and ex[1] == (1, 2, 0, 33, 2)
    assert list(decomp.cyclic_rows(10, 4, 1)) == [1, 5, 9]
    assert [decomp.partition_device(i, 3) for i in range(5)] == [0, 1, 2, 0, 1]
    with pytest.raises(ValueError):
        decomp.slabs(5, 3, 2)
