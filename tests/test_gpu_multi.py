"""Multi-GPU paths on PHYSICAL GPUs (NVLink peers).  Every test here skips
unless the box shows at least two CUDA devices, so the same suite exercises
real peers as soon as it runs on a multi-GPU node (the single-GPU box covers
the same code on logical devices / processes sharing GPU 0: test_gpu_more).

Covers SURVEY §8(e): the fused dot peer-allreduce and the NCCL allreduce
(one process driving all GPUs, and one process per GPU), Mandelbrot cyclic
rows, the heat slabs with the halo exchange fused into the pass kernel as
peer stores (one process, and one process per GPU over CUDA IPC), 2-D heat
row slabs, cross-device copy, and a 2-rank bench.py line."""

from __future__ import annotations

import hashlib
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu() -> int:
    from paper_1810_11482_b200 import _native

    _native.load()
    return _native.device_count()


@pytest.fixture(scope="module")
def ngpu():
    n = _ngpu()
    if n < 2:
        pytest.skip(f"{n} GPU on this box: multi-GPU paths are exercised on logical devices "
                    "and processes sharing GPU 0 (tests/test_gpu_more.py)")
    return n


@pytest.fixture(scope="module")
def rtp(ngpu):
    """A Runtime over up to 4 physical GPUs."""
    from paper_1810_11482_b200 import Runtime

    rt = Runtime(devices=list(range(min(ngpu, 4))))
    yield rt
    rt.close()


def test_dot_fused_peer_allreduce_physical(rtp):
    from paper_1810_11482_b200.bench.harness import DotShards

    devices = rtp.get_all_devices().get()
    rng = np.random.default_rng(11)
    n = 4_000_037 * len(devices)
    a, b = rng.random(n, dtype=np.float32), rng.random(n, dtype=np.float32)
    exp = oracle.dot_f32(a, b, threads=0)
    shards = DotShards(devices, a, b)
    assert shards.fused  # distinct physical GPUs, no communicator: the fused kernel
    for _ in range(6):
        shards.enqueue().get(timeout=60)
        vals = [np.frombuffer(r.enqueue_read(0, 8).get(), np.float64)[0] for r in shards.R]
        assert len({v.tobytes() for v in vals}) == 1
        assert abs(vals[0] - exp) <= 1e-12 * abs(exp)


def test_nccl_allreduce_group_physical(rtp):
    from paper_1810_11482_b200.collectives import Communicator

    devices = rtp.get_all_devices().get()
    comm = Communicator.single_process(rtp, devices)
    try:
        bufs = [d.create_buffer(64).get() for d in devices]
        for g, b in enumerate(bufs):
            b.enqueue_write(0, np.arange(8, dtype=np.float64) * (g + 1))
        comm.allreduce(bufs, count=8, dtype="f64").get(timeout=60)
        total = sum(range(1, len(devices) + 1))
        for b in bufs:
            assert np.frombuffer(b.enqueue_read(0, 64).get(), np.float64).tolist() == \
                (np.arange(8) * total).tolist()
        ubufs = [d.create_buffer(16).get() for d in devices]
        for g, b in enumerate(ubufs):
            b.enqueue_write(0, np.full(4, 2**32 - 1 - g, np.uint32))
        comm.allreduce(ubufs, count=4, dtype="u32").get(timeout=60)
        want = int(sum(np.uint64(2**32 - 1 - g) for g in range(len(devices))) % 2**32)
        for b in ubufs:
            assert np.frombuffer(b.enqueue_read(0, 16).get(), np.uint32).tolist() == [want] * 4
        # dot through the builtin + one NCCL allreduce
        from paper_1810_11482_b200.bench.harness import dot_multi

        rng = np.random.default_rng(12)
        a, b = rng.random(3_000_001, dtype=np.float32), rng.random(3_000_001, dtype=np.float32)
        got = dot_multi(devices, a, b, comm=comm)
        exp = oracle.dot_f32(a, b, threads=0)
        assert abs(got - exp) <= 1e-12 * abs(exp)
    finally:
        comm.close()


def test_mandelbrot_cyclic_rows_physical_config3(rtp, golden):
    from paper_1810_11482_b200.bench.harness import mandelbrot_multi

    devices = rtp.get_all_devices().get()
    for chunks in (1, 8):
        counts = mandelbrot_multi(devices, 7680, 4320, 2000, chunks=chunks)
        assert hashlib.sha256(counts.tobytes()).hexdigest() == golden["mandelbrot"][7]["sha256"]


@pytest.mark.parametrize("fused", [True, False])
def test_heat_slabs_physical(rtp, fused):
    from paper_1810_11482_b200.bench.harness import heat_multi

    x = np.random.default_rng(13).random((1 << 22) + 5)
    x[70_000:71_000] = -x[70_000:71_000]  # some tiles take the unfused update
    got = heat_multi(rtp.get_all_devices().get(), x, 301, halo=96, fused=fused)
    exp = oracle.heat(x, 301, threads=0)
    assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))


def test_heat2d_row_slabs_physical(rtp):
    from paper_1810_11482_b200.bench.harness import heat2d_multi

    w, h = 1030, 517
    x = np.random.default_rng(14).random(w * h)
    got = heat2d_multi(rtp.get_all_devices().get(), x, w, h, 25)
    exp = oracle.heat2d(x, w, h, 25, threads=0)
    assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))


def test_copy_across_physical_gpus(rtp):
    from paper_1810_11482_b200 import copy

    d0, d1 = rtp.get_all_devices().get()[:2]
    payload = np.random.default_rng(15).integers(0, 256, 3 << 20, dtype=np.uint8)
    a, b = d0.create_buffer(payload.size).get(), d1.create_buffer(payload.size + 64).get()
    a.enqueue_write(0, payload)
    copy(a, 0, b, 64, payload.size).get(timeout=60)
    assert b.enqueue_read(64, payload.size).get() == payload.tobytes()


def _two_procs(script: str, marker: str, extra_args=(), timeout=600):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK=str(r),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), TEST_DEVICE=str(r))
        procs.append(subprocess.Popen([sys.executable, "-c", script, REPO, *extra_args], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=timeout) for p in procs]
    for r, (out, err) in enumerate(outs):
        assert marker.format(r) in out, out[-500:] + err[-2000:]


def test_dot_fused_one_process_per_gpu(ngpu):
    from test_gpu_more import IPC_DOT_SCRIPT

    _two_procs(IPC_DOT_SCRIPT, "rank {} ipc ok")


def test_heat_slabs_one_process_per_gpu(ngpu):
    from test_gpu_more import IPC_HEAT_SCRIPT

    _two_procs(IPC_HEAT_SCRIPT, "rank {} heat ipc ok", ("2000003", "250"))


def test_dot_nccl_one_process_per_gpu(ngpu):
    """scripts/bench_dot_dist.py under torchrun: dot_f32 then one
    ncclAllReduce per step (and the fused combine), checked against the
    oracle inside the script."""
    for combine in ("nccl", "fused"):
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        r = subprocess.run(
            [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
             "--master-addr", "127.0.0.1", "--master-port", str(port),
             os.path.join(REPO, "scripts", "bench_dot_dist.py"), "--elements", str(1 << 24),
             "--steps", "3", "--combine", combine],
            cwd=REPO, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-1000:] + r.stderr[-3000:]


def test_bench_two_ranks(ngpu):
    """bench.py --gpus 2 without torchrun: two ranks, one per GPU, one line."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "100", "--warmup",
                        "3", "--configs", "", "--cpu-seconds", "0", "--overhead-ks", "10",
                        "--e2e-steps", "4"], cwd=REPO, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and not line["oversubscribed"]
    assert len(line["clocks_per_rank"]) == 2
    assert {c["ordinal"] for c in line["clocks_per_rank"]} == {0, 1}
