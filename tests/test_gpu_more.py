"""More API behaviour on the B200: tracing (reference event log), adversarial
byte ranges (reference test_buffer.py hypothesis case), multi-device heat
with a temporal-blocking halo, dot over two logical devices."""

from __future__ import annotations

import os
import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_1810_11482_b200 import OobAccessError, Runtime
from paper_1810_11482_b200.bindings import kernel_source

pytestmark = pytest.mark.gpu


def test_event_log_records_ops_in_order():
    with Runtime(devices=[0], record_events=True) as rt:
        dev = rt.get_all_devices().get()[0]
        obj = rt.device_objects()[0]
        buf = dev.create_buffer(4096 * 8).get()
        prog = dev.create_program_with_source(kernel_source("partition")).get()
        prog.build("partition").get()
        s1 = dev.create_stream()
        buf.enqueue_write(0, bytes(4096 * 8), s1)
        prog.run([buf, 0, 4096], "partition", (16, 1, 1), (256, 1, 1), s1)
        buf.enqueue_read(0, 64, s1).get()
        log = obj.event_log()
        assert [e.op for e in log] == ["write", "run", "read"]
        assert [e.amount for e in log] == [4096 * 8, 4096, 64]
        assert all(e.engine == "cuda0-s1" and e.stream == s1 for e in log)
        assert all(0 <= e.start <= e.end for e in log)
        assert log[0].end <= log[1].start + 1e-3 and log[1].end <= log[2].start + 1e-3


def test_event_log_empty_when_off(rt):
    assert rt.device_objects()[0].event_log() == []


_RT = {}


def _dev():
    if "rt" not in _RT:
        _RT["rt"] = Runtime(devices=[0])
    return _RT["rt"].get_all_devices().get()[0]


@given(st.integers(0, 256), st.integers(0, 256), st.binary(max_size=256))
@settings(max_examples=150, deadline=None)
def test_adversarial_ranges_never_corrupt(offset, size, blob):
    dev = _dev()
    buf = dev.create_buffer(128).get()
    try:
        buf.enqueue_write(offset, blob)
    except OobAccessError:
        assert offset + len(blob) > 128
    try:
        data = buf.enqueue_read_sync(offset, size)
        assert offset + size <= 128 and len(data) == size
    except OobAccessError:
        assert offset + size > 128


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("halo,steps", [(64, 200), (16, 50), (7, 22), (1, 9)])
def test_heat_multi_device_temporal_halo(rt2, halo, steps, fused):
    from paper_1810_11482_b200.bench.harness import heat_multi

    import oracle

    devices = rt2.get_all_devices().get()
    x = np.random.default_rng(halo).random(200_003)
    got = heat_multi(devices, x, steps, halo=halo, fused=fused)
    assert got.tobytes() == oracle.heat(x, steps, threads=0).tobytes()


@pytest.mark.parametrize("parts,halo,steps", [(4, 64, 301), (5, 3, 40), (3, 64, 64), (2, 96, 250)])
def test_heat_fused_exchange_many_slabs(parts, halo, steps):
    """Peer-store halo exchange between several slabs (logical devices on
    GPU 0, each with its own streams, so passes really run concurrently and
    the cross-device ordering is exercised), on data that sends some warps
    down the unfused update path."""
    from paper_1810_11482_b200 import Runtime
    from paper_1810_11482_b200.bench.harness import heat_multi

    import oracle

    x = np.random.default_rng(parts).random(50_000 * parts + 17)
    x[1000:2500] = np.random.default_rng(1).standard_normal(1500)
    with Runtime(devices=[0] * parts) as rt:
        devices = rt.get_all_devices().get()
        got = heat_multi(devices, x, steps, halo=halo, fused=True)
    exp = oracle.heat(x, steps, threads=0)
    assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))


def test_heat_fused_exchange_real_peers():
    """Two physical GPUs when the box has them (NVLink peer stores)."""
    from paper_1810_11482_b200 import Runtime, _native
    from paper_1810_11482_b200.bench.harness import heat_multi

    import oracle

    if _native.device_count() < 2:
        pytest.skip("one GPU on this box: peer stores exercised on logical devices only")
    x = np.random.default_rng(5).random(1_000_003)
    with Runtime(devices=[0, 1]) as rt:
        got = heat_multi(rt.get_all_devices().get(), x, 200, halo=64, fused=True)
    assert got.tobytes() == oracle.heat(x, 200, threads=0).tobytes()


def test_dot_two_logical_devices_host_sum(rt2):
    from paper_1810_11482_b200.bench.harness import dot_multi

    import oracle

    devices = rt2.get_all_devices().get()
    a = np.random.default_rng(3).random(3_000_001, dtype=np.float32)
    b = np.random.default_rng(4).random(3_000_001, dtype=np.float32)
    got = dot_multi(devices, a, b, fused=False)  # partials summed on the host
    exp = oracle.dot_f32(a, b)
    assert abs(got - exp) <= 1e-12 * abs(exp)


@pytest.mark.parametrize("parts", [1, 2, 3, 5])
def test_dot_fused_peer_allreduce(parts):
    """Dot product with the cross-device sum fused into the reduction kernel
    (peer-memory exchange, rank-order sum): every device holds the same
    bits, within 1e-12 of the oracle; repeated rounds reuse the exchange
    blocks (parity slots, monotonic counters)."""
    from paper_1810_11482_b200.bench.harness import DotShards

    import oracle

    rng = np.random.default_rng(parts)
    a = rng.random(1_000_003 * parts, dtype=np.float32)
    b = rng.random(1_000_003 * parts, dtype=np.float32)
    exp = oracle.dot_f32(a, b, threads=0)
    with Runtime(devices=[0] * parts) as rt:
        shards = DotShards(rt.get_all_devices().get(), a, b, fused=True)
        for _ in range(5):
            shards.enqueue().get(timeout=60)
            vals = [np.frombuffer(r.enqueue_read(0, 8).get(), np.float64)[0] for r in shards.R]
            assert len(set(v.tobytes() for v in vals)) == 1
            assert abs(vals[0] - exp) <= 1e-12 * abs(exp)


FAULT_SCRIPT = r"""
import sys
sys.path.insert(0, sys.argv[1])
import numpy as np
from paper_1810_11482_b200 import Runtime, InternalError, when_all
from paper_1810_11482_b200.bindings import kernel_source

rt = Runtime(devices=[0])
dev = rt.get_all_devices().get()[0]
n = 1 << 20
A, B, C = (dev.create_buffer(n * 8).get() for _ in range(3))
p = dev.create_program_with_source(kernel_source("stream")).get()
p.build("triad").get()
p.run([A, B, C, 3.0, n], "triad", (n // 256, 1, 1), (256, 1, 1)).get()   # healthy
# corrupt the device pointer behind A (test-only): the kernel faults on the GPU
obj = rt.local._buffer(A.gid)
good = obj.ptr
obj.ptr = 0x10
bad = p.run([A, B, C, 3.0, n], "triad", (n // 256, 1, 1), (256, 1, 1))
after = B.enqueue_read(0, 8)           # queued behind the faulting kernel
chain = when_all([bad, after])
cont = bad.then(lambda v: "ran")       # armed before the fault lands
seen = []
for name, tok in (("then", cont), ("kernel", bad), ("read", after), ("when_all", chain)):
    try:
        tok.get(timeout=60)
        seen.append(name + ":ok")
    except InternalError as exc:
        seen.append(name + ":InternalError")
    except TimeoutError:
        seen.append(name + ":timeout")
# the context is poisoned (sticky error): new work fails instead of hanging
try:
    p.run([B, B, C, 3.0, n], "triad", (n // 256, 1, 1), (256, 1, 1)).get(timeout=60)
    seen.append("new:ok")
except InternalError:
    seen.append("new:InternalError")
except TimeoutError:
    seen.append("new:timeout")
obj.ptr = good
print(" ".join(seen), flush=True)
import os
os._exit(0)
"""


def test_device_fault_fails_tokens_not_hangs():
    """A kernel fault (sticky CUDA error) comes back as InternalError on the
    faulting op, on ops queued behind it and on their when_all, and later
    ops fail fast (SURVEY §5 failure detection).  Runs in a subprocess: the
    CUDA context is unusable afterwards."""
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", FAULT_SCRIPT, repo], capture_output=True,
                       text=True, timeout=300)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-500:]
    assert line == ("then:InternalError kernel:InternalError read:InternalError "
                    "when_all:InternalError new:InternalError"), line


@pytest.mark.parametrize("parts,w,h,steps", [(2, 130, 67, 9), (3, 129, 50, 12), (4, 1024, 256, 5),
                                             (1, 64, 64, 3)])
def test_heat2d_fused_row_slabs(parts, w, h, steps):
    """2-D heat over row slabs on concurrently running logical devices, ghost
    rows refreshed by peer stores from the step kernel; even and odd widths
    (row-batch and per-cell kernels)."""
    from paper_1810_11482_b200.bench.harness import heat2d_multi

    import oracle

    x = np.random.default_rng(parts * 100 + w).random(w * h)
    with Runtime(devices=[0] * parts) as rt:
        got = heat2d_multi(rt.get_all_devices().get(), x, w, h, steps)
    exp = oracle.heat2d(x, w, h, steps, threads=0)
    assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))


PLAIN_MANDEL_SCRIPT = r"""
import sys, hashlib, json
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
from flows import device_mandelbrot
from paper_1810_11482_b200 import Runtime
golden = json.load(open(sys.argv[1] + "/tests/golden/golden.json"))
with Runtime(devices=[0]) as rt:
    dev = rt.get_all_devices().get()[0]
    raw = device_mandelbrot(dev, 7680, 4320, 2000)
    assert hashlib.sha256(raw).hexdigest() == golden["mandelbrot"][7]["sha256"]
print("plain ok")
"""


def test_mandelbrot_plain_kernel_config3():
    """The kernel without cycle detection (OFL_MANDEL_PERIOD=0, the FP64
    roofline reference) still reproduces the reference's config-3 counts."""
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", PLAIN_MANDEL_SCRIPT, repo], capture_output=True,
                       text=True, timeout=300, env=dict(os.environ, OFL_MANDEL_PERIOD="0"))
    assert r.stdout.strip().endswith("plain ok"), r.stdout[-500:] + r.stderr[-1500:]


def test_stream_fifo_random_schedules(dev):
    """Reference test_acceptance.py:286-308 in spirit: random schedules of
    writes and reads on one stream behave exactly like their sequential
    application (every read sees the state at its position), over many
    schedules, plus a second stream joined by synchronize()."""
    rng = np.random.default_rng(2018)
    size = 256
    buf = dev.create_buffer(size).get()
    s1 = dev.create_stream()
    for schedule in range(200):
        model = bytearray(size)
        buf.enqueue_write(0, bytes(size)).get()
        checks = []
        for _ in range(int(rng.integers(5, 25))):
            off = int(rng.integers(0, size))
            n = int(rng.integers(0, size - off + 1))
            if rng.random() < 0.6:
                data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
                buf.enqueue_write(off, data)
                model[off:off + n] = data
            else:
                checks.append((buf.enqueue_read(off, n), bytes(model[off:off + n])))
        for tok, want in checks:
            assert tok.get(timeout=30) == want, schedule
        # a write on another stream becomes visible after synchronize()
        data = rng.integers(0, 256, 16, dtype=np.uint8).tobytes()
        buf.enqueue_write(8, data, s1)
        dev.synchronize().get(timeout=30)
        model[8:24] = data
        assert buf.enqueue_read(0, size).get(timeout=30) == bytes(model), schedule


IPC_DOT_SCRIPT = r"""
import os, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import torch.distributed as dist
import oracle
from paper_1810_11482_b200 import Runtime
from paper_1810_11482_b200.collectives import ProcessPeerGroup
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
n = 3_000_001
rng = np.random.default_rng(7)
a = rng.random(n, dtype=np.float32); b = rng.random(n, dtype=np.float32)
lo, hi = n * rank // world, n * (rank + 1) // world
import os
with Runtime(devices=[int(os.environ.get("TEST_DEVICE", "0"))]) as rt:
    dev = rt.get_all_devices().get()[0]
    A = dev.create_buffer((hi - lo) * 4).get(); B = dev.create_buffer((hi - lo) * 4).get()
    R = dev.create_buffer(8).get()
    A.enqueue_write(0, np.ascontiguousarray(a[lo:hi])); B.enqueue_write(0, np.ascontiguousarray(b[lo:hi]))
    grp = ProcessPeerGroup(rt, dev)
    exp = oracle.dot_f32(a, b, threads=0)
    vals = []
    for _ in range(4):
        grp.dot_f32(A, B, R, hi - lo).get(timeout=60)
        vals.append(np.frombuffer(R.enqueue_read(0, 8).get(), np.float64)[0])
    assert all(v.tobytes() == vals[0].tobytes() for v in vals)
    assert abs(vals[0] - exp) <= 1e-12 * abs(exp), (vals[0], exp)
    got = [None] * world
    dist.all_gather_object(got, vals[0].tobytes())
    assert len(set(got)) == 1
    dist.barrier()
    grp.close()
print(f"rank {rank} ipc ok", flush=True)
"""


def test_dot_fused_across_processes_ipc():
    """One process per device (two processes sharing GPU 0 here): exchange
    blocks mapped through CUDA IPC, partials exchanged inside the kernel;
    both ranks end with the identical total, within 1e-12 of the oracle."""
    import socket
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK=str(r),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", IPC_DOT_SCRIPT, repo], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=300) for p in procs]
    for r, (out, err) in enumerate(outs):
        assert f"rank {r} ipc ok" in out, out[-500:] + err[-2000:]


def test_c_abi_example_runs(tmp_path):
    """examples/triad_c_abi.c: a pure-C host drives libofl.so (streams,
    pinned memory, copies, the triad, ticket wait) — the boundary a cgo /
    JNI / N-API binding of the reference's dispatch seam would use."""
    import subprocess

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(repo, "paper_1810_11482_b200", "lib")
    exe = str(tmp_path / "triad_c")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-I", os.path.join(repo, "include"),
                    os.path.join(repo, "examples", "triad_c_abi.c"), "-L", lib, "-lofl",
                    f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 mismatches" in r.stdout


def test_python_examples_run():
    """examples/listing2_sum.py (the paper's workflow listing on this API) and,
    when the reference package is installed in baseline/_ref,
    examples/reference_runtime_on_b200.py (the unmodified reference runtime
    driving the B200 through offloadrt_backend.attach)."""
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(repo, "examples", "listing2_sum.py")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert ": 1000" in r.stdout
    ref = os.path.join(repo, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "offloadrt")):
        pytest.skip("reference package not installed (baseline/_ref)")
    env = dict(os.environ, PYTHONPATH=ref + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, os.path.join(repo, "examples", "reference_runtime_on_b200.py")],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "matches numpy" in r.stdout


IPC_HEAT_SCRIPT = r"""
import sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import torch.distributed as dist
import oracle
from paper_1810_11482_b200 import Runtime
from paper_1810_11482_b200.bench.harness import ProcessHeatSlabs
dist.init_process_group("gloo")
rank = dist.get_rank()
x = np.random.default_rng(3).random(int(sys.argv[2]) if len(sys.argv) > 2 else 40_001)
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 45
import os
with Runtime(devices=[int(os.environ.get("TEST_DEVICE", "0"))]) as rt:
    dev = rt.get_all_devices().get()[0]
    slabs = ProcessHeatSlabs(rt, dev, x, halo=16 if x.size < 100_000 else 96)
    slabs.run(steps).get(timeout=120)
    got = slabs.gather()
    slabs.close()
assert got.tobytes() == oracle.heat(x, steps, threads=0).tobytes()
print(f"rank {rank} heat ipc ok", flush=True)
"""


def test_heat_slabs_across_processes_ipc():
    """One process per device (two processes sharing GPU 0 here): slab
    buffers and completion counters shared through CUDA IPC, passes ordered
    by device-side gate kernels, halos stored straight into the neighbour's
    ghost cells: bit-identical to the single-device heat equation."""
    import socket
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK=str(r),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", IPC_HEAT_SCRIPT, repo], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=300) for p in procs]
    for r, (out, err) in enumerate(outs):
        assert f"rank {r} heat ipc ok" in out, out[-500:] + err[-2000:]
