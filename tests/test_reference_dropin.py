"""The reference's own Runtime, handles, when_all and bench harness driving
the CUDA dispatch through ``paper_1810_11482_b200.offloadrt_backend.attach``
(Option B), and the reference's futures test module run
against this package's futures.

Where the reference package comes from: ``/root/reference/pkg/src`` in the
build container, or ``baseline/_ref`` (the offline ``pip install --target``
of the reference that travels to the GPU box).  Nothing here copies
reference code; the reference is imported and run as-is.

* CPU (``-m "not gpu"``): against the null test double of libofl.so
  (tests/fakes/null_ofl.c), so the plumbing — gid routing by locality,
  reference handles' synchronous errors, reference ``when_all`` over CUDA
  device tokens, failed tokens, cross-locality ``copy``, unregister — is
  checked without a device; plus ``pkg/tests/test_futures.py`` with
  ``offloadrt.futures`` / ``offloadrt.errors`` aliased to this package.
* GPU: the same plumbing on a B200, then the reference's ``flows``-style
  data paths and its bench harness (``run_stencil``, ``run_sum``,
  ``run_mandelbrot``, ``run_partition`` — each validates the device's
  output against the reference's own oracle and raises
  ``ValidationFailedError`` on a mismatch) and the body of
  ``test_acceptance.py:56-88`` checked against tests/golden and oracle/.
"""

from __future__ import annotations

import os
import subprocess
import sys
import textwrap

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC_CANDIDATES = ("/root/reference/pkg/src", os.path.join(REPO, "baseline", "_ref"))
REF_TESTS = "/root/reference/pkg/tests"


def _ref_src():
    for p in REF_SRC_CANDIDATES:
        if os.path.isfile(os.path.join(p, "offloadrt", "__init__.py")):
            return p
    return None


PLUMBING = textwrap.dedent(
    r"""
    import sys, threading, time
    sys.path[:0] = [REF_SRC, REPO]
    import numpy as np
    from offloadrt import Runtime, when_all, copy
    from offloadrt.errors import BadArgsError, NotBuiltError, OobAccessError, UnknownGidError
    from offloadrt.bench import kernel_source
    from paper_1810_11482_b200.offloadrt_backend import attach, CudaLocality

    def raises(exc, fn):
        try:
            fn()
        except exc as e:
            return e
        raise AssertionError(f"{exc.__name__} not raised")

    rt = Runtime(backend="host")
    cuda = attach(rt, devices=[0])
    assert cuda.locality_id == 1 and rt.registry.self_locality_id == 0
    raises(ValueError, lambda: attach(rt, devices=[0], locality_id=0))
    devs = rt.get_all_devices().get()
    host, dev = devs[0], devs[-1]
    assert len(devs) == 2 and dev.gid.locality_id == 1
    assert type(dev).__module__ == "offloadrt.handles", type(dev)
    assert rt.dispatch(dev.gid) is cuda
    assert dev.device_info().get().capability >= (10, 0)
    assert [d.gid for d in rt.get_all_devices(10, 0).get()][-1] == dev.gid

    # buffers through the reference's BufferHandle
    b = dev.create_buffer(64).get()
    assert type(b).__module__ == "offloadrt.handles" and b.gid.locality_id == 1
    b.enqueue_write(0, bytes(range(64)))
    assert b.enqueue_read(8, 8).get(timeout=30) == bytes(range(8, 16))
    assert b.enqueue_read_sync(0, 4) == bytes(range(4))
    raises(OobAccessError, lambda: b.enqueue_write(60, b"12345"))
    raises(BadArgsError, lambda: b.enqueue_read(-1, 2))
    raises(BadArgsError, lambda: dev.create_buffer(0))

    # streams and synchronize
    assert dev.create_stream() == 1 and dev.create_stream() == 2
    w = [b.enqueue_write(0, bytes([i]) * 8, i % 3) for i in range(200)]
    assert when_all(w).get(timeout=30) is None          # the REFERENCE when_all
    assert dev.synchronize().get(timeout=30) is None

    # programs: build errors, launch-shape errors, failed runs
    p = dev.create_program_with_source(kernel_source("sum")).get()
    raises(NotBuiltError, lambda: p.run([b, b, 1], "sum", (1, 1, 1), (1, 1, 1)).get(timeout=30))
    p.build("sum").get(timeout=120)
    raises(BadArgsError, lambda: p.run([b, b, 2**32], "sum", (1, 1, 1), (1, 1, 1)))
    raises(BadArgsError, lambda: p.run([b, b, True], "sum", (1, 1, 1), (1, 1, 1)))
    hb = host.create_buffer(64).get()
    raises(BadArgsError, lambda: p.run([hb, b, 1], "sum", (1, 1, 1), (1, 1, 1)))
    e = raises(OobAccessError, lambda: when_all(
        [b.enqueue_write(0, b"x"), p.run([b, b, 17], "sum", (1, 1, 1), (32, 1, 1))]).get(timeout=30))
    assert "16" in str(e), e
    p.run([b, b, 16], "sum", (1, 1, 1), (32, 1, 1)).get(timeout=30)

    # then() chains and continuations over CUDA tokens, inside the reference's futures
    fired = threading.Event()
    when_all([b.enqueue_write(0, bytes(64))]).then(lambda _: fired.set())
    assert fired.wait(30)

    # copy across localities (reference handles.py:119-145: read, then write)
    b.enqueue_write(0, bytes(range(100, 164)))
    copy(b, 0, hb, 0, 64).get(timeout=30)
    assert hb.enqueue_read(0, 64).get(timeout=30) == bytes(range(100, 164))
    copy(hb, 8, b, 0, 8).get(timeout=30)
    assert b.enqueue_read(0, 8).get(timeout=30) == bytes(range(108, 116))

    # lifetime: unregister through the dispatch the reference selects
    rt.dispatch(b.gid).unregister(b.gid).get(timeout=30)
    raises(UnknownGidError, lambda: b.enqueue_read(0, 1).get(timeout=30))
    print("PLUMBING OK", flush=True)
    """
)

GPU_DATA = textwrap.dedent(
    r"""
    import hashlib, json, math
    sys.path.insert(0, TESTS)
    import oracle                                   # this repo's checker
    import flows                                    # tests/flows.py, the reference flows' shape
    from offloadrt.bench import (MandelbrotConfig, PartitionConfig, StencilConfig,
                                 TimingProtocol, enqueue_partition_round,
                                 prepare_partitions, run_mandelbrot, run_partition,
                                 run_stencil, run_sum)
    golden = json.load(open(GOLDEN))
    sha = lambda b: hashlib.sha256(b).hexdigest()
    proto = TimingProtocol(iterations=2, discard=1)

    # the reference bench harness validates each output against ITS OWN oracle
    for n in (1 << 10, 1 << 20):
        assert run_stencil(StencilConfig(n=n), dev, proto).validated
    for n in (1000, 1 << 20):
        assert run_sum(n, dev, proto).validated
    assert run_mandelbrot(MandelbrotConfig(width=96, height=64, max_iter=300), dev, proto).validated
    rep = run_partition(PartitionConfig(m=1, partitions=4), [dev], proto)
    assert rep.validated

    # test_acceptance.py:56-88 body: outputs byte-identical to the reference's
    rng = np.random.default_rng(101)
    for n in (2**3, 2**10, 2**20):
        x = rng.random(n)
        assert flows.device_stencil(dev, x) == oracle.stencil(x).tobytes(), n
    for n in (2**3, 2**10, 2**20):
        v = rng.integers(0, 2**32, size=n, dtype=np.uint32)
        rb = dev.create_buffer(4).get()
        ib = dev.create_buffer(n * 4).get()
        sp = dev.create_program_with_source(kernel_source("sum")).get()
        sp.build("sum").get(timeout=120)
        ib.enqueue_write(0, v.tobytes())
        sp.run([ib, rb, n], "sum", (1, 1, 1), (32, 1, 1))
        assert int(np.frombuffer(rb.enqueue_read(0, 4).get(timeout=60), np.uint32)[0]) == oracle.sum_u32(v)
    for case in golden["mandelbrot"]:
        if case["width"] * case["height"] > 1 << 20:
            continue
        w, h = case["width"], case["height"]
        ob = dev.create_buffer(w * h * 4).get()
        mp = dev.create_program_with_source(kernel_source("mandelbrot")).get()
        mp.build("mandelbrot").get(timeout=120)
        mp.run([ob, w, h, *case["viewport"], case["esc"], case["max_iter"]], "mandelbrot",
               (math.ceil(w * h / 256), 1, 1), (256, 1, 1))
        assert sha(ob.enqueue_read(0, w * h * 4).get(timeout=60)) == case["sha256"], (w, h)
    n, parts = prepare_partitions(PartitionConfig(m=1, partitions=4), [dev])
    assert n == 2_097_152
    out = np.frombuffer(b"".join(t.get(timeout=120) for t in enqueue_partition_round(parts)), np.float64)
    assert out.size == n and np.abs(out - 1.0).max() <= 1e-12
    for case in golden["stencil"]:
        if "seed" in case:
            x = np.random.default_rng(case["seed"]).random(case["n"])
            assert sha(flows.device_stencil(dev, x)) == case["sha256"], case["n"]
    print("GPU DATA OK", flush=True)
    """
)

TAIL = "rt.close()\nprint('CLOSED', flush=True)\n"


def _script(gpu: bool, ref_src: str) -> str:
    body = PLUMBING + (GPU_DATA if gpu else "") + TAIL
    return (body.replace("REF_SRC", repr(ref_src)).replace("REPO", repr(REPO))
            .replace("TESTS", repr(os.path.join(REPO, "tests")))
            .replace("GOLDEN", repr(os.path.join(REPO, "tests", "golden", "golden.json"))))


@pytest.fixture(scope="module")
def ref_src():
    p = _ref_src()
    if p is None:
        pytest.skip("reference package not importable here (no /root/reference, no baseline/_ref)")
    return p


def test_reference_runtime_over_cuda_dispatch_null_abi(ref_src):
    from test_host_logic_cpu import FAKE_LIB, FAKE_SRC

    os.makedirs(os.path.dirname(FAKE_LIB), exist_ok=True)
    subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-o", FAKE_LIB, FAKE_SRC], check=True)
    script = _script(False, ref_src)
    # the null double computes nothing: the OOB check is the bindings' pre-check
    env = dict(os.environ, OFL_LIB=FAKE_LIB, PYTHONDONTWRITEBYTECODE="1")
    r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PLUMBING OK" in r.stdout and "CLOSED" in r.stdout


@pytest.mark.gpu
def test_reference_runtime_over_cuda_dispatch_b200(ref_src):
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1")
    env.pop("OFL_LIB", None)
    r = subprocess.run([sys.executable, "-c", _script(True, ref_src)], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "GPU DATA OK" in r.stdout and "CLOSED" in r.stdout


SHIM_PLUGIN = textwrap.dedent(
    r"""
    # pytest plugin: offloadrt.futures / offloadrt.errors -> this package's
    import sys, types
    sys.path.insert(0, REPO)
    import paper_1810_11482_b200.errors as errors
    import paper_1810_11482_b200.futures as futures
    pkg = types.ModuleType("offloadrt")
    pkg.__path__ = []
    pkg.futures, pkg.errors = futures, errors
    sys.modules["offloadrt"] = pkg
    sys.modules["offloadrt.futures"] = futures
    sys.modules["offloadrt.errors"] = errors
    """
)


def test_reference_futures_suite_against_ours(tmp_path):
    """/root/reference/pkg/tests/test_futures.py — every futures law the
    reference tests (incl. :104-113 first error wins, random DAGs, racing
    fulfillers) — run unmodified against paper_1810_11482_b200.futures."""
    src = os.path.join(REF_TESTS, "test_futures.py")
    if not os.path.isfile(src):
        pytest.skip("reference test suite not present here")
    (tmp_path / "ofl_shim_plugin.py").write_text(SHIM_PLUGIN.replace("REPO", repr(REPO)))
    env = dict(os.environ, PYTHONPATH=str(tmp_path), PYTHONDONTWRITEBYTECODE="1")
    r = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "--noconftest", "-p", "ofl_shim_plugin",
         "-p", "no:cacheprovider", "--rootdir", str(tmp_path), "-c", os.devnull, src],
        env=env, capture_output=True, text=True, timeout=600, cwd=str(tmp_path))
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout, r.stdout[-2000:]


def test_device_info_equals_reference_snapshot(ref_src):
    """A daemon's DeviceInfo decoded by the reference client (its own class)
    equals this package's snapshot of the same device (reference
    tests/test_transport.py:54-59 compares the two)."""
    sys.path.insert(0, ref_src)
    try:
        from offloadrt.device import DeviceInfo as RefInfo
    finally:
        sys.path.remove(ref_src)
    from paper_1810_11482_b200.device import DeviceInfo

    ours = DeviceInfo("cuda0", (10, 0), 191502876672, 148)
    ref = RefInfo("cuda0", (10, 0), 191502876672, 148)
    assert ref == ours and ours == ref and hash(ours) == hash(DeviceInfo("cuda0", (10, 0),
                                                                         191502876672, 148))
    assert ours != RefInfo("cuda1", (10, 0), 191502876672, 148)
    assert ours != ("cuda0", (10, 0), 191502876672, 148)
