"""Host-side logic of the CUDA runtime on CPU: handles, dispatch, argument
validation, bindings' out-of-bounds pre-checks, device tokens and when_all
over device tokens — driven against the null test double of libofl.so
(tests/fakes/null_ofl.c: same C-ABI, no device, every op completes at once).
Runs in a subprocess so the double never leaks into this process's
libofl handle; the product path never loads it on its own."""

from __future__ import annotations

import os
import subprocess
import sys
import textwrap

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAKE_SRC = os.path.join(REPO, "tests", "fakes", "null_ofl.c")
FAKE_LIB = os.path.join(REPO, "tests", "fakes", "_build", "libnull_ofl.so")

SCRIPT = textwrap.dedent(
    r"""
    import sys
    sys.path.insert(0, REPO_PATH)
    import numpy as np
    from paper_1810_11482_b200 import (Runtime, when_all, make_ready, BadArgsError,
        LaunchConfigError, NotBuiltError, OobAccessError, CompileError, UnknownGidError)
    from paper_1810_11482_b200.bindings import kernel_source

    def raises(exc, fn):
        try:
            fn()
        except exc:
            return
        raise AssertionError(f"{exc.__name__} not raised")

    with Runtime(devices=[0, 0]) as rt:
        d0, d1 = rt.get_all_devices().get()
        assert d0.info.name == "cuda0" and d0.info.capability == (10, 0)
        assert d0.create_stream() == 1 and d0.create_stream() == 2
        raises(BadArgsError, lambda: d0.create_buffer(0))
        buf = d0.create_buffer(64).get()
        raises(OobAccessError, lambda: buf.enqueue_write(60, b"12345"))
        raises(BadArgsError, lambda: buf.enqueue_read(-1, 1))
        buf.enqueue_write(0, b"abcdefgh")
        assert buf.enqueue_read(0, 8).get() == b"abcdefgh"   # fake copies synchronously
        out = bytearray(4)
        buf.enqueue_read_into(2, out).get()
        assert bytes(out) == b"cdef"

        p = d0.create_program_with_source(kernel_source("sum")).get()
        raises(NotBuiltError, lambda: p.run([buf, buf, 1], "sum", (1,1,1), (1,1,1)).get())
        p.build("sum").get()
        raises(BadArgsError, lambda: p.run([buf], "sum", (1,1,1), (1,1,1)).get())
        raises(BadArgsError, lambda: p.run([buf, 3, buf], "sum", (1,1,1), (1,1,1)).get())
        raises(BadArgsError, lambda: p.run([buf, buf, 2**32], "sum", (1,1,1), (1,1,1)))
        raises(BadArgsError, lambda: p.run([buf, buf, True], "sum", (1,1,1), (1,1,1)))
        raises(LaunchConfigError, lambda: p.run([buf, buf, 1], "sum", (0,1,1), (1,1,1)))
        raises(LaunchConfigError, lambda: p.run([buf, buf, 1], "sum", (2**20,1,1), (2**13,1,1)))
        other = d1.create_buffer(8).get()
        raises(BadArgsError, lambda: p.run([other, buf, 1], "sum", (1,1,1), (1,1,1)))
        # sum reading 17 words from a 16-word buffer: OOB at index 16
        raises(OobAccessError, lambda: p.run([buf, buf, 17], "sum", (1,1,1), (1,1,1)).get())
        p.run([buf, buf, 16], "sum", (1,1,1), (1,1,1)).get()

        s = d0.create_program_with_source(kernel_source("stencil")).get()
        s.build("stencil").get()
        x = d0.create_buffer(99 * 8).get()
        y = d0.create_buffer(100 * 8).get()
        try:
            s.run([x, y, 100], "stencil", (4,1,1), (32,1,1)).get()
        except OobAccessError as e:
            assert "index 99 " in str(e), e
        else:
            raise AssertionError("no OOB")
        raises(BadArgsError, lambda: s.run([y, y, 100], "stencil", (4,1,1), (32,1,1)).get())

        q = d0.create_program_with_source("kernel k(x : buffer_f64) { x[0] = nope; }").get()
        raises(CompileError, lambda: q.build("k").get())

        # device tokens + when_all chains (summarised per stream)
        prev = make_ready(None)
        toks = []
        for i in range(2000):
            w = buf.enqueue_write(0, bytes([i % 256]) * 8, i % 3)
            toks.append(w)
            prev = when_all([prev, w])
        assert prev.get() is None and all(t.done() for t in toks)
        fired = []
        when_all(toks[-5:]).then(lambda _: fired.append(1))
        import time
        t0 = time.time()
        while not fired and time.time() - t0 < 5:
            time.sleep(0.01)
        assert fired, "continuation never fired"
        assert d0.synchronize().get() is None

        # when_all runs every input's finish step and fails with its error
        # (reference futures.py:189-216; pkg/tests/test_futures.py:104-113)
        from paper_1810_11482_b200.completion import DeviceToken
        buf.enqueue_write(0, bytes(range(64)))
        big = d0.create_buffer(1 << 20).get()
        payload = np.random.default_rng(1).integers(0, 256, 1 << 20, dtype=np.uint8)
        big.enqueue_write(0, payload)
        out = bytearray(1 << 20)                       # pageable: lands via staging
        assert when_all([big.enqueue_read_into(0, out)]).get() is None
        assert bytes(out) == payload.tobytes(), "read_into not visible after when_all.get()"
        out2 = bytearray(1 << 20)
        seen = []
        agg = when_all([make_ready(), when_all([big.enqueue_read_into(0, out2)])])
        agg.then(lambda _: seen.append(bytes(out2) == payload.tobytes()))
        t0 = time.time()
        while not seen and time.time() - t0 < 5:
            time.sleep(0.01)
        assert seen == [True], f"then() on the aggregate ran before the landing: {seen}"
        out3 = bytearray(16)
        r = big.enqueue_read_into(0, out3)
        assert when_all([r]).done() and bytes(out3) == payload[:16].tobytes()
        st = rt.local._device(d0.gid).stream(0)
        tk = st.tail()
        def boom():
            raise OobAccessError("kernel buffer index 7 out of range")
        bad = DeviceToken(st, tk, boom)
        try:
            when_all([buf.enqueue_write(0, b"x"), bad, buf.enqueue_write(0, b"y")]).get()
        except OobAccessError as e:
            assert "index 7" in str(e)
        else:
            raise AssertionError("finish error swallowed by when_all")
        assert bad.is_failed() and "index 7" in str(bad.error())
        bad2 = DeviceToken(st, tk, boom)
        got = []
        when_all([bad2]).then(lambda _: got.append("ok")).then(
            lambda _: None)._on_done(lambda t: got.append(type(t.error()).__name__))
        t0 = time.time()
        while not got and time.time() - t0 < 5:
            time.sleep(0.01)
        assert got == ["OobAccessError"], got
        # large reads to pageable memory: chunked D2H collected in parallel
        huge = d0.create_buffer((9 << 20) + 24).get()
        pl = np.random.default_rng(2).integers(0, 256, (9 << 20) + 24, dtype=np.uint8)
        huge.enqueue_write(0, pl)                     # pageable staged write (> 8 MiB: 2 slots)
        assert huge.enqueue_read(0, pl.size).get() == pl.tobytes()
        assert huge.enqueue_read(8, 5 << 20).get() == pl[8:8 + (5 << 20)].tobytes()
        o = bytearray(pl.size)
        assert huge.enqueue_read_into(0, o).get() is o and bytes(o) == pl.tobytes()
        o2 = np.zeros(6 << 20, np.uint8)
        assert when_all([huge.enqueue_read_into(16, o2)]).get() is None
        assert o2.tobytes() == pl[16:16 + (6 << 20)].tobytes()
        dropped = huge.enqueue_read(0, pl.size)
        del dropped
        d0.synchronize().get()
        # launch plans / pinned-write plans: reused only for the same objects
        # under an unchanged registry generation
        from paper_1810_11482_b200 import pinned_empty
        tp = d0.create_program_with_source(kernel_source("stream")).get()
        tp.build("triad").get()
        TA, TB, TC = (d0.create_buffer(8 * 64).get() for _ in range(3))
        targs = [TA, TB, TC, 3.0, 64]
        g, blk = (1, 1, 1), (64, 1, 1)
        for _ in range(3):
            tp.run(targs, "triad", g, blk).get()
        assert tp._qc is not None and tp._qc[3][0] is TA
        targs[3] = 5.0                                  # a changed element: full path again
        tp.run(targs, "triad", g, blk).get()
        assert tp._qc[3][3] == 5.0
        pin = pinned_empty(64)
        pin[:] = 1
        TB.enqueue_write(0, pin).get()
        assert TB._wq is not None
        pin[:] = 7                                      # same array, new contents: re-sent
        TB.enqueue_write(0, pin).get()
        assert TB.enqueue_read(0, 64).get() == bytes([7]) * 64
        TB.enqueue_write(64, pin).get()                 # other offset: full path
        assert TB.enqueue_read(64, 64).get() == bytes([7]) * 64
        rt.registry.unregister(TC.gid)                  # generation moves: plans invalid
        raises(UnknownGidError, lambda: tp.run(targs, "triad", g, blk).get())
        rt.registry.unregister(TB.gid)
        raises(UnknownGidError, lambda: TB.enqueue_write(0, pin).get())
        bad3 = DeviceToken(st, tk, boom)
        assert when_all([when_all([bad3])]).is_failed()

        rt.registry.unregister(buf.gid)
        raises(UnknownGidError, lambda: buf.enqueue_read(0, 1).get())
    print("HOST-LOGIC OK")
    """
)


@pytest.fixture(scope="module")
def fake_lib():
    os.makedirs(os.path.dirname(FAKE_LIB), exist_ok=True)
    subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-o", FAKE_LIB, FAKE_SRC], check=True)
    return FAKE_LIB


def test_host_logic_against_null_abi(fake_lib):
    env = dict(os.environ, OFL_LIB=fake_lib)
    r = subprocess.run([sys.executable, "-c", SCRIPT.replace("REPO_PATH", repr(REPO))], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "HOST-LOGIC OK" in r.stdout


CALL_SRC = os.path.join(REPO, "paper_1810_11482_b200", "csrc", "oflcall.c")

CALL_SCRIPT = textwrap.dedent(
    r"""
    import ctypes, importlib.util, sys
    spec = importlib.util.spec_from_file_location("_oflcall", MOD_PATH)
    m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m)
    lib = ctypes.CDLL(LIB_PATH)
    addr = lambda f: ctypes.cast(f, ctypes.c_void_p).value
    try:
        m.h2d(1, 2, 3, 4)
        raise AssertionError("unbound call accepted")
    except RuntimeError:
        pass
    m.bind(addr(lib.ofl_h2d), addr(lib.ofl_stream_op), addr(lib.ofl_wait))
    s = ctypes.c_void_p()
    assert lib.ofl_stream_create(0, ctypes.byref(s)) == 0
    src = (ctypes.c_char * 8).from_buffer_copy(b"abcdefgh")
    dst = (ctypes.c_char * 8)()
    t1 = m.h2d(s.value, ctypes.addressof(dst), ctypes.addressof(src), 8)
    assert bytes(dst) == b"abcdefgh" and t1 >= 1
    t2 = m.stream_op(s.value, 3, 0, 0, 0, 3.0, 1024)
    assert t2 == t1 + 1                      # tickets come back as the C side wrote them
    assert m.h2d(0, 0, 0, 0) == -2           # a failing status comes back negated
    assert m.stream_op(None, 3, 0, 0, 0, 3, 8) == -2
    assert m.wait(s.value, t2) == 0
    for bad in (lambda: m.h2d(1, 2, 3), lambda: m.h2d(-1, 0, 0, 0), lambda: m.stream_op(1, 3, 0, 0, 0, "x", 1)):
        try:
            bad()
            raise AssertionError("bad call accepted")
        except (TypeError, OverflowError):
            pass
    print("OFLCALL OK")
    """
)


def test_oflcall_module_against_null_abi(fake_lib, tmp_path):
    """csrc/oflcall.c (the vectorcall path for ofl_h2d / ofl_stream_op):
    tickets and negated statuses round-trip, argument errors raise."""
    import sysconfig

    mod = str(tmp_path / ("_oflcall" + sysconfig.get_config_var("EXT_SUFFIX")))
    subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-I" + sysconfig.get_paths()["include"],
                    "-o", mod, CALL_SRC], check=True)
    script = CALL_SCRIPT.replace("MOD_PATH", repr(mod)).replace("LIB_PATH", repr(fake_lib))
    r = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OFLCALL OK" in r.stdout


BIND_SCRIPT = textwrap.dedent(
    r"""
    import os, sys, tempfile
    sys.path.insert(0, REPO_PATH)
    from paper_1810_11482_b200 import device
    assert device._cpulist("0-3,8,10-11\n") == {0, 1, 2, 3, 8, 10, 11}
    assert device._cpulist("") == set()
    assert device.pci_bus_id(0) == "0000:00:00.0"          # the null ABI's address
    root = tempfile.mkdtemp()
    assert device.local_cpus(0, sysfs=root) is None         # no sysfs entry: unknown
    os.makedirs(os.path.join(root, "0000:00:00.0"))
    allowed = sorted(os.sched_getaffinity(0))
    with open(os.path.join(root, "0000:00:00.0", "local_cpulist"), "w") as f:
        f.write(",".join(map(str, allowed)))
    assert device.local_cpus(0, sysfs=root) == set(allowed)
    # the GPU's CPUs are everything we may use: nothing to bind
    device.local_cpus = lambda o, sysfs=None: set(allowed)
    assert device.bind_host_to_device(0) is None
    if len(allowed) > 1:
        device.local_cpus = lambda o, sysfs=None: {allowed[0]}
        info = device.bind_host_to_device(0)
        assert info == {"pci_bus_id": "0000:00:00.0", "cpus": 1, "of": len(allowed)}, info
        assert os.sched_getaffinity(0) == {allowed[0]}
    device.local_cpus = lambda o, sysfs=None: {10 ** 6}     # none of them allowed
    assert device.bind_host_to_device(0) is None
    print("BIND OK")
    """
)


def test_bind_host_to_device_against_null_abi(fake_lib):
    """NUMA-local host binding (bench.py, one rank per GPU): sysfs cpulist
    parsing, no-op when the GPU's CPUs are all allowed or unknown, every
    thread restricted otherwise."""
    env = dict(os.environ, OFL_LIB=fake_lib)
    r = subprocess.run([sys.executable, "-c", BIND_SCRIPT.replace("REPO_PATH", repr(REPO))],
                       env=env, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "BIND OK" in r.stdout
