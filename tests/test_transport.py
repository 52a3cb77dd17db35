"""Remote localities (transport.py): the parcel protocol, the daemon serving
this runtime's devices, and Runtime.connect — against this package on both
ends and against the reference on either end (reference test_acceptance.py:
212-244 location transparency, test_wire.py round trips and decoder fuzz).

CPU: the local CUDA runtimes use the null test double of libofl.so
(tests/fakes/null_ofl.c), so these check the plumbing; the reference daemon
(host backend) computes for real, so our client driving it checks results.
GPU: the daemon serves the B200 and the four benchmarks must be
byte-identical locally and over loopback."""

from __future__ import annotations

import os
import random
import subprocess
import sys
import textwrap

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC_CANDIDATES = ("/root/reference/pkg/src", os.path.join(REPO, "baseline", "_ref"))


def _ref_src():
    for p in REF_SRC_CANDIDATES:
        if os.path.isfile(os.path.join(p, "offloadrt", "__init__.py")):
            return p
    return None


def test_codec_round_trip_and_fuzz():
    from paper_1810_11482_b200 import transport as T
    from paper_1810_11482_b200.errors import WireFormatError
    from paper_1810_11482_b200.registry import GlobalId, ObjectKind

    rng = random.Random(1810)
    for _ in range(2000):
        gid = GlobalId(rng.getrandbits(32), ObjectKind(rng.randint(1, 3)), rng.getrandbits(64),
                       rng.getrandbits(32))
        op = rng.choice(list(T.Opcode))
        payload = bytes(rng.getrandbits(8) for _ in range(rng.randint(0, 64)))
        rid = rng.getrandbits(64)
        frame = T.encode(op, rid, gid, payload)
        assert len(frame) == T.HEADER_SIZE + len(payload)
        assert T.decode(frame) == (op, rid, gid, payload)
    for _ in range(5000):  # the decoder is total: only WireFormatError
        blob = bytes(rng.getrandbits(8) for _ in range(rng.randint(0, 80)))
        if rng.random() < 0.5:
            blob = b"PCL1" + blob
        try:
            T.decode(blob)
        except WireFormatError:
            pass
    args = [("buffer", GlobalId(7, ObjectKind.BUFFER, 3, 9)), ("f64", -2.5), ("u32", 2**32 - 1)]
    packed = T.pack_run_args("k", (1, 2, 3), (4, 5, 6), 7, args)
    assert T.unpack_run_args(packed) == ("k", (1, 2, 3), (4, 5, 6), 7, args)


def test_codec_matches_reference_bytes():
    ref = _ref_src()
    if ref is None:
        pytest.skip("reference not importable here")
    script = textwrap.dedent(r"""
        import random, sys
        sys.path[:0] = [__REF__, __REPO__]
        from offloadrt.transport import wire as W
        from offloadrt.registry import GlobalId as RG, ObjectKind as RK
        from offloadrt.device import DeviceInfo as RI
        from paper_1810_11482_b200 import transport as T
        from paper_1810_11482_b200.registry import GlobalId, ObjectKind
        from paper_1810_11482_b200.device import DeviceInfo
        rng = random.Random(7)
        for _ in range(500):
            f = (rng.getrandbits(32), rng.randint(1, 3), rng.getrandbits(64), rng.getrandbits(32))
            op = rng.choice([1, 2, 3, 4, 5, 6, 7, 8, 9, 128, 129]); rid = rng.getrandbits(64)
            pl = bytes(rng.getrandbits(8) for _ in range(rng.randint(0, 40)))
            a = W.encode(W.Parcel(W.Opcode(op), rid, RG(f[0], RK(f[1]), f[2], f[3]), pl))
            b = T.encode(op, rid, GlobalId(f[0], ObjectKind(f[1]), f[2], f[3]), pl)
            assert a == b
        args_r = [("buffer", RG(3, RK(2), 5, 6)), ("f64", 0.1), ("u32", 77)]
        args_o = [("buffer", GlobalId(3, ObjectKind(2), 5, 6)), ("f64", 0.1), ("u32", 77)]
        assert W.pack_run_args("sum", (1,1,1), (32,1,1), 2, args_r) == T.pack_run_args("sum", (1,1,1), (32,1,1), 2, args_o)
        di = RI("cuda0", (10, 0), 1 << 37, 148)
        assert W.pack_device_info(di) == T.pack_device_info(DeviceInfo("cuda0", (10, 0), 1 << 37, 148))
        print("CODEC OK")
    """).replace("__REF__", repr(ref)).replace("__REPO__", repr(REPO))
    r = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, timeout=120,
                       env=dict(os.environ, PYTHONDONTWRITEBYTECODE="1"))
    assert r.returncode == 0 and "CODEC OK" in r.stdout, r.stdout + r.stderr


OURS_BOTH_ENDS = textwrap.dedent(r"""
    import sys, threading
    sys.path.insert(0, __REPO__)
    import numpy as np
    from paper_1810_11482_b200 import (Runtime, when_all, copy, OobAccessError, BadArgsError,
        NotBuiltError, UnknownGidError, CompileError, TransportLostError)
    from paper_1810_11482_b200.bindings import kernel_source
    from paper_1810_11482_b200.transport import serve

    def raises(exc, fn):
        try:
            fn()
        except exc as e:
            return e
        raise AssertionError(f"{exc.__name__} not raised")

    served = Runtime(devices=[0], locality_id=9)
    daemon = serve("127.0.0.1:0", served)
    client = Runtime(devices=[0])
    info = client.connect(daemon.address)
    assert info.locality_id == 9
    raises(ValueError, lambda: client.connect(daemon.address))   # locality already known
    devs = client.get_all_devices().get()
    assert [d.gid.locality_id for d in devs] == [0, 9]
    local, remote = devs
    assert remote.device_info().get(timeout=30).capability == (10, 0)
    b = remote.create_buffer(1 << 20).get(timeout=30)
    assert b.gid.locality_id == 9
    data = np.random.default_rng(1).integers(0, 256, 1 << 20, dtype=np.uint8)
    b.enqueue_write(0, data)
    assert b.enqueue_read(0, 1 << 20).get(timeout=30) == data.tobytes()
    out = bytearray(64)
    assert b.enqueue_read_into(64, out).get(timeout=30) is out and bytes(out) == data[64:128].tobytes()
    raises(OobAccessError, lambda: b.enqueue_write((1 << 20) - 2, b"xyz"))
    s1 = remote.create_stream()
    toks = [b.enqueue_write(i * 8, bytes([i]) * 8, s1) for i in range(100)]
    assert when_all(toks).get(timeout=30) is None
    assert remote.synchronize().get(timeout=30) is None
    # programs: errors come back through REPLY_ERR with their types
    p = remote.create_program_with_source(kernel_source("sum")).get(timeout=30)
    raises(BadArgsError, lambda: p.run([b, b, 1], "sum", (1, 1, 1), (1, 1, 1)).get(timeout=30))  # NotBuilt flattens to BAD_ARGS on the wire
    p.build("sum").get(timeout=30)
    raises(OobAccessError, lambda: p.run([b, b, (1 << 18) + 1], "sum", (1, 1, 1), (32, 1, 1)).get(timeout=30))
    p.run([b, b, 16], "sum", (1, 1, 1), (32, 1, 1)).get(timeout=30)
    q = remote.create_program_with_source("kernel k(x : buffer_f64) { x[0] = nope; }").get(timeout=30)
    e = raises(CompileError, lambda: q.build("k").get(timeout=30))
    assert "1:" in str(e)
    raises(BadArgsError, lambda: p.run([b, 3.5, b], "sum", (1, 1, 1), (1, 1, 1)).get(timeout=30))
    # copy across localities goes through the host
    lb = local.create_buffer(256).get()
    copy(b, 0, lb, 0, 256).get(timeout=30)
    assert lb.enqueue_read(0, 256).get() == b.enqueue_read(0, 256).get(timeout=30)
    copy(lb, 8, b, 1000, 16).get(timeout=30)
    assert b.enqueue_read(1000, 16).get(timeout=30) == lb.enqueue_read(8, 16).get()
    # a continuation on a remote token
    fired = threading.Event()
    b.enqueue_read(0, 8).then(lambda _: fired.set())
    assert fired.wait(30)
    # unregister, then use: UnknownGidError over the wire
    client.dispatch(b.gid).unregister(b.gid).get(timeout=30)
    raises(UnknownGidError, lambda: b.enqueue_read(0, 1).get(timeout=30))
    # connection loss fails pending and later requests with TransportLostError
    daemon.stop()
    served.close()
    import time
    time.sleep(0.2)
    raises(TransportLostError, lambda: remote.create_buffer(64).get(timeout=30))
    client.close()
    print("TRANSPORT OK", flush=True)
""")


def _fake_env():
    from test_host_logic_cpu import FAKE_LIB, FAKE_SRC

    os.makedirs(os.path.dirname(FAKE_LIB), exist_ok=True)
    subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-o", FAKE_LIB, FAKE_SRC], check=True)
    return dict(os.environ, OFL_LIB=FAKE_LIB, PYTHONDONTWRITEBYTECODE="1")


def test_our_client_and_daemon_null_abi():
    r = subprocess.run([sys.executable, "-c", OURS_BOTH_ENDS.replace("__REPO__", repr(REPO))],
                       env=_fake_env(), capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "TRANSPORT OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


REF_CLIENT = textwrap.dedent(r"""
    import sys
    sys.path[:0] = [__REF__, __REPO__]
    import numpy as np
    from offloadrt import Runtime as RefRuntime, when_all
    from offloadrt.errors import OobAccessError, NotBuiltError, UnknownGidError
    from offloadrt.bench import kernel_source
    from paper_1810_11482_b200 import Runtime
    from paper_1810_11482_b200.transport import serve

    def raises(exc, fn):
        try:
            fn()
        except exc as e:
            return e
        raise AssertionError(f"{exc.__name__} not raised")

    served = Runtime(devices=[0], locality_id=21)
    daemon = serve("127.0.0.1:0", served)
    with RefRuntime(backend="host") as client:
        client.connect(daemon.address)
        devs = client.get_all_devices().get()
        remote = [d for d in devs if d.gid.locality_id == 21][0]
        assert type(remote).__module__ == "offloadrt.handles"
        b = remote.create_buffer(4096).get(timeout=30)
        payload = bytes(range(256)) * 16
        b.enqueue_write(0, payload)
        assert b.enqueue_read(0, 4096).get(timeout=30) == payload
        raises(OobAccessError, lambda: b.enqueue_write(4090, b"12345678"))
        p = remote.create_program_with_source(kernel_source("sum")).get(timeout=30)
        raises(Exception, lambda: p.run([b, b, 1], "sum", (1, 1, 1), (1, 1, 1)).get(timeout=30))
        p.build("sum").get(timeout=30)
        raises(OobAccessError, lambda: p.run([b, b, 1025], "sum", (1, 1, 1), (32, 1, 1)).get(timeout=30))
        assert when_all([b.enqueue_write(0, b"x" * 8), p.run([b, b, 8], "sum", (1, 1, 1), (32, 1, 1))]).get(timeout=30) is None
        client.dispatch(b.gid).unregister(b.gid).get(timeout=30)
        raises(UnknownGidError, lambda: b.enqueue_read(0, 1).get(timeout=30))
    daemon.stop()
    served.close()
    print("REF CLIENT OK", flush=True)
""")


def test_reference_client_against_our_daemon_null_abi():
    ref = _ref_src()
    if ref is None:
        pytest.skip("reference not importable here")
    r = subprocess.run([sys.executable, "-c",
                        REF_CLIENT.replace("__REF__", repr(ref)).replace("__REPO__", repr(REPO))],
                       env=_fake_env(), capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "REF CLIENT OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


OUR_CLIENT_REF_DAEMON = textwrap.dedent(r"""
    import sys
    sys.path[:0] = [__REF__, __REPO__, __TESTS__]
    import numpy as np
    import oracle
    from offloadrt import Runtime as RefRuntime
    from offloadrt.transport.daemon import serve as ref_serve
    from paper_1810_11482_b200 import Runtime
    import flows

    daemon_rt = RefRuntime(backend="host", devices=1, locality_id=11)
    daemon = ref_serve("127.0.0.1:0", daemon_rt)
    with Runtime(devices=[0]) as client:
        client.connect(daemon.address)
        remote = [d for d in client.get_all_devices().get() if d.gid.locality_id == 11][0]
        assert remote.info.name.startswith("host")
        rng = np.random.default_rng(77)
        x = rng.random(4096)
        assert flows.device_stencil(remote, x) == oracle.stencil(x).tobytes()
        v = rng.integers(0, 2**32, 4096, dtype=np.uint32)
        ib = remote.create_buffer(v.nbytes).get(timeout=60)
        rb = remote.create_buffer(4).get(timeout=60)
        from paper_1810_11482_b200.bindings import kernel_source
        sp = remote.create_program_with_source(kernel_source("sum")).get(timeout=60)
        sp.build("sum").get(timeout=120)
        ib.enqueue_write(0, v.tobytes())
        sp.run([ib, rb, v.size], "sum", (1, 1, 1), (32, 1, 1))
        assert int(np.frombuffer(rb.enqueue_read(0, 4).get(timeout=60), np.uint32)[0]) == oracle.sum_u32(v)
        raw = flows.device_mandelbrot(remote, 48, 32, 256)
        assert raw == oracle.mandelbrot(48, 32, max_iter=256).tobytes()
    daemon.stop()
    daemon_rt.close()
    print("OUR CLIENT OK", flush=True)
""")


def test_our_client_against_reference_daemon():
    """Runtime.connect to the reference's own daemon (host backend): our
    handles drive its devices, which compute for real — outputs equal the
    oracle's."""
    ref = _ref_src()
    if ref is None:
        pytest.skip("reference not importable here")
    script = (OUR_CLIENT_REF_DAEMON.replace("__REF__", repr(ref)).replace("__REPO__", repr(REPO))
              .replace("__TESTS__", repr(os.path.join(REPO, "tests"))))
    r = subprocess.run([sys.executable, "-c", script], env=_fake_env(), capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "OUR CLIENT OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.gpu
def test_location_transparency_b200(golden):
    """test_acceptance.py:212-244 on the B200: the four benchmarks through a
    local device and through the daemon over loopback are byte-identical
    (and match the reference's golden outputs)."""
    import hashlib
    import math

    import numpy as np

    import flows
    import oracle
    from paper_1810_11482_b200 import Runtime
    from paper_1810_11482_b200.bench.harness import (PartitionConfig, enqueue_partition_round,
                                                     prepare_partitions)
    from paper_1810_11482_b200.bindings import kernel_source
    from paper_1810_11482_b200.transport import serve

    served = Runtime(devices=[0], locality_id=21)
    daemon = serve("127.0.0.1:0", served)
    try:
        with Runtime(devices=[0]) as client:
            client.connect(daemon.address)
            devices = client.get_all_devices().get()
            local = devices[0]
            remote = [d for d in devices if d.gid.locality_id == 21][0]
            rng = np.random.default_rng(77)
            x = rng.random(1 << 20)
            assert flows.device_stencil(local, x) == flows.device_stencil(remote, x) \
                == oracle.stencil(x).tobytes()

            def dsum(dev, v):
                ib, rb = dev.create_buffer(v.nbytes).get(), dev.create_buffer(4).get()
                sp = dev.create_program_with_source(kernel_source("sum")).get()
                sp.build("sum").get(timeout=120)
                ib.enqueue_write(0, v.tobytes())
                sp.run([ib, rb, v.size], "sum", (1, 1, 1), (32, 1, 1))
                return int(np.frombuffer(rb.enqueue_read(0, 4).get(timeout=60), np.uint32)[0])

            v = rng.integers(0, 2**32, size=1 << 20, dtype=np.uint32)
            assert dsum(local, v) == dsum(remote, v) == oracle.sum_u32(v)
            case = golden["mandelbrot"][6]  # 960x540 @2000 from the reference
            w, h = case["width"], case["height"]
            outs = []
            for dev in (local, remote):
                ob = dev.create_buffer(w * h * 4).get()
                mp = dev.create_program_with_source(kernel_source("mandelbrot")).get()
                mp.build("mandelbrot").get(timeout=120)
                mp.run([ob, w, h, *case["viewport"], case["esc"], case["max_iter"]],
                       "mandelbrot", (math.ceil(w * h / 256), 1, 1), (256, 1, 1))
                outs.append(ob.enqueue_read(0, w * h * 4).get(timeout=60))
            assert outs[0] == outs[1]
            assert hashlib.sha256(outs[0]).hexdigest() == case["sha256"]
            got = {}
            for tag, dev in (("local", local), ("remote", remote)):
                _, parts = prepare_partitions(PartitionConfig(m=1, partitions=2), [dev])
                got[tag] = b"".join(t.get(timeout=120) for t in enqueue_partition_round(parts))
            assert got["local"] == got["remote"]
    finally:
        daemon.stop()
        served.close()
