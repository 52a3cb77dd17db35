"""Remote localities: the parcel protocol, a daemon serving this runtime's
CUDA devices, and the client proxy ``Runtime.connect`` attaches.

Wire compatibility with the reference (/root/reference/pkg/src/offloadrt/
transport/wire.py:1-20,55-70,159-172): one frame is a 34-byte little-endian
header — magic ``PCL1``, u64 request id, u8 opcode, the target gid as u32
locality + u8 kind + u64 sequence + u32 nonce, u32 payload length — then
the payload.  Replies echo the request id; REPLY_ERR carries a u8 wire code
and a UTF-8 message (errors.py:92-96).  Request payloads per opcode follow
wire.py:159-172.  So a reference client (``offloadrt.Runtime.connect``)
can drive the B200s behind ``serve``, and ``Runtime.connect`` here can drive
a reference daemon (host or sim devices) — location transparency both ways
(reference test_acceptance.py:212-244).

Design (not a translation of the reference's): frames are sent with
``sendmsg`` of header + payload (a 256 MiB read reply is never copied into a
joined frame), received into one preallocated ``bytearray`` per frame
(``recv_into``), and a WRITE's data is handed to the dispatch as a
``memoryview`` of that buffer — the CUDA write stages it straight from
there.  The daemon decodes and enqueues on the connection's receive thread
(arrival order = per-stream device order, as the reference requires) and
replies from token continuations, so requests complete out of order; the
client matches replies by request id.
"""

from __future__ import annotations

import itertools
import socket
import struct
import threading
from enum import IntEnum
from typing import Optional

from .errors import (
    BadArgsError,
    BadMagicError,
    LengthMismatchError,
    TransportLostError,
    TruncatedFrameError,
    UnknownOpcodeError,
    WireFormatError,
    error_from_wire,
    error_to_wire,
)
from .futures import CompletionToken, Promise, make_failed, make_ready, when_all
from .registry import GlobalId, ObjectKind

MAGIC = b"PCL1"
HEADER = struct.Struct("<4sQBIBQII")  # magic, request id, opcode, gid (4 fields), payload length
HEADER_SIZE = HEADER.size  # 34
GID = struct.Struct("<IBQI")
MAX_PAYLOAD = 1 << 31
_U32 = struct.Struct("<I")
_U64 = struct.Struct("<Q")
_F64 = struct.Struct("<d")
_GRID = struct.Struct("<6I")


class Opcode(IntEnum):
    DISCOVER = 1
    CREATE_BUFFER = 2
    WRITE = 3
    READ = 4
    CREATE_PROGRAM = 5
    BUILD = 6
    RUN = 7
    DEVICE_INFO = 8
    UNREGISTER = 9
    REPLY_OK = 128
    REPLY_ERR = 129


_OPCODES = frozenset(int(o) for o in Opcode)
NULL_GID = GlobalId(0, ObjectKind.DEVICE, 0, 0)


def _kind(raw: int):
    return ObjectKind(raw) if raw in (1, 2, 3) else raw


# -- codec --------------------------------------------------------------------------


def encode_gid(gid) -> bytes:
    return GID.pack(gid.locality_id, int(gid.kind), gid.sequence, gid.nonce)


def decode_gid(buf, offset: int = 0) -> GlobalId:
    loc, kind, seq, nonce = GID.unpack_from(buf, offset)
    return GlobalId(loc, _kind(kind), seq, nonce)


def header(opcode: int, request_id: int, gid, payload_len: int) -> bytes:
    if payload_len > MAX_PAYLOAD:
        raise BadArgsError(f"payload of {payload_len} bytes exceeds 2^31")
    return HEADER.pack(MAGIC, request_id, int(opcode), gid.locality_id, int(gid.kind),
                       gid.sequence, gid.nonce, payload_len)


def encode(opcode: int, request_id: int, gid, payload=b"") -> bytes:
    """One whole frame (tests and small messages; the sockets send header
    and payload separately)."""
    return header(opcode, request_id, gid, len(payload)) + bytes(payload)


def decode(buf) -> tuple:
    """(opcode, request_id, gid, payload) of exactly one frame; malformed
    input raises a WireFormatError subclass, never anything else."""
    buf = bytes(buf)
    if buf[:4] != MAGIC:
        if len(buf) < 4 and MAGIC.startswith(buf):
            raise TruncatedFrameError(f"frame of {len(buf)} bytes is shorter than the header")
        raise BadMagicError("frame does not start with PCL1")
    if len(buf) < HEADER_SIZE:
        raise TruncatedFrameError(f"frame of {len(buf)} bytes is shorter than the header")
    _, rid, op, loc, kind, seq, nonce, n = HEADER.unpack_from(buf, 0)
    if op not in _OPCODES:
        raise UnknownOpcodeError(f"opcode {op} is not defined")
    if len(buf) < HEADER_SIZE + n:
        raise TruncatedFrameError(f"payload_len={n} but only {len(buf) - HEADER_SIZE} bytes present")
    if len(buf) > HEADER_SIZE + n:
        raise LengthMismatchError(f"{len(buf) - HEADER_SIZE - n} trailing bytes after frame")
    return Opcode(op), rid, GlobalId(loc, _kind(kind), seq, nonce), buf[HEADER_SIZE:]


def _pack_str(s: str) -> bytes:
    raw = s.encode("utf-8")
    return _U32.pack(len(raw)) + raw


def _unpack_str(buf, off: int) -> tuple:
    (n,) = _U32.unpack_from(buf, off)
    off += 4
    if off + n > len(buf):
        raise BadArgsError("string extends past payload")
    return bytes(buf[off:off + n]).decode("utf-8"), off + n


def pack_device_info(info) -> bytes:
    return (_pack_str(info.name) + _U32.pack(info.capability[0]) + _U32.pack(info.capability[1])
            + _U64.pack(info.memory_bytes) + _U32.pack(info.compute_units))


def unpack_device_info(buf, off: int = 0) -> tuple:
    from .device import DeviceInfo

    name, off = _unpack_str(buf, off)
    major, minor = struct.unpack_from("<II", buf, off)
    (mem,) = _U64.unpack_from(buf, off + 8)
    (units,) = _U32.unpack_from(buf, off + 16)
    return DeviceInfo(name, (major, minor), mem, units), off + 20


def pack_run_args(name: str, grid, block, stream: int, args) -> bytes:
    out = [_pack_str(name), _GRID.pack(*grid, *block), _U32.pack(stream), _U32.pack(len(args))]
    for tag, value in args:
        if tag == "buffer":
            out.append(b"\x00" + encode_gid(value))
        elif tag == "f64":
            out.append(b"\x01" + _F64.pack(value))
        elif tag == "u32":
            out.append(b"\x02" + _U32.pack(value))
        else:
            raise BadArgsError(f"unknown kernel argument tag {tag!r}")
    return b"".join(out)


def unpack_run_args(buf) -> tuple:
    name, off = _unpack_str(buf, 0)
    g = _GRID.unpack_from(buf, off)
    off += 24
    stream, count = struct.unpack_from("<II", buf, off)
    off += 8
    args = []
    for _ in range(count):
        tag = buf[off]
        off += 1
        if tag == 0:
            args.append(("buffer", decode_gid(buf, off)))
            off += GID.size
        elif tag == 1:
            args.append(("f64", _F64.unpack_from(buf, off)[0]))
            off += 8
        elif tag == 2:
            args.append(("u32", _U32.unpack_from(buf, off)[0]))
            off += 4
        else:
            raise BadArgsError(f"unknown kernel argument tag {tag}")
    return name, g[:3], g[3:], stream, args


def pack_discover_reply(locality_id: int, devices) -> bytes:
    out = [_U32.pack(locality_id), _U32.pack(len(devices))]
    for gid, info in devices:
        out.append(encode_gid(gid))
        out.append(pack_device_info(info))
    return b"".join(out)


def unpack_discover_reply(buf) -> tuple:
    loc, count = struct.unpack_from("<II", buf, 0)
    off, devices = 8, []
    for _ in range(count):
        gid = decode_gid(buf, off)
        info, off = unpack_device_info(buf, off + GID.size)
        devices.append((gid, info))
    return loc, devices


# -- sockets ------------------------------------------------------------------------


def _recv_into(sock: socket.socket, view: memoryview) -> None:
    while view:
        got = sock.recv_into(view)
        if not got:
            raise ConnectionError("connection closed")
        view = view[got:]


def read_frame(sock: socket.socket) -> tuple:
    """(opcode, request_id, gid, payload: bytearray) of the next frame."""
    head = bytearray(HEADER_SIZE)
    _recv_into(sock, memoryview(head))
    magic, rid, op, loc, kind, seq, nonce, n = HEADER.unpack(head)
    if magic != MAGIC:
        raise BadMagicError("frame does not start with PCL1")
    if op not in _OPCODES:
        raise UnknownOpcodeError(f"opcode {op} is not defined")
    payload = bytearray(n)
    if n:
        _recv_into(sock, memoryview(payload))
    return Opcode(op), rid, GlobalId(loc, _kind(kind), seq, nonce), payload


def send_frame(sock: socket.socket, lock: threading.Lock, opcode: int, request_id: int, gid,
               payload=b"", tail=None) -> None:
    """One frame: header, payload and an optional `tail` buffer appended to
    the payload without joining them (a WRITE's data is sent in place)."""
    tail_n = memoryview(tail).nbytes if tail is not None else 0
    head = header(opcode, request_id, gid, len(payload) + tail_n)
    with lock:
        if len(payload) + tail_n < (64 << 10):
            sock.sendall(head + bytes(payload) + (bytes(tail) if tail_n else b""))
            return
        parts = [memoryview(head), memoryview(payload).cast("B")]
        if tail_n:
            parts.append(memoryview(tail).cast("B"))
        while parts:  # sendmsg may send part of the gathered buffers
            sent = sock.sendmsg(parts)
            while sent and parts:
                if sent >= len(parts[0]):
                    sent -= len(parts[0])
                    parts.pop(0)
                else:
                    parts[0] = parts[0][sent:]
                    sent = 0


# -- daemon -------------------------------------------------------------------------


class _Connection:
    def __init__(self, daemon: "Daemon", sock: socket.socket):
        self.daemon = daemon
        self.sock = sock
        self.lock = threading.Lock()
        self.thread = threading.Thread(target=self._serve, name="ofl-parcel-conn", daemon=True)
        self.thread.start()

    def _serve(self) -> None:
        try:
            while True:
                op, rid, gid, payload = read_frame(self.sock)
                try:
                    token = self._execute(op, gid, payload)
                except Exception as exc:  # noqa: BLE001 - a request failure is a REPLY_ERR
                    self._reply_err(rid, gid, exc)
                    continue
                token._on_done(lambda t, rid=rid, gid=gid: self._finish(rid, gid, t))
        except (OSError, ConnectionError, WireFormatError):
            pass  # peer gone or unparseable stream: drop this connection only
        finally:
            try:
                self.sock.close()
            except OSError:
                pass
            self.daemon._forget(self)

    def _execute(self, op: int, gid, body: bytearray) -> CompletionToken:
        rt = self.daemon.runtime
        local = rt.local
        if op == Opcode.DISCOVER:
            major, minor = struct.unpack_from("<II", body, 0)
            devs = [(g, i) for g, i in rt.local_device_table() if i.meets(major, minor)]
            return make_ready(pack_discover_reply(rt.registry.self_locality_id, devs))
        if op == Opcode.DEVICE_INFO:
            return local.device_info(gid).then(pack_device_info)
        if op == Opcode.CREATE_BUFFER:
            return local.create_buffer(gid, _U64.unpack_from(body, 0)[0]).then(encode_gid)
        if op == Opcode.WRITE:
            (offset,) = _U64.unpack_from(body, 0)
            (stream,) = _U32.unpack_from(body, 8)
            # the write stages straight from the receive buffer (it may be
            # reused once the call returns, as for any pageable write)
            return local.write(gid, offset, memoryview(body)[12:], stream).then(lambda _: b"")
        if op == Opcode.READ:
            offset, size = struct.unpack_from("<QQ", body, 0)
            (stream,) = _U32.unpack_from(body, 16)
            return local.read(gid, offset, size, stream)
        if op == Opcode.CREATE_PROGRAM:
            return local.create_program(gid, bytes(body).decode("utf-8")).then(encode_gid)
        if op == Opcode.BUILD:
            return local.build(gid, bytes(body).decode("utf-8")).then(lambda _: b"")
        if op == Opcode.RUN:
            name, grid, block, stream, args = unpack_run_args(body)
            return local.run(gid, name, grid, block, stream, args).then(lambda _: b"")
        if op == Opcode.UNREGISTER:
            return local.unregister(gid).then(lambda _: b"")
        raise UnknownOpcodeError(f"request opcode {int(op)} not servable")

    def _finish(self, rid: int, gid, token: CompletionToken) -> None:
        err = token.error()
        if err is not None:
            self._reply_err(rid, gid, err)
            return
        try:
            send_frame(self.sock, self.lock, Opcode.REPLY_OK, rid, gid, token._value or b"")
        except OSError:
            pass  # peer gone; the receive loop notices

    def _reply_err(self, rid: int, gid, exc: BaseException) -> None:
        code, message = error_to_wire(exc)
        try:
            send_frame(self.sock, self.lock, Opcode.REPLY_ERR, rid, gid,
                       bytes([code]) + message.encode("utf-8"))
        except OSError:
            pass

    def close(self) -> None:
        try:
            self.sock.shutdown(socket.SHUT_RDWR)
        except OSError:
            pass


class Daemon:
    """Accepts parcel connections and serves them against a Runtime (its
    ``local`` dispatch, device table and locality id)."""

    def __init__(self, runtime, host: str = "127.0.0.1", port: int = 0):
        self.runtime = runtime
        self._listener = socket.create_server((host, port))
        self.address = "%s:%d" % self._listener.getsockname()[:2]
        self.port = self._listener.getsockname()[1]
        self._lock = threading.Lock()
        self._conns: set = set()
        self._stopped = False
        self._thread = threading.Thread(target=self._accept, name="ofl-parcel-accept", daemon=True)
        self._thread.start()

    def _accept(self) -> None:
        while True:
            try:
                sock, _ = self._listener.accept()
            except OSError:
                return
            sock.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
            with self._lock:
                if self._stopped:
                    sock.close()
                    return
                self._conns.add(_Connection(self, sock))

    def _forget(self, conn) -> None:
        with self._lock:
            self._conns.discard(conn)

    def stop(self) -> None:
        with self._lock:
            self._stopped = True
            conns = list(self._conns)
        self._listener.close()
        for c in conns:
            c.close()

    def __enter__(self) -> "Daemon":
        return self

    def __exit__(self, *exc) -> None:
        self.stop()


def serve(address: str, runtime) -> Daemon:
    """Bind ``host:port`` (port 0 picks one) and serve ``runtime``."""
    host, _, port = address.rpartition(":")
    return Daemon(runtime, host or "127.0.0.1", int(port))


# -- client -------------------------------------------------------------------------


class RemoteLocality:
    """Dispatch proxy for one connected daemon: the dispatch surface of
    CudaDispatch / the reference's LocalDispatch over one pipelined TCP
    connection.  Requests go out in call order (per-stream device order
    rides on it); a lost connection fails every pending token with
    TransportLostError."""

    def __init__(self, sock: socket.socket, address: str):
        self._sock = sock
        self.address = address
        self.locality_id = 0
        self.devices: list = []
        self._send_lock = threading.Lock()
        self._pending_lock = threading.Lock()
        self._pending: dict = {}
        self._ids = itertools.count(1)
        self._dead: Optional[BaseException] = None
        # client-side stream bookkeeping (fresh ids per device; the last
        # token per (device, stream) for synchronize)
        self._stream_ids: dict = {}
        self._last: dict = {}
        self._track_lock = threading.Lock()
        self._reader = threading.Thread(target=self._read_loop, name="ofl-parcel-reader",
                                        daemon=True)
        self._reader.start()

    def _request(self, op: int, gid, payload=b"", tail=None) -> CompletionToken:
        promise = Promise()
        if self._dead is not None:
            return make_failed(TransportLostError(f"connection to {self.address} lost"))
        rid = next(self._ids)
        with self._pending_lock:
            self._pending[rid] = promise
        try:
            send_frame(self._sock, self._send_lock, op, rid, gid, payload, tail)
        except OSError as exc:
            self._fail_all(exc)
        if self._dead is not None:  # the reader may have drained _pending first
            with self._pending_lock:
                self._pending.pop(rid, None)
            promise.try_set_error(TransportLostError(f"connection to {self.address} lost"))
        return promise.token

    def _read_loop(self) -> None:
        try:
            while True:
                op, rid, _, payload = read_frame(self._sock)
                with self._pending_lock:
                    promise = self._pending.pop(rid, None)
                if promise is None:
                    continue
                if op == Opcode.REPLY_ERR:
                    code = payload[0] if payload else 5
                    msg = bytes(payload[1:]).decode("utf-8", "replace") if payload else "empty error"
                    promise.try_set_error(error_from_wire(code, msg))
                else:
                    promise.try_set_value(bytes(payload))
        except (OSError, ConnectionError, WireFormatError) as exc:
            self._fail_all(exc)

    def _fail_all(self, cause: BaseException) -> None:
        with self._pending_lock:
            self._dead = cause
            pending, self._pending = self._pending, {}
        for p in pending.values():
            p.try_set_error(TransportLostError(f"connection to {self.address} lost"))

    def close(self) -> None:
        try:
            self._sock.shutdown(socket.SHUT_RDWR)
        except OSError:
            pass
        self._sock.close()

    def _track(self, device, stream: int, token: CompletionToken) -> CompletionToken:
        if device is not None:
            with self._track_lock:
                self._last[(device, stream)] = token
        return token

    # -- dispatch surface ---------------------------------------------------------
    def discover(self, major: int = 0, minor: int = 0) -> CompletionToken:
        return self._request(Opcode.DISCOVER, NULL_GID, struct.pack("<II", major, minor)).then(
            unpack_discover_reply)

    def device_info(self, device_gid) -> CompletionToken:
        return self._request(Opcode.DEVICE_INFO, device_gid).then(
            lambda p: unpack_device_info(p, 0)[0])

    def create_stream(self, device_gid) -> int:
        with self._track_lock:
            ids = self._stream_ids.setdefault(device_gid, itertools.count(1))
        return next(ids)

    def synchronize(self, device_gid) -> CompletionToken:
        with self._track_lock:
            toks = [t for (d, _), t in self._last.items() if d == device_gid]
        return when_all(toks)

    def create_buffer(self, device_gid, size: int, shareable: bool = False) -> CompletionToken:
        if shareable:
            return make_failed(BadArgsError("shareable buffers are local to a process"))
        return self._request(Opcode.CREATE_BUFFER, device_gid, _U64.pack(size)).then(decode_gid)

    def write(self, buffer_gid, offset, data, stream, device=None) -> CompletionToken:
        # the data goes out in place (sendmsg); the request is fully sent when
        # this returns, so the caller may reuse it, as with any write
        body = data if isinstance(data, bytes) else memoryview(data).cast("B")
        prefix = _U64.pack(offset) + _U32.pack(stream)
        return self._track(device, stream, self._request(Opcode.WRITE, buffer_gid, prefix,
                                                         body).then(lambda _: None))

    def read(self, buffer_gid, offset, size, stream, device=None) -> CompletionToken:
        payload = struct.pack("<QQI", offset, size, stream)
        return self._track(device, stream, self._request(Opcode.READ, buffer_gid, payload))

    def read_into(self, buffer_gid, offset, out, stream, device=None) -> CompletionToken:
        n = memoryview(out).nbytes

        def land(data: bytes):
            memoryview(out).cast("B")[:n] = data
            return out

        return self.read(buffer_gid, offset, n, stream, device).then(land)

    def read_rows_into(self, *args, **kwargs) -> CompletionToken:
        return make_failed(BadArgsError("enqueue_read_rows_into is local to this process"))

    def copy(self, src_gid, src_off, dst_gid, dst_off, size) -> CompletionToken:
        return make_failed(BadArgsError("copy across localities goes through the host"))

    def create_program(self, device_gid, source: str) -> CompletionToken:
        return self._request(Opcode.CREATE_PROGRAM, device_gid, source.encode("utf-8")).then(
            decode_gid)

    def build(self, program_gid, kernel_name: str) -> CompletionToken:
        return self._request(Opcode.BUILD, program_gid, kernel_name.encode("utf-8")).then(
            lambda _: None)

    def run(self, program_gid, kernel_name, grid, block, stream, args, device=None,
            items=None) -> CompletionToken:
        payload = pack_run_args(kernel_name, tuple(grid), tuple(block), stream, args)
        return self._track(device, stream,
                           self._request(Opcode.RUN, program_gid, payload).then(lambda _: None))

    def unregister(self, gid) -> CompletionToken:
        return self._request(Opcode.UNREGISTER, gid).then(lambda _: None)


def connect(address: str, timeout: float = 10.0) -> RemoteLocality:
    """Open a connection and discover the daemon's locality id and devices."""
    host, _, port = address.rpartition(":")
    sock = socket.create_connection((host or "127.0.0.1", int(port)), timeout=timeout)
    sock.settimeout(None)
    sock.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)
    proxy = RemoteLocality(sock, address)
    try:
        proxy.locality_id, proxy.devices = proxy.discover(0, 0).get(timeout)
    except BaseException:
        proxy.close()
        raise
    return proxy
