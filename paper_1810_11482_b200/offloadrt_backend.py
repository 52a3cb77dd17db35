"""Plug the CUDA dispatch into an unmodified ``offloadrt.Runtime``.

The reference routes every handle operation through
``Runtime.dispatch(gid)`` (/root/reference/pkg/src/offloadrt/runtime.py:
178-184): gids of its own locality go to ``LocalDispatch``, any other
locality id to the proxy registered in ``Runtime._connections`` — the same
slot a remote daemon's ``RemoteLocality`` occupies after ``Runtime.connect``
(runtime.py:204-216, transport/client.py:134-195).  ``attach`` registers a
:class:`CudaLocality` there under a locality id of its own, so the CUDA
devices join the reference's ``get_all_devices()`` (after its local
devices, ordered by locality id) and the reference's handles, ``when_all``
and ``copy`` drive them unchanged.

The locality id must differ from the reference runtime's own
(``registry.self_locality_id``, 0 by default) and from every connected
daemon's: ``Runtime.dispatch`` sends gids of its own locality to
``LocalDispatch``, which would reject the CUDA gids with UnknownGidError.
``attach`` picks the smallest free id above all known ones unless told.

Usage (the whole reference-side change)::

    from offloadrt import Runtime, when_all
    from paper_1810_11482_b200.offloadrt_backend import attach

    rt = Runtime(backend="host")          # the reference runtime, unmodified
    cuda = attach(rt)                      # B200s as locality 1
    dev = rt.get_all_devices().get()[-1]   # a reference DeviceHandle on cuda0
    ...
    rt.close()                             # closes the CUDA locality too
"""

from __future__ import annotations

from typing import Optional, Sequence

from . import errors as _ours
from .futures import _FAILED, _PENDING, CompletionToken
from .runtime import Runtime as _CudaRuntime


def _ref_error(exc: BaseException) -> BaseException:
    """The reference's exception of the same name (errors.py:12-87 of the
    reference; identical taxonomy), so ``except offloadrt.errors.X`` keeps
    working for errors raised by the CUDA locality — what a RemoteLocality
    does when it decodes a wire error (transport/client.py)."""
    if not isinstance(exc, _ours.OffloadError):
        return exc
    import offloadrt.errors as ref

    cls = getattr(ref, type(exc).__name__, None)
    if cls is None or not issubclass(cls, ref.OffloadError):
        cls = ref.InternalError
    if isinstance(exc, _ours.CompileError):
        out = cls(exc.message, exc.line, exc.col) if cls is ref.CompileError else cls(str(exc))
    else:
        out = cls(*exc.args)
    out.__cause__ = exc
    return out


class _Mapped(CompletionToken):
    """A token mirroring an inner token of this package with errors mapped
    to the reference's classes.  Completion stays lazy: polling, blocking
    and arming go straight to the inner token (a device token keeps its
    direct CUDA-event wait; nothing is armed unless someone registers a
    continuation)."""

    __slots__ = ("_inner",)

    def __init__(self, inner: CompletionToken):
        super().__init__()
        self._inner = inner

    def _adopt(self, inner=None) -> None:
        t = self._inner
        if t._state == _FAILED:
            self._try_complete(error=_ref_error(t._error))
        else:
            self._try_complete(value=t._value)

    def _poll(self) -> bool:
        if self._state != _PENDING:
            return True
        if self._inner.done():
            self._adopt()
        return self._state != _PENDING

    def _block(self, timeout) -> bool:
        if self._state != _PENDING:
            return True
        if self._inner._state == _PENDING and not self._inner._block(timeout):
            return False
        self._adopt()
        return True

    def _arm(self) -> None:
        self._inner._on_done(self._adopt)


def _mapped(tok: CompletionToken) -> CompletionToken:
    if tok._state != _PENDING:
        if tok._state == _FAILED:
            from .futures import make_failed

            return make_failed(_ref_error(tok._error))
        return tok
    return _Mapped(tok)


class CudaLocality:
    """The dispatch surface of ``LocalDispatch`` (runtime.py:30-120 of the
    reference) served by this package's ``CudaDispatch``, plus the proxy
    attributes the reference's Runtime reads from a connection
    (``locality_id``, ``devices``, ``close``)."""

    def __init__(self, devices: Optional[Sequence[int]] = None, locality_id: int = 1,
                 record_events: bool = False):
        self.locality_id = locality_id
        self.runtime = _CudaRuntime(backend="cuda", devices=devices, locality_id=locality_id,
                                    record_events=record_events)
        self._d = self.runtime.local
        # (gid, DeviceInfo) pairs, the shape of RemoteLocality.devices
        self.devices = list(self.runtime.local_device_table())

    # -- the dispatch surface (reference runtime.py:46-120) ---------------------
    # Every result token is wrapped so that failures carry the reference's
    # exception classes; synchronous raises are mapped the same way.
    def device_info(self, device_gid):
        return _mapped(self._d.device_info(device_gid))

    def create_stream(self, device_gid) -> int:
        try:
            return self._d.create_stream(device_gid)
        except Exception as exc:  # noqa: BLE001
            raise _ref_error(exc) from exc

    def synchronize(self, device_gid):
        return _mapped(self._d.synchronize(device_gid))

    def create_buffer(self, device_gid, size: int):
        return _mapped(self._d.create_buffer(device_gid, size))

    def write(self, buffer_gid, offset, data, stream, device=None):
        return _mapped(self._d.write(buffer_gid, offset, data, stream, device=device))

    def read(self, buffer_gid, offset, size, stream, device=None):
        return _mapped(self._d.read(buffer_gid, offset, size, stream, device=device))

    def create_program(self, device_gid, source: str):
        return _mapped(self._d.create_program(device_gid, source))

    def build(self, program_gid, kernel_name: str):
        return _mapped(self._d.build(program_gid, kernel_name))

    def run(self, program_gid, kernel_name, grid, block, stream, args, device=None):
        return _mapped(self._d.run(program_gid, kernel_name, tuple(grid), tuple(block), stream,
                                   list(args), device=device))

    def unregister(self, gid):
        return _mapped(self._d.unregister(gid))

    # -- proxy lifetime ----------------------------------------------------------
    def close(self) -> None:
        self.runtime.close()


def _known_localities(ref_runtime) -> set:
    ids = {ref_runtime.registry.self_locality_id}
    ids.update(getattr(ref_runtime, "_connections", {}).keys())
    ids.update(getattr(ref_runtime, "_remote_devices", {}).keys())
    return ids


def attach(ref_runtime, devices: Optional[Sequence[int]] = None,
           locality_id: Optional[int] = None, record_events: bool = False) -> CudaLocality:
    """Register the CUDA devices with an ``offloadrt.Runtime`` as one more
    locality, exactly as ``Runtime.connect`` registers a daemon
    (reference runtime.py:204-216).  Returns the CudaLocality; the
    reference runtime's ``close()`` closes it."""
    known = _known_localities(ref_runtime)
    if locality_id is None:
        locality_id = max(known) + 1
    elif locality_id in known:
        raise ValueError(f"locality {locality_id} is already in use by this runtime")
    from offloadrt.registry import LocalityInfo  # the reference package

    loc = CudaLocality(devices, locality_id, record_events)
    try:
        ref_runtime.registry.add_locality(LocalityInfo(locality_id, "cuda"), loc)
    except Exception:
        loc.close()
        raise
    ref_runtime._connections[locality_id] = loc
    ref_runtime._remote_devices[locality_id] = loc.devices
    return loc
