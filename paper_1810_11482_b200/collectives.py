"""NCCL collectives on runtime buffers (BASELINE config 4).

The reference has no collective (cross-device traffic is
read -> host -> write).  Here an allreduce is one ``ncclAllReduce`` enqueued
on each participating buffer's default stream, in place, so a reduction
kernel followed by the allreduce never touches the host; the returned
token completes when every rank's stream has passed the collective.

Two ways to form a communicator:

* ``Communicator.single_process(rt, devices)`` — one process driving several
  GPUs (ncclCommInitAll; the devices must be distinct physical GPUs, NCCL
  refuses two ranks on one GPU);
* ``Communicator.from_process_group(rt, device)`` — one process per GPU
  under torchrun; the NCCL unique id travels over torch.distributed.
"""

from __future__ import annotations

import ctypes
from typing import Optional, Sequence

from . import _native
from .errors import BadArgsError
from .futures import CompletionToken, when_all

_DTYPES = {"u32": _native.DT_U32, "f64": _native.DT_F64, "f32": _native.DT_F32}
_OPS = {"sum": _native.OP_SUM, "max": _native.OP_MAX}


class Communicator:
    def __init__(self, rt, devices: Sequence, comms: list):
        self._rt = rt
        self.devices = list(devices)
        self._comms = comms

    @classmethod
    def single_process(cls, rt, devices: Sequence) -> "Communicator":
        lib = _native.load()
        _native.check(lib.ofl_nccl_available(_native.nccl_library_path().encode()), "nccl")
        objs = [rt.local._device(d.gid) for d in devices]
        ordinals = [o.ordinal for o in objs]
        if len(set(ordinals)) != len(ordinals):
            raise BadArgsError("NCCL needs one rank per physical GPU")
        arr = (ctypes.c_int * len(ordinals))(*ordinals)
        out = (ctypes.c_void_p * len(ordinals))()
        _native.check(lib.ofl_nccl_init_all(len(ordinals), arr, out), "ncclCommInitAll")
        return cls(rt, devices, [out[i] for i in range(len(ordinals))])

    @classmethod
    def from_process_group(cls, rt, device, group=None) -> "Communicator":
        import torch.distributed as dist

        lib = _native.load()
        _native.check(lib.ofl_nccl_available(_native.nccl_library_path().encode()), "nccl")
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            _native.check(lib.ofl_nccl_unique_id(uid), "ncclGetUniqueId")
        box = [uid.raw if rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        uid = ctypes.create_string_buffer(box[0], 128)
        comm = ctypes.c_void_p()
        ordinal = rt.local._device(device.gid).ordinal
        _native.check(
            lib.ofl_nccl_init_rank(world, rank, ordinal, uid, ctypes.byref(comm)),
            "ncclCommInitRank",
        )
        return cls(rt, [device], [comm.value])

    def allreduce(self, buffers: Sequence, count: int, dtype: str = "f64", op: str = "sum",
                  stream: int = 0) -> CompletionToken:
        """In-place allreduce of the first `count` elements of each buffer
        (one buffer per local rank, in device order)."""
        if len(buffers) != len(self._comms):
            raise BadArgsError("one buffer per local rank")
        dt, ro = _DTYPES[dtype], _OPS[op]
        lib = _native.load()
        objs = [self._rt.local._buffer(b.gid) for b in buffers]
        streams = [o.device.stream(stream) for o in objs]
        if len(objs) == 1:
            t = ctypes.c_uint64()
            o, s = objs[0], streams[0]
            _native.check(
                lib.ofl_allreduce(self._comms[0], s.ptr, o.ptr, o.ptr, count, dt, ro,
                                  ctypes.byref(t)),
                "ncclAllReduce",
            )
            return s.token(t.value)
        n = len(objs)
        comms = (ctypes.c_void_p * n)(*self._comms)
        sts = (ctypes.c_void_p * n)(*[s.ptr for s in streams])
        ptrs = (ctypes.c_void_p * n)(*[o.ptr for o in objs])
        tickets = (ctypes.c_uint64 * n)()
        _native.check(
            lib.ofl_allreduce_group(n, comms, sts, ptrs, ptrs, count, dt, ro, tickets),
            "ncclAllReduce (group)",
        )
        return when_all([s.token(tickets[i]) for i, s in enumerate(streams)])

    def close(self) -> None:
        lib = _native.load()
        for c in self._comms:
            lib.ofl_comm_destroy(c)
        self._comms = []


def destroy(comm: Optional[Communicator]) -> None:
    if comm is not None:
        comm.close()


class PeerGroup:
    """Exchange blocks for reductions fused into kernels across the devices
    this process drives (``ofl_dot_f32_allreduce``): one small zero-filled
    block per device, written by every member over NVLink peer stores.  The
    round counter orders successive reductions on the group (double-buffered
    slots, monotonically increasing arrival counters, no resets)."""

    def __init__(self, rt, devices: Sequence):
        lib = _native.load()
        if not 1 <= len(devices) <= 16:
            raise BadArgsError("a peer group has 1..16 members")
        nbytes = lib.ofl_xchg_bytes()
        self._rt = rt
        self.devices = list(devices)
        self.blocks = [d.create_buffer(nbytes).get() for d in self.devices]
        objs = [rt.local._buffer(b.gid) for b in self.blocks]
        G = len(objs)
        self.ptrs = (ctypes.c_void_p * G)(*[o.ptr for o in objs])
        self.ordinals = (ctypes.c_int * G)(*[o.device.ordinal for o in objs])
        self.round = 0

    def dot_f32(self, a_bufs: Sequence, b_bufs: Sequence, out_bufs: Sequence,
                counts: Sequence[int]) -> CompletionToken:
        """Per-member fp32 dot of its shard, summed across the group inside
        the kernels; every out buffer's first f64 holds the identical total."""
        G = len(self.devices)
        if not (len(a_bufs) == len(b_bufs) == len(out_bufs) == len(counts) == G):
            raise BadArgsError("one shard per group member")
        lib = _native.load()
        local = self._rt.local
        toks = []
        ticket = ctypes.c_uint64()
        for g in range(G):
            A, B, R = (local._buffer(x.gid) for x in (a_bufs[g], b_bufs[g], out_bufs[g]))
            n = int(counts[g])
            if n > min(A.elements("buffer_f32"), B.elements("buffer_f32")) or R.size_bytes < 8:
                raise BadArgsError("shard larger than its buffers")
            st = A.device.stream(0)
            _native.check(lib.ofl_dot_f32_allreduce(
                st.ptr, A.ptr, B.ptr, R.ptr, n, g, G, self.ptrs, self.ordinals, self.round,
                ctypes.byref(ticket)), "fused dot allreduce")
            toks.append(st.token(ticket.value))
        self.round += 1
        return when_all(toks)


class ProcessPeerGroup:
    """The fused cross-device reduction for one process per GPU (torchrun):
    every rank allocates its exchange block, the 64-byte CUDA IPC handles
    travel over torch.distributed (host side only, once), and each rank maps
    the others' blocks — the reduction kernel then stores into and waits on
    peer memory exactly as in ``PeerGroup``, with no collective call on the
    data path."""

    def __init__(self, rt, device, group=None):
        import torch.distributed as dist

        lib = _native.load()
        self._rt = rt
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if not 1 <= self.world <= 16:
            raise BadArgsError("a peer group has 1..16 members")
        self.block = device.create_buffer(lib.ofl_xchg_bytes(), shareable=True).get()
        obj = rt.local._buffer(self.block.gid)
        self.ordinal = obj.device.ordinal
        handle = ctypes.create_string_buffer(64)
        _native.check(lib.ofl_ipc_handle(obj.ptr, handle), "ipc handle")
        handles = [None] * self.world
        dist.all_gather_object(handles, handle.raw, group=group)
        ptrs = []
        self._opened = []
        for r, h in enumerate(handles):
            if r == self.rank:
                ptrs.append(obj.ptr)
                continue
            p = ctypes.c_void_p()
            _native.check(lib.ofl_ipc_open(self.ordinal, h, ctypes.byref(p)), "ipc open")
            self._opened.append(p.value)
            ptrs.append(p.value)
        self.ptrs = (ctypes.c_void_p * self.world)(*ptrs)
        # the mapped peers are reached through IPC mappings: no extra peer
        # enabling on this side (cudaIpcMemLazyEnablePeerAccess did it)
        self.ordinals = (ctypes.c_int * self.world)(*([self.ordinal] * self.world))
        self.round = 0
        dist.barrier(group=group)  # every block exists and is mapped before use

    def dot_f32(self, a_buf, b_buf, out_buf, n: int) -> CompletionToken:
        """This rank's shard dot, summed across the ranks inside the kernel;
        out_buf's first f64 holds the total (identical bits on every rank)."""
        lib = _native.load()
        local = self._rt.local
        A, B, R = (local._buffer(x.gid) for x in (a_buf, b_buf, out_buf))
        if n > min(A.elements("buffer_f32"), B.elements("buffer_f32")) or R.size_bytes < 8:
            raise BadArgsError("shard larger than its buffers")
        st = A.device.stream(0)
        ticket = ctypes.c_uint64()
        _native.check(lib.ofl_dot_f32_allreduce(
            st.ptr, A.ptr, B.ptr, R.ptr, n, self.rank, self.world, self.ptrs, self.ordinals,
            self.round, ctypes.byref(ticket)), "fused dot allreduce")
        self.round += 1
        return st.token(ticket.value)

    def close(self) -> None:
        lib = _native.load()
        for p in self._opened:
            lib.ofl_ipc_close(self.ordinal, p)
        self._opened = []
