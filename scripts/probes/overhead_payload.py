"""Probe: why the 4 KiB-payload futurized chain can beat the raw chain.

Times, per step (H2D payload + triad N=1024 on one stream):
  raw      — ofl_bench_raw_chain mode 0 (cudaMemcpyAsync + the launch ofl_stream_op issues)
  capi     — the product C-ABI without futures (ofl_h2d + ofl_stream_op from Python)
  futures  — the futurized API (enqueue_write + program.run + when_all chain)
for payloads of 8 B and 4 KiB.  Run on the GPU box: python scripts/probes/overhead_payload.py
"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

from paper_1810_11482_b200 import Runtime, _native, make_ready, pinned_empty, when_all  # noqa: E402
from paper_1810_11482_b200.bindings import kernel_source  # noqa: E402


def main():
    lib = _native.load()
    rt = Runtime(devices=[0])
    dev = rt.get_all_devices().get()[0]
    n = 1024
    A, B, C = (dev.create_buffer(n * 8).get() for _ in range(3))
    D = dev.create_buffer(65536).get()
    prog = dev.create_program_with_source(kernel_source("stream")).get()
    prog.build("triad").get()
    st = rt.device_objects()[0].stream(0)
    dptr = rt.local._buffer(D.gid).ptr
    aptr, bptr, cptr = (rt.local._buffer(x.gid).ptr for x in (A, B, C))
    steps = 10000
    args = [A, B, C, 3.0, n]
    grid, block = ((n + 255) // 256, 1, 1), (256, 1, 1)
    for nbytes in (8, 4096, 65536):
        payload = pinned_empty(nbytes)
        payload[:] = 1

        def raw():
            secs = ctypes.c_double()
            _native.check(lib.ofl_bench_raw_chain(st.ptr, dptr, payload.ctypes.data, nbytes, aptr,
                                                  bptr, cptr, n, steps, 0, ctypes.byref(secs)), "raw")
            return secs.value

        def capi():
            t = ctypes.c_uint64()
            ref = ctypes.byref(t)
            dev.synchronize().get()
            t0 = time.perf_counter()
            for _ in range(steps):
                lib.ofl_h2d(st.ptr, dptr, payload.ctypes.data, nbytes, ref)
                lib.ofl_stream_op(st.ptr, 3, aptr, bptr, cptr, 3.0, n, ref)
            dev.synchronize().get()
            return time.perf_counter() - t0

        def fut():
            dev.synchronize().get()
            t0 = time.perf_counter()
            prev = make_ready(None)
            for _ in range(steps):
                w = D.enqueue_write(0, payload)
                r = prog.run(args, "triad", grid, block)
                prev = when_all([prev, w, r])
            prev.get()
            return time.perf_counter() - t0

        for f in (raw, capi, fut):
            f()
        res = {f.__name__: min(f() for _ in range(3)) / steps * 1e6 for f in (raw, capi, fut)}
        print(f"payload {nbytes:6d} B: " + ", ".join(f"{k} {v:.2f} us/step" for k, v in res.items()))
    rt.close()


if __name__ == "__main__":
    main()
