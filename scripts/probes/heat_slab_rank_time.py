"""Probe: one rank's share of config 2 at world W (the middle slab: both
neighbours, halo 96, 1000 steps in passes of <= 96) timed alone on one GPU,
its strips stored into local stand-in ghost buffers.  Without the exchange
latency this is the per-GPU compute time a W-GPU run is bounded by; ideal =
the single-GPU time / W.  python scripts/probes/heat_slab_rank_time.py"""
from __future__ import annotations

import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402

from paper_1810_11482_b200 import Runtime, _native  # noqa: E402
from paper_1810_11482_b200.bench import decomp  # noqa: E402


def main() -> None:
    n, steps, h = 1 << 28, 1000, 96
    lib = _native.load()
    with Runtime(devices=[0]) as rt:
        dev = rt.get_all_devices().get()[0]
        dobj = rt.device_objects()[0]
        st = dobj.stream(0)
        for world in (1, 2, 4, 8):
            sl = decomp.slabs(n, world, h)[world // 2]
            m = sl.length
            A, B = dev.create_buffer(m * 8).get(), dev.create_buffer(m * 8).get()
            G = dev.create_buffer(4 * h * 8).get()
            A.enqueue_write(0, np.random.default_rng(1).random(m)).get()
            pa, pb, pg = (rt.local._buffer(b.gid).ptr for b in (A, B, G))
            ks = [min(h, steps - d) for d in range(0, steps, h)]
            tk = ctypes.c_uint64()

            def run() -> float:
                dev.synchronize().get()
                t0 = time.perf_counter()
                cur, nxt = pa, pb
                for k in ks:
                    _native.check(lib.ofl_heat_slab(
                        st.ptr, cur, nxt, m, k, sl.left, sl.left + sl.owned,
                        pg if sl.left else None, 0, pg + 2 * h * 8 if sl.right else None, 0, h,
                        ctypes.byref(tk)), "slab pass")
                    cur, nxt = nxt, cur
                st.wait_ticket(tk.value)
                return time.perf_counter() - t0

            run()
            ms = min(run() for _ in range(3)) * 1e3
            print(json.dumps({"world": world, "slab_cells": m, "passes": len(ks),
                              "ms": round(ms, 3)}), flush=True)
            del A, B, G


if __name__ == "__main__":
    main()
