"""Probe: where a 256 MiB enqueue_read -> bytes spends its time.

  a. D2H into a pinned array (the link alone)
  b. enqueue_read(0, n).get() (chunked D2H + parallel copy into a new bytes)
  c. host only: the copy threads filling a fresh bytes object from pinned
     memory (hostmem.memcpy), with and without MADV_HUGEPAGE
  d. pageable enqueue_write from a numpy array (staging copies + DMA)
python scripts/probes/read_bytes_probe.py
"""

from __future__ import annotations

import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402

from paper_1810_11482_b200 import Runtime, hostmem, pinned_empty  # noqa: E402

libc = ctypes.CDLL(None, use_errno=True)
MADV_HUGEPAGE = 14


def best(fn, reps=5) -> float:
    fn()
    out = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        out.append(time.perf_counter() - t0)
    return min(out)


def main() -> None:
    n = 1 << 28
    rt = Runtime(devices=[0])
    dev = rt.get_all_devices().get()[0]
    buf = dev.create_buffer(n).get()
    pin = pinned_empty(n)
    pin[:] = 3
    page = np.full(n, 5, np.uint8)
    res = {}
    res["a_d2h_pinned_gbs"] = n / best(lambda: buf.enqueue_read_into(0, pin).get()) / 1e9
    res["b_read_bytes_gbs"] = n / best(lambda: buf.enqueue_read(0, n).get()) / 1e9

    def host_fill(advise: bool) -> None:
        out = bytes(n)
        addr = id(out) + hostmem._BYTES_OFF
        if advise:
            lo = (addr + (2 << 20) - 1) & ~((2 << 20) - 1)
            hi = (addr + n) & ~((2 << 20) - 1)
            libc.madvise(ctypes.c_void_p(lo), ctypes.c_size_t(hi - lo), MADV_HUGEPAGE)
        hostmem.memcpy(addr, pin._address(), n)

    res["c_host_fill_fresh_gbs"] = n / best(lambda: host_fill(False)) / 1e9
    res["c_host_fill_fresh_huge_gbs"] = n / best(lambda: host_fill(True)) / 1e9
    warm = bytearray(n)
    waddr = ctypes.addressof((ctypes.c_char * n).from_buffer(warm))
    res["c_host_fill_prefaulted_gbs"] = n / best(lambda: hostmem.memcpy(waddr, pin._address(), n)) / 1e9
    res["e_read_into_prefaulted_bytearray_gbs"] = n / best(lambda: buf.enqueue_read_into(0, warm).get()) / 1e9
    for mb in (2, 4, 16, 32, 64):
        hostmem.READ_CHUNK = mb << 20
        res[f"e_read_into_prefaulted_chunk{mb}MiB_gbs"] = n / best(lambda: buf.enqueue_read_into(0, warm).get()) / 1e9
    hostmem.READ_CHUNK = 8 << 20

    def settled_then_collect() -> None:
        tok = buf.enqueue_read_into(0, warm)
        dev.synchronize().get()  # every chunk landed: collect is host copies only
        tok.get()

    res["e_read_into_prefaulted_d2h_then_collect_gbs"] = n / best(settled_then_collect) / 1e9
    pin2 = pinned_empty(n)
    s1 = dev.create_stream()

    def fill_during_d2h() -> None:
        tok = buf.enqueue_read_into(0, pin2, s1)
        host_fill(True)
        tok.get()

    res["e_host_fill_huge_during_d2h_gbs"] = n / best(fill_during_d2h) / 1e9
    res["d_write_pageable_gbs"] = n / best(lambda: buf.enqueue_write(0, page).get()) / 1e9
    res["d_write_pinned_gbs"] = n / best(lambda: buf.enqueue_write(0, pin).get()) / 1e9
    for f in ("enabled", "defrag"):
        try:
            with open(f"/sys/kernel/mm/transparent_hugepage/{f}") as fh:
                res[f"thp_{f}"] = fh.read().strip()
        except OSError:
            pass
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in res.items()}))
    rt.close()


if __name__ == "__main__":
    main()
