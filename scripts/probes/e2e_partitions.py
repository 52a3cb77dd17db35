"""Probe: end-to-end triad (host buffers) as Alg. 1 partitions.

Each step of N=2^25 fp64 is cut into P partitions; partition job j runs on
stream j mod S with its own device buffer triplet (write b_p, write c_p, run,
read_into a_p), so the D2H of one partition overlaps the H2D of the next on
the full-duplex link.  Prints GB/s (24 B/element, same count as bench.py's
e2e) per (P, S).  python scripts/probes/e2e_partitions.py
"""

from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402

from paper_1810_11482_b200 import Runtime, pinned_empty  # noqa: E402
from paper_1810_11482_b200.bindings import kernel_source  # noqa: E402


def main() -> None:
    n = 1 << 25
    s = 3.0
    steps = int(os.environ.get("STEPS", "20"))
    rt = Runtime(devices=[0])
    dev = rt.get_all_devices().get()[0]
    rng = np.random.default_rng(20180214)
    b = pinned_empty(n * 8, np.float64)
    c = pinned_empty(n * 8, np.float64)
    a = pinned_empty(n * 8, np.float64)
    b[:] = rng.random(n)
    c[:] = rng.random(n)
    expect = b + s * c
    prog = dev.create_program_with_source(kernel_source("stream")).get()
    prog.build("triad").get()
    out = []
    for P in (1, 2, 4, 8, 16, 32):
        for S in (2, 3, 4):
            m = n // P
            sets = [tuple(dev.create_buffer(m * 8).get() for _ in range(3)) + (dev.create_stream(),)
                    for _ in range(S)]
            grid, block = ((m + 255) // 256, 1, 1), (256, 1, 1)

            def run(k_steps: int) -> None:
                last = [None] * S
                j = 0
                for _ in range(k_steps):
                    for p in range(P):
                        A, B, C, st = sets[j % S]
                        lo, hi = p * m, (p + 1) * m
                        B.enqueue_write(0, b[lo:hi], st)
                        C.enqueue_write(0, c[lo:hi], st)
                        prog.run([A, B, C, s, m], "triad", grid, block, st)
                        if last[j % S] is not None and j >= 4 * S:
                            last[j % S].get()  # bound the queue depth
                        last[j % S] = A.enqueue_read_into(0, a[lo:hi], st)
                        j += 1
                for t in last:
                    if t is not None:
                        t.get()

            run(2)
            a[:] = 0
            t0 = time.perf_counter()
            run(steps)
            dt = time.perf_counter() - t0
            ok = bool(np.array_equal(a.view(np.uint64), expect.view(np.uint64)))
            gbs = 24 * n * steps / dt / 1e9
            rec = {"P": P, "S": S, "gbs": round(gbs, 2), "ms_per_step": round(dt / steps * 1e3, 3), "ok": ok}
            print(json.dumps(rec), flush=True)
            out.append(rec)
            del sets
    rt.close()


if __name__ == "__main__":
    main()
