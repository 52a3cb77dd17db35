"""Probe: split the chunked Mandelbrot end to end into its kernels alone and
its strided reads alone (per chunk count, banded vs interleaved rows)."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

from paper_1810_11482_b200 import Runtime, when_all  # noqa: E402
from paper_1810_11482_b200.bench.harness import MandelbrotTiles  # noqa: E402


def timed(fn, reps=5):
    fn()
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        best = min(best, (time.perf_counter() - t0) / reps * 1e3)
    return best


with Runtime(devices=[0]) as rt:
    dev = rt.get_all_devices().get()[0]
    for chunks in (1, 4, 8, 16, 32):
        for inter in (False, True):
            t = MandelbrotTiles([dev], 7680, 4320, 2000, chunks=chunks, interleave=inter)
            w, G = t.width, 1
            re0, re1, im0, im1 = t.viewport
            sid = t.streams[0][0]

            def kernels():
                toks = []
                for k0, step, cnt, buf in t.parts[0]:
                    first = k0
                    items = (first + (cnt - 1) * step + 1) * w
                    toks.append(t.progs[0].run([buf, w, t.height, re0, re1, im0, im1, t.esc,
                                                t.max_iter, first, step], "mandelbrot_rows",
                                               (math.ceil(items / 256), 1, 1), (256, 1, 1), sid))
                when_all(toks).get()

            def reads():
                toks = [buf.enqueue_read_rows_into(0, t.image, w * 4, cnt, k0 * w * 4,
                                                   step * w * 4, sid)
                        for k0, step, cnt, buf in t.parts[0]]
                when_all(toks).get()

            full = timed(lambda: when_all(t.enqueue()).get())
            print(f"chunks {chunks:3d} interleave {inter!s:5}: kernels {timed(kernels):.3f} ms, "
                  f"reads {timed(reads):.3f} ms, full {full:.3f} ms")
