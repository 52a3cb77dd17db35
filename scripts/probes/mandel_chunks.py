"""Probe: end-to-end Mandelbrot (config 3, image into pinned host memory)
through MandelbrotTiles for chunk counts x {interleaved, banded} rows."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

from paper_1810_11482_b200 import Runtime, when_all  # noqa: E402
from paper_1810_11482_b200.bench.harness import MandelbrotTiles  # noqa: E402

with Runtime(devices=[0]) as rt:
    dev = rt.get_all_devices().get()[0]
    for chunks in (4, 8, 12, 16, 32):
        for inter in (False, True):
            t = MandelbrotTiles([dev], 7680, 4320, 2000, chunks=chunks, interleave=inter)
            when_all(t.enqueue()).get()
            best = 1e9
            for _ in range(3):
                t0 = time.perf_counter()
                for _ in range(5):
                    when_all(t.enqueue()).get()
                best = min(best, (time.perf_counter() - t0) / 5 * 1e3)
            import hashlib
            ok = hashlib.sha256(bytes(t.image)).hexdigest().startswith("367317a504ab42ba")
            print(f"sha ok {ok} ", end="")
            print(f"chunks {chunks:3d} {'interleaved' if inter else 'banded'}: {best:.3f} ms")
