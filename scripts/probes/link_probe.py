"""Host link probe: H2D / D2H throughput with 1..4 concurrent copies on
distinct streams (pinned host memory, 256 MiB each), through the public API."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

from paper_1810_11482_b200 import Runtime, pinned_empty, when_all  # noqa: E402

n = 32 << 20  # f64 elements = 256 MiB
with Runtime(devices=[0]) as rt:
    d = rt.get_all_devices().get()[0]
    streams = [0] + [d.create_stream() for _ in range(3)]
    bufs = [d.create_buffer(n * 8).get() for _ in range(4)]
    hosts = [pinned_empty(n * 8, np.float64) for _ in range(4)]
    for h in hosts:
        h[:] = 1.0
    for k in (1, 2, 4):
        for name in ("h2d", "d2h", "both"):
            toks = []
            for _ in range(2):  # warm
                toks = [bufs[i].enqueue_write(0, hosts[i], streams[i]) for i in range(k)]
                when_all(toks).get()
            t0 = time.perf_counter()
            reps = 4
            for _ in range(reps):
                toks = []
                for i in range(k):
                    if name in ("h2d", "both"):
                        toks.append(bufs[i].enqueue_write(0, hosts[i], streams[i]))
                    if name in ("d2h", "both"):
                        j = (i + k) % 4 if name == "both" else i
                        toks.append(bufs[j].enqueue_read_into(0, hosts[j], streams[j]))
                when_all(toks).get()
            dt = time.perf_counter() - t0
            moved = reps * k * n * 8 * (2 if name == "both" else 1)
            print(f"{k} stream(s) {name}: {moved / dt / 1e9:.1f} GB/s")
