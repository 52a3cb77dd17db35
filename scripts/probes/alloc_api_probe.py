"""create_buffer / drop timing through the API (buffers >= 2 MiB are VMM
mappings, smaller ones come from the stream-ordered pool), and whether a
drop waits for a kernel running on another stream."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))

from paper_1810_11482_b200 import Runtime  # noqa: E402
from test_gpu_memory import _long_heat  # noqa: E402

with Runtime(devices=[0]) as rt:
    d = rt.get_all_devices().get()[0]
    for size in (1 << 10, 1 << 20, 64 << 20, 1 << 30, 8 << 30):
        for rep in range(2):
            t0 = time.perf_counter()
            b = d.create_buffer(size).get()
            t1 = time.perf_counter()
            rt.registry.unregister(b.gid)
            del b
            t2 = time.perf_counter()
            print(f"{size >> 10:>9} KiB rep {rep}: create {1e3 * (t1 - t0):8.2f} ms  drop {1e3 * (t2 - t1):6.2f} ms",
                  flush=True)
    s1 = d.create_stream()
    tok, keep = _long_heat(d, s1)
    t0 = time.perf_counter()
    for size in (1 << 10, 64 << 20, 1 << 30):
        b = d.create_buffer(size).get()
        rt.registry.unregister(b.gid)
        del b
    print(f"create+drop 1 KiB, 64 MiB, 1 GiB during a 50 ms kernel: {1e3 * (time.perf_counter() - t0):.2f} ms, "
          f"kernel still running: {not tok.done()}", flush=True)
    tok.get()
