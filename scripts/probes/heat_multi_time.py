"""Multi-device heat (config 2 shape: 2^28 f64, 1000 steps, halo 64) on G
logical devices of one GPU: fused peer-store exchange vs copy() exchange.
On one B200 the slabs share the SMs, so this measures the exchange and
launch overhead, not multi-GPU scaling.  Usage: python scripts/probes/heat_multi_time.py G..."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

from paper_1810_11482_b200 import Runtime  # noqa: E402
from paper_1810_11482_b200.bench.harness import HeatSlabs  # noqa: E402

n, steps = 1 << 28, 1000
x = np.random.default_rng(0).random(n)
for G in [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]:
    for fused in (True, False):
        with Runtime(devices=[0] * G) as rt:
            devs = rt.get_all_devices().get()
            slabs = HeatSlabs(devs, x, halo=64, fused=fused)
            t = slabs.run(64)  # warm-up pass
            for d in devs:
                d.synchronize().get()
            t0 = time.perf_counter()
            t = slabs.run(steps)
            if t is not None:
                t.get()
            for d in devs:
                d.synchronize().get()
            dt = time.perf_counter() - t0
        print(f"G={G} fused={fused}: {dt * 1e3:.1f} ms for {steps} steps", flush=True)
