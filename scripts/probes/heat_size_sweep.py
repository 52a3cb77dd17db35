"""Probe: heat builtin time vs field size (1000 steps): a fixed cost per
pass shows up as a floor at small n.  python scripts/probes/heat_size_sweep.py"""
from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402

from paper_1810_11482_b200 import Runtime  # noqa: E402
from paper_1810_11482_b200.bench.harness import _builtin  # noqa: E402


def main() -> None:
    steps = int(os.environ.get("STEPS", "1000"))
    sizes = [int(s) for s in os.environ.get("SIZES", "65536,1048576,4194304,11184810,33554432,67108864,268435456").split(",")]
    with Runtime(devices=[0]) as rt:
        dev = rt.get_all_devices().get()[0]
        prog = _builtin(dev, "heat")
        for n in sizes:
            X, Y = dev.create_buffer(n * 8).get(), dev.create_buffer(n * 8).get()
            X.enqueue_write(0, np.random.default_rng(1).random(n)).get()
            args = [X, Y, n, steps]
            grid = ((n + 255) // 256, 1, 1)
            prog.run(args, "heat", grid, (256, 1, 1)).get()
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                prog.run(args, "heat", grid, (256, 1, 1)).get()
                ts.append(time.perf_counter() - t0)
            ms = min(ts) * 1e3
            print(json.dumps({"n": n, "steps": steps, "ms": round(ms, 3),
                              "ns_per_Gcellstep": round(ms * 1e6 / (n * steps) * 1e3, 3),
                              "cellsteps_per_s": round(n * steps / (ms * 1e-3) / 1e12, 3)}), flush=True)
            del X, Y


if __name__ == "__main__":
    main()
