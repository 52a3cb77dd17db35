"""Probe: config 2 end to end (pinned host field in, 1000 steps, field out)
with bench.HeatChunks over piece / buffer-set counts, against the
monolithic write -> heat -> read.  Every line checks the reference sha256.
python scripts/probes/heat_e2e_chunks.py"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402

from paper_1810_11482_b200 import Runtime, pinned_empty, when_all  # noqa: E402
from paper_1810_11482_b200.bench import HeatChunks  # noqa: E402

REF = "7439c751212816525f75ab244e524a4344d44e53bb1061dab990808754b9fe9b"


def main() -> None:
    n, steps = 1 << 28, 1000
    with Runtime(devices=[0]) as rt:
        dev = rt.get_all_devices().get()[0]
        x = pinned_empty(n * 8, np.float64)
        x[:] = np.random.default_rng(20180214).random(n)
        out = pinned_empty(n * 8, np.float64)
        combos = [tuple(map(int, c.split("x"))) for c in
                  os.environ.get("COMBOS", "8x2,8x3,16x2,16x3,16x4,24x6,32x3,32x4,64x3").split(",")]
        for chunks, sets in combos:
            hc = HeatChunks(dev, n, steps, chunks=chunks, sets=sets)
            ts = []
            for _ in range(3):
                out[:1] = 0
                dev.synchronize().get()
                t0 = time.perf_counter()
                when_all(hc.enqueue(x, out)).get()
                ts.append(time.perf_counter() - t0)
            ok = hashlib.sha256(out).hexdigest() == REF
            print(json.dumps({"chunks": chunks, "sets": sets, "e2e_ms": round(min(ts) * 1e3, 2),
                              "all_ms": [round(t * 1e3, 1) for t in ts], "bitexact": ok}),
                  flush=True)
            del hc


if __name__ == "__main__":
    main()
