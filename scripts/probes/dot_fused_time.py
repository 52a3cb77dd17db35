"""Fused dot + peer-memory allreduce vs the dot builtin: device time per round
on G logical devices of one GPU (the exchange/latency cost; multi-GPU scaling
needs a multi-GPU box).  python scripts/probes/dot_fused_time.py"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

from paper_1810_11482_b200 import Runtime  # noqa: E402
from paper_1810_11482_b200.bench.harness import DotShards  # noqa: E402

for n in (1 << 12, 1 << 31):
    a = np.random.default_rng(1).random(n, dtype=np.float32)
    b = np.random.default_rng(2).random(n, dtype=np.float32)
    for G in (1, 2, 4):
        for fused in (True, False):
            with Runtime(devices=[0] * G) as rt:
                sh = DotShards(rt.get_all_devices().get(), a, b, fused=fused)
                for _ in range(3):
                    t = sh.enqueue()
                    if t is not None:
                        t.get()
                    for d in sh.devices:
                        d.synchronize().get()
                K = 50 if n > 1 << 20 else 2000
                t0 = time.perf_counter()
                for _ in range(K):
                    t = sh.enqueue()
                for d in sh.devices:
                    d.synchronize().get()
                dt = (time.perf_counter() - t0) / K
                val = sh.result()
            print(f"n=2^{n.bit_length() - 1} G={G} fused={fused}: {dt * 1e6:.1f} us/round  "
                  f"result {val:.6f}", flush=True)
