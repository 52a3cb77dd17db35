"""cProfile of the pipelined futures chain (write 8 B + triad N=1024 +
when_all per step) on the real library: where the per-future cost goes."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1810_11482_b200 import Runtime, make_ready, pinned_empty, when_all  # noqa: E402
from paper_1810_11482_b200.bindings import kernel_source  # noqa: E402

rt = Runtime(devices=[0])
dev = rt.get_all_devices().get()[0]
n = 1024
A, B, C, D = (dev.create_buffer(n * 8).get() for _ in range(4))
p = dev.create_program_with_source(kernel_source("stream")).get()
p.build("triad").get()
payload = pinned_empty(8)
args = [A, B, C, 3.0, n]
grid, blk = (4, 1, 1), (256, 1, 1)
K = int(os.environ.get("K", 20000))


def chain():
    prev = make_ready(None)
    for _ in range(K):
        w = D.enqueue_write(0, payload)
        r = p.run(args, "triad", grid, blk)
        prev = when_all([prev, w, r])
    prev.get()


chain()
t0 = time.perf_counter()
chain()
print(f"chain step {(time.perf_counter() - t0) / K * 1e6:.2f} us")
cProfile.run("chain()", "/tmp/prof.out")
pstats.Stats("/tmp/prof.out").sort_stats("tottime").print_stats(14)
