"""Host-side cost of the futurized API per operation, measured against the
null test double of libofl.so (no device): isolates the Python + ctypes
layers.  Usage: OFL_LIB=tests/fakes/_build/libnull_ofl.so python scripts/host_overhead_probe.py [--profile]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_11482_b200 import Runtime, make_ready, pinned_empty, when_all
from paper_1810_11482_b200.bindings import kernel_source

rt = Runtime(devices=[0])
dev = rt.get_all_devices().get()[0]
n = 1024
A, B, C, D = (dev.create_buffer(n * 8).get() for _ in range(4))
p = dev.create_program_with_source(kernel_source("stream")).get(); p.build("triad").get()
payload = pinned_empty(8)
args = [A, B, C, 3.0, n]; grid = (4, 1, 1); blk = (256, 1, 1)
K = 100000

def run_only():
    for _ in range(K): p.run(args, "triad", grid, blk)
def write_only():
    for _ in range(K): D.enqueue_write(0, payload)
def chain():
    prev = make_ready(None)
    for _ in range(K):
        w = D.enqueue_write(0, payload); r = p.run(args, "triad", grid, blk)
        prev = when_all([prev, w, r])
    prev.get()

for name, fn in (("run", run_only), ("write", write_only), ("chain step", chain)):
    t0 = time.perf_counter(); fn(); dt = time.perf_counter() - t0
    print(f"{name:12s} {dt / K * 1e6:7.2f} us")
if "--profile" in sys.argv:
    import cProfile, pstats
    cProfile.run("chain()", "/tmp/prof.out")
    pstats.Stats("/tmp/prof.out").sort_stats("tottime").print_stats(18)
