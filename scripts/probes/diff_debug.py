"""Dump one differential-fuzz plan (tests/test_gpu_differential.py) with both
runtimes' outcomes side by side.  python scripts/probes/diff_debug.py SEED"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [os.path.join(REPO, "tests"), REPO]
import test_gpu_differential as T  # noqa: E402

seed = int(sys.argv[1])
gen = T.worlds.__wrapped__() if hasattr(T.worlds, "__wrapped__") else None
src = T._ref_src()
sys.path.insert(0, src)
import offloadrt  # noqa: E402
from offloadrt.bench import kernel_source as rks  # noqa: E402
import paper_1810_11482_b200 as ours  # noqa: E402
from paper_1810_11482_b200.bindings import kernel_source as oks  # noqa: E402

sources = {"stream": oks("stream"), "stencil2d": oks("stencil2d"), "stencil": rks("stencil"),
           "sum": rks("sum"), "mandelbrot": rks("mandelbrot")}
rrt = offloadrt.Runtime(backend="host", devices=1)
ort = ours.Runtime(devices=[0])
ops = T._plan(seed)
tr, to = set(), set()
own = []
a = T._execute(T.World(offloadrt, rrt, rrt.get_all_devices().get()[0], sources), ops, tr, own)
own.extend([-1] * (len(a) - len(own)))
b = T._execute(T.World(ours, ort, ort.get_all_devices().get()[0], sources), ops, to)
for i, op in enumerate(ops):
    print("OP", i, repr(op)[:200])
for i, (x, y) in enumerate(zip(a, b)):
    flag = "  " if T._same(x, y) else "XX"
    print(flag, i, "op", own[i], repr(x)[:160], "|", repr(y)[:160])
print("tainted", tr, to)
from collections import Counter  # noqa: E402
print("outcome kinds (reference):", Counter(o[0] if o[0] != "final" else "final-" + o[2] for o in a))
print("data comparisons:", sum(1 for o in a if isinstance(o[-1], bytes) and o[-1]))
