"""Small instances of every builtin/bound kernel and one NVRTC kernel, for
compute-sanitizer (scripts/sanitize.sh).  Results are checked by tests/ -m
gpu; here only the memory/race/sync behaviour matters."""
import numpy as np

from paper_1810_11482_b200 import Runtime
from paper_1810_11482_b200.bindings import kernel_source

with Runtime(devices=[0]) as rt:
    d = rt.get_all_devices().get()[0]
    rng = np.random.default_rng(3)
    n = 100_001
    X, Y = d.create_buffer(n * 8).get(), d.create_buffer(n * 8).get()
    X.enqueue_write(0, rng.random(n))
    bp = d.create_builtin_program().get()
    for name in ("heat", "dot_f32", "mandelbrot_rows"):
        bp.build(name).get()
    g = ((n + 255) // 256, 1, 1), (256, 1, 1)
    bp.run([X, Y, n, 130], "heat", *g).get()          # fused path
    X.enqueue_write(0, rng.standard_normal(n))
    bp.run([X, Y, n, 65], "heat", *g).get()           # unfused path + split pass
    for m in (700, 1024, 1500):                        # general-path windows: one window,
        bp.run([X, Y, m, 20], "heat", *g).get()       # exactly one, flush at both ends
    for op in ("copy", "scale", "add", "triad"):
        p = d.create_program_with_source(kernel_source("stream")).get()
        p.build(op).get()
        args = {"copy": [Y, X, n], "scale": [Y, X, 2.0, n], "add": [Y, X, X, n],
                "triad": [Y, X, X, 3.0, n]}[op]
        p.run(args, op, *g).get()
    F1 = d.create_buffer(n * 4).get()
    F1.enqueue_write(0, rng.random(n, dtype=np.float32))
    O = d.create_buffer(8).get()
    bp.run([F1, F1, O, n], "dot_f32", *g).get()
    M = d.create_buffer(97 * 61 * 4).get()
    bp.run([M, 97, 61, -2.0, 1.0, -1.5, 1.5, 4.0, 300, 1, 3], "mandelbrot_rows", *g).get()
    pp = d.create_program_with_source(kernel_source("partition")).get()
    pp.build("partition").get()
    pp.run([X, 7, n], "partition", *g).get()
    U = d.create_buffer(n * 4).get()
    U.enqueue_write(0, rng.integers(0, 2**32, n, dtype=np.uint32))
    R = d.create_buffer(4).get()
    sp = d.create_program_with_source(kernel_source("sum")).get()
    sp.build("sum").get()
    sp.run([U, R, n], "sum", (1, 1, 1), (32, 1, 1)).get()
    # an unbound kernel: NVRTC path
    src = ("kernel inc(a : buffer_u32, n : scalar_u32) { if (gtid < n) { a[gtid] = a[gtid] + u32(1); } }")
    jp = d.create_program_with_source(src).get()
    jp.build("inc").get()
    jp.run([U, n], "inc", *g).get()
    # 2-D stencil (row batch + per-cell kernels)
    w2, h2 = 130, 67
    S2a, S2b = d.create_buffer(w2 * h2 * 8).get(), d.create_buffer(w2 * h2 * 8).get()
    S2a.enqueue_write(0, rng.random(w2 * h2))
    p2 = d.create_program_with_source(kernel_source("stencil2d")).get()
    p2.build("stencil2d").get()
    p2.run([S2a, S2b, w2, h2], "stencil2d", (64, 1, 1), (256, 1, 1)).get()
    p2.run([S2a, S2b, w2 - 1, h2], "stencil2d", (64, 1, 1), (256, 1, 1)).get()
    print("workloads ok")

# multi-device paths with peer stores / peer atomics (logical devices)
from paper_1810_11482_b200.bench.harness import DotShards, heat2d_multi, heat_multi  # noqa: E402

with Runtime(devices=[0, 0, 0]) as rt3:
    devs = rt3.get_all_devices().get()
    rng = np.random.default_rng(9)
    heat_multi(devs, rng.random(30_001), 70, halo=16, fused=True)
    heat2d_multi(devs, rng.random(66 * 40), 66, 40, 5)
    sh = DotShards(devs, rng.random(90_001, dtype=np.float32), rng.random(90_001, dtype=np.float32),
                   fused=True)
    sh.enqueue().get(timeout=60)
    sh.enqueue().get(timeout=60)
    print("multi-device ok")
