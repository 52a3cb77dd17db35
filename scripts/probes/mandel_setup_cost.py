import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1810_11482_b200 import Runtime
from paper_1810_11482_b200.bindings import kernel_source
with Runtime(devices=[0]) as rt:
    d = rt.get_all_devices().get()[0]
    w, h = 7680, 4320
    O = d.create_buffer(w * h * 4).get()
    p = d.create_program_with_source(kernel_source("mandelbrot")).get(); p.build("mandelbrot").get()
    g = ((w * h + 255) // 256, 1, 1)
    for it in (1, 16, 64, 2000):
        args = [O, w, h, -2.0, 1.0, -1.5, 1.5, 4.0, it]
        for _ in range(3): p.run(args, "mandelbrot", g, (256, 1, 1)).get()
        t0 = time.perf_counter()
        for _ in range(20): p.run(args, "mandelbrot", g, (256, 1, 1))
        p.run(args, "mandelbrot", g, (256, 1, 1)).get()
        print(it, (time.perf_counter() - t0) / 21 * 1e3, "ms")
    # viewport far from the set: all escape at once (setup + interior test + store)
    args = [O, w, h, 10.0, 13.0, 10.0, 13.0, 4.0, 2000]
    p.run(args, "mandelbrot", g, (256, 1, 1)).get()
    t0 = time.perf_counter()
    for _ in range(20): p.run(args, "mandelbrot", g, (256, 1, 1))
    p.run(args, "mandelbrot", g, (256, 1, 1)).get()
    print("far", (time.perf_counter() - t0) / 21 * 1e3, "ms")
