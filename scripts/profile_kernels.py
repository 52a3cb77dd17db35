"""Run one workload a few times through the public API — the target of an
ncu capture (`ncu --set full -k regex:<kernel> -c 1 ... python
scripts/profile_kernels.py <workload>`).  Workloads at BASELINE sizes:
triad (2^25 f64), stencil (2^28 f64, one step), heat (2^28, 1000 steps),
mandel (7680x4320 @2000), dot (2^31 f32), sum (2^28 u32)."""

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

from paper_1810_11482_b200 import Runtime  # noqa: E402
from paper_1810_11482_b200.bindings import kernel_source  # noqa: E402


def main(which: str, reps: int = 3):
    with Runtime(devices=[0]) as rt:
        d = rt.get_all_devices().get()[0]
        if which == "triad":
            n = 1 << 25
            A, B, C = (d.create_buffer(n * 8).get() for _ in range(3))
            B.enqueue_write(0, np.ones(n))
            C.enqueue_write(0, np.ones(n))
            p = d.create_program_with_source(kernel_source("stream")).get()
            p.build("triad").get()
            for _ in range(reps):
                p.run([A, B, C, 3.0, n], "triad", (n // 256, 1, 1), (256, 1, 1))
        elif which == "heat_time":  # tuning sweeps: config 2 timed, no oracle
            import ctypes

            from paper_1810_11482_b200 import _native

            lib = _native.load()
            n = 1 << 28
            X, Y = d.create_buffer(n * 8).get(), d.create_buffer(n * 8).get()
            X.enqueue_write(0, np.random.default_rng(0).random(n))
            p = d.create_builtin_program().get()
            p.build("heat").get()
            p.run([X, Y, n, 64], "heat", (n // 256, 1, 1), (256, 1, 1))
            st = rt.device_objects()[0].stream(0)
            e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
            lib.ofl_event_create(0, ctypes.byref(e0))
            lib.ofl_event_create(0, ctypes.byref(e1))
            lib.ofl_event_record(e0, st.ptr)
            p.run([X, Y, n, 1000], "heat", (n // 256, 1, 1), (256, 1, 1))
            lib.ofl_event_record(e1, st.ptr)
            ms = ctypes.c_float()
            lib.ofl_event_elapsed_ms(e0, e1, ctypes.byref(ms))
            print(f"heat 2^28 x 1000 steps: {ms.value:.2f} ms")
        elif which in ("stencil", "heat"):
            n = 1 << 28
            X, Y = d.create_buffer(n * 8).get(), d.create_buffer(n * 8).get()
            X.enqueue_write(0, np.random.default_rng(0).random(n))
            if which == "stencil":
                p = d.create_program_with_source(kernel_source("stencil")).get()
                p.build("stencil").get()
                for _ in range(reps):
                    p.run([X, Y, n], "stencil", (n // 256, 1, 1), (256, 1, 1))
            else:
                p = d.create_builtin_program().get()
                p.build("heat").get()
                # config 2's schedule: 1000 steps = 12 passes of ~83 steps
                p.run([X, Y, n, 1000], "heat", (n // 256, 1, 1), (256, 1, 1))
        elif which == "mandel":
            w, h = 7680, 4320
            O = d.create_buffer(w * h * 4).get()
            p = d.create_program_with_source(kernel_source("mandelbrot")).get()
            p.build("mandelbrot").get()
            for _ in range(reps):
                p.run([O, w, h, -2.0, 1.0, -1.5, 1.5, 4.0, 2000], "mandelbrot",
                      ((w * h) // 256, 1, 1), (256, 1, 1))
        elif which == "dot":
            n = 1 << 31
            A, B, R = d.create_buffer(n * 4).get(), d.create_buffer(n * 4).get(), d.create_buffer(8).get()
            p = d.create_builtin_program().get()
            p.build("dot_f32").get()
            for _ in range(reps):
                p.run([A, B, R, n], "dot_f32", (n // 256, 1, 1), (256, 1, 1))
        elif which == "sum":
            n = 1 << 28
            I, R = d.create_buffer(n * 4).get(), d.create_buffer(4).get()
            p = d.create_program_with_source(kernel_source("sum")).get()
            p.build("sum").get()
            for _ in range(reps):
                p.run([I, R, n], "sum", (1, 1, 1), (32, 1, 1))
        d.synchronize().get()


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 3)
