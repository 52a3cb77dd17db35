"""A kernel with no hand-written binding (NVRTC path): an element-wise
fp64 kernel over 2^25 elements, back-to-back launches, GB/s — how far the
generic codegen is from the bound STREAM kernels."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

from paper_1810_11482_b200 import Runtime, _native  # noqa: E402

SRC = """
kernel axpby(y : buffer_f64, x : buffer_f64, a : scalar_f64, b : scalar_f64, n : scalar_u32) {
    if (gtid < n) { y[gtid] = a * x[gtid] + b * y[gtid]; }
}
"""
n = 1 << 25
with Runtime(devices=[0]) as rt:
    d = rt.get_all_devices().get()[0]
    lib = _native.load()
    X, Y = d.create_buffer(n * 8).get(), d.create_buffer(n * 8).get()
    X.enqueue_write(0, np.random.default_rng(0).random(n))
    p = d.create_program_with_source(SRC).get()
    p.build("axpby").get()
    g = ((n + 255) // 256, 1, 1), (256, 1, 1)
    for _ in range(5):
        p.run([Y, X, 0.5, 0.25, n], "axpby", *g)
    st = rt.device_objects()[0].stream(0)
    e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
    lib.ofl_event_create(0, ctypes.byref(e0))
    lib.ofl_event_create(0, ctypes.byref(e1))
    K = 200
    lib.ofl_event_record(e0, st.ptr)
    for _ in range(K):
        p.run([Y, X, 0.5, 0.25, n], "axpby", *g)
    lib.ofl_event_record(e1, st.ptr)
    ms = ctypes.c_float()
    lib.ofl_event_elapsed_ms(e0, e1, ctypes.byref(ms))
    t = ms.value / K
    print(f"NVRTC axpby 2^25 f64: {t * 1e3:.1f} us/launch, {24 * n / (t * 1e-3) / 1e9:.1f} GB/s")
