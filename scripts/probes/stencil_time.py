"""One stencil.k step over 2^28 f64 cells, back-to-back launches ping-ponging
(CUDA events): the single-step kernel's launch-shape sweep
(OFL_STENCIL_VARIANT).  python scripts/probes/stencil_time.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

from paper_1810_11482_b200 import Runtime, _native  # noqa: E402
from paper_1810_11482_b200.bindings import kernel_source  # noqa: E402

n = 1 << 28
with Runtime(devices=[0]) as rt:
    d = rt.get_all_devices().get()[0]
    lib = _native.load()
    X, Y = d.create_buffer(n * 8).get(), d.create_buffer(n * 8).get()
    X.enqueue_write(0, np.random.default_rng(0).random(n))
    p = d.create_program_with_source(kernel_source("stencil")).get()
    p.build("stencil").get()
    g = ((n + 255) // 256, 1, 1), (256, 1, 1)
    for k in range(4):
        p.run([X, Y, n] if k % 2 == 0 else [Y, X, n], "stencil", *g)
    st = rt.device_objects()[0].stream(0)
    e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
    lib.ofl_event_create(0, ctypes.byref(e0))
    lib.ofl_event_create(0, ctypes.byref(e1))
    K = 50
    lib.ofl_event_record(e0, st.ptr)
    for k in range(K):
        p.run([X, Y, n] if k % 2 == 0 else [Y, X, n], "stencil", *g)
    lib.ofl_event_record(e1, st.ptr)
    ms = ctypes.c_float()
    lib.ofl_event_elapsed_ms(e0, e1, ctypes.byref(ms))
    t = ms.value / K
    print(f"variant {os.environ.get('OFL_STENCIL_VARIANT', '0')}: {t * 1e3:.1f} us/step, "
          f"{16 * n / (t * 1e-3) / 1e9:.1f} GB/s")
