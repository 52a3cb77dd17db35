import ctypes, os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1810_11482_b200 import Runtime, _native
from paper_1810_11482_b200.bindings import kernel_source
n = 1 << 28
with Runtime(devices=[0]) as rt:
    d = rt.get_all_devices().get()[0]; lib = _native.load()
    X, Y, Z = d.create_buffer(n * 8).get(), d.create_buffer(n * 8).get(), d.create_buffer(n * 8).get()
    X.enqueue_write(0, np.random.default_rng(0).random(n))
    p = d.create_program_with_source(kernel_source("stream")).get(); p.build("copy").get()
    g = ((n + 255) // 256, 1, 1), (256, 1, 1)
    st = rt.device_objects()[0].stream(0)
    e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
    lib.ofl_event_create(0, ctypes.byref(e0)); lib.ofl_event_create(0, ctypes.byref(e1))
    for mode in ("same", "pingpong"):
        K = 50
        for k in range(4): p.run([Y, X, n], "copy", *g)
        lib.ofl_event_record(e0, st.ptr)
        for k in range(K):
            if mode == "same": p.run([Y, X, n], "copy", *g)
            else: p.run([Y, X, n] if k % 2 == 0 else [X, Y, n], "copy", *g)
        lib.ofl_event_record(e1, st.ptr)
        ms = ctypes.c_float(); lib.ofl_event_elapsed_ms(e0, e1, ctypes.byref(ms))
        t = ms.value / K
        print(f"copy 2^28 {mode}: {t*1e3:.1f} us, {16*n/(t*1e-3)/1e9:.1f} GB/s")
