"""Quick probe: triad GB/s through the API at N=2^25 (dev helper)."""
import ctypes, sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_1810_11482_b200 import Runtime, _native
from paper_1810_11482_b200.bindings import kernel_source

n = 1 << 25
with Runtime(devices=[0]) as rt:
    dev = rt.get_all_devices().get()[0]
    A, B, C = (dev.create_buffer(n * 8).get() for _ in range(3))
    rng = np.random.default_rng(1)
    b = rng.random(n); c = rng.random(n)
    B.enqueue_write(0, b.tobytes()); C.enqueue_write(0, c.tobytes())
    p = dev.create_program_with_source(kernel_source("stream")).get(); p.build("triad").get()
    args = [A, B, C, 3.0, n]; grid = ((n + 255) // 256, 1, 1); blk = (256, 1, 1)
    for _ in range(5): p.run(args, "triad", grid, blk)
    dev.synchronize().get()
    lib = _native.load()
    st = rt.device_objects()[0].stream(0)
    e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
    lib.ofl_event_create(0, ctypes.byref(e0)); lib.ofl_event_create(0, ctypes.byref(e1))
    K = 200
    lib.ofl_event_record(e0, st.ptr)
    t0 = time.perf_counter()
    for _ in range(K): p.run(args, "triad", grid, blk)
    t1 = time.perf_counter()
    lib.ofl_event_record(e1, st.ptr)
    ms = ctypes.c_float()
    lib.ofl_event_elapsed_ms(e0, e1, ctypes.byref(ms))
    print(f"triad: {ms.value/K*1e3:.1f} us/launch, {24*n*K/(ms.value*1e-3)/1e9:.1f} GB/s; host enqueue {(t1-t0)/K*1e6:.2f} us/op")
    got = np.frombuffer(A.enqueue_read(0, n * 8).get(), np.float64)
    print("bitexact:", np.array_equal(got, b + 3.0 * c))
