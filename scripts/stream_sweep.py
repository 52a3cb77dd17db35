"""Tuning sweep of STREAM launch shapes (OFL_STREAM_VARIANT) on one B200."""
import ctypes, os, subprocess, sys, json
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

def probe():
    import numpy as np
    from paper_1810_11482_b200 import Runtime, _native
    from paper_1810_11482_b200.bindings import kernel_source
    lib = _native.load()
    n = 1 << 25
    out = {}
    with Runtime(devices=[0]) as rt:
        dev = rt.get_all_devices().get()[0]
        A, B, C = (dev.create_buffer(n * 8).get() for _ in range(3))
        B.enqueue_write(0, np.ones(n)); C.enqueue_write(0, np.ones(n))
        p = dev.create_program_with_source(kernel_source("stream")).get()
        st = rt.device_objects()[0].stream(0)
        e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
        lib.ofl_event_create(0, ctypes.byref(e0)); lib.ofl_event_create(0, ctypes.byref(e1))
        for op, nb, args in (("triad", 24, [A, B, C, 3.0, n]), ("copy", 16, [A, B, n])):
            p.build(op).get()
            for _ in range(20): p.run(args, op, (n // 256, 1, 1), (256, 1, 1))
            K = 400
            lib.ofl_event_record(e0, st.ptr)
            for _ in range(K): p.run(args, op, (n // 256, 1, 1), (256, 1, 1))
            lib.ofl_event_record(e1, st.ptr)
            ms = ctypes.c_float(); lib.ofl_event_elapsed_ms(e0, e1, ctypes.byref(ms))
            out[op] = round(nb * n * K / (ms.value * 1e-3) / 1e9, 1)
    print(json.dumps(out))

if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "probe":
        probe(); sys.exit(0)
    res = {}
    for v in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else range(16))]:
        env = dict(os.environ, OFL_STREAM_VARIANT=str(v))
        r = subprocess.run([sys.executable, __file__, "probe"], env=env, capture_output=True, text=True)
        res[v] = r.stdout.strip() or r.stderr[-300:]
        print(v, res[v], flush=True)
