"""Mandelbrot config 3 kernel time + SM clock under load (NVML), for the
fused/unfused sweep: OFL_MANDEL_FUSED=0/1 python scripts/probes/mandel_clock.py"""
import ctypes
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import pynvml  # noqa: E402

from paper_1810_11482_b200 import Runtime, _native  # noqa: E402
from paper_1810_11482_b200.bindings import kernel_source  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
with Runtime(devices=[0]) as rt:
    d = rt.get_all_devices().get()[0]
    lib = _native.load()
    w, hh = 7680, 4320
    O = d.create_buffer(w * hh * 4).get()
    p = d.create_program_with_source(kernel_source("mandelbrot")).get()
    p.build("mandelbrot").get()
    args = [O, w, hh, -2.0, 1.0, -1.5, 1.5, 4.0, 2000]
    g = ((w * hh + 255) // 256, 1, 1), (256, 1, 1)
    for _ in range(3):
        p.run(args, "mandelbrot", *g)
    d.synchronize().get()
    st = rt.device_objects()[0].stream(0)
    e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
    lib.ofl_event_create(0, ctypes.byref(e0))
    lib.ofl_event_create(0, ctypes.byref(e1))
    clocks, power, stop = [], [], threading.Event()

    def sample():
        while not stop.is_set():
            clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            power.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000)
            time.sleep(0.005)

    th = threading.Thread(target=sample)
    th.start()
    K = int(os.environ.get("K", "50"))
    lib.ofl_event_record(e0, st.ptr)
    for _ in range(K):
        p.run(args, "mandelbrot", *g)
    lib.ofl_event_record(e1, st.ptr)
    ms = ctypes.c_float()
    lib.ofl_event_elapsed_ms(e0, e1, ctypes.byref(ms))
    stop.set()
    th.join()
    c = sorted(clocks)
    print(f"FUSED={os.environ.get('OFL_MANDEL_FUSED', '1')} K={K}: {ms.value / K:.3f} ms/launch, "
          f"sm clock median {c[len(c) // 2]} MHz (min {c[0]}), power max {max(power):.0f} W")
