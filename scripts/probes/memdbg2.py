import sys, time
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from paper_1810_11482_b200 import Runtime, OutOfMemoryError
from test_gpu_memory import _long_heat
with Runtime(devices=[0]) as rt:
    dev = rt.get_all_devices().get()[0]
    if len(sys.argv) > 1:
        try:
            dev.create_buffer(1 << 40).get()
        except OutOfMemoryError:
            print("oom as expected")
    for trial in range(3):
        s1 = dev.create_stream()
        tok, keep = _long_heat(dev, s1)
        t0 = time.perf_counter()
        tmp = dev.create_buffer(1 << 20).get()
        t1 = time.perf_counter()
        rt.registry.unregister(tmp.gid); del tmp
        t2 = time.perf_counter()
        fresh = dev.create_buffer(32 << 20).get()
        t3 = time.perf_counter()
        print(trial, "alloc1 %.2f ms free %.2f ms alloc2 %.2f ms done=%s" % ((t1-t0)*1e3, (t2-t1)*1e3, (t3-t2)*1e3, tok.done()), flush=True)
        tok.get()
