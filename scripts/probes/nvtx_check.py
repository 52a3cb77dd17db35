import sys; sys.path.insert(0, '.')
import numpy as np
from paper_1810_11482_b200 import Runtime
with Runtime(devices=[0]) as rt:
    dev = rt.get_all_devices().get()[0]
    n = 1 << 20
    X, Y = dev.create_buffer(n * 8).get(), dev.create_buffer(n * 8).get()
    X.enqueue_write(0, np.random.default_rng(1).random(n)).get()
    p = dev.create_builtin_program().get(); p.build("heat").get()
    p.run([X, Y, n, 200], "heat", (n // 256, 1, 1), (256, 1, 1)).get()
    print("done")
