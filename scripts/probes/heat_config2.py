"""Config 2 (2^28 f64 x 1000 steps, the `heat` builtin) timed with CUDA
events under whatever OFL_HEAT_* sweep switches are set, checked against
the reference's sha256 (tests/golden/golden_long.json).  One line of JSON.
Used by scripts/heat_sweep.sh (a new process per kernel variant: the
switches are read once per process)."""

import ctypes
import hashlib
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

from paper_1810_11482_b200 import Runtime, _native, pinned_empty  # noqa: E402

n, steps = 1 << 28, 1000
ref = next(c for c in json.load(open(os.path.join(REPO, "tests/golden/golden_long.json")))["heat"]
           if c["n"] == n and c["steps"] == steps)
lib = _native.load()
with Runtime(devices=[0]) as rt:
    d = rt.get_all_devices().get()[0]
    x = pinned_empty(n * 8, np.float64)
    x[:] = np.random.default_rng(ref["seed"]).random(n)
    X, Y = d.create_buffer(n * 8).get(), d.create_buffer(n * 8).get()
    p = d.create_builtin_program().get()
    p.build("heat").get()
    st = rt.device_objects()[0].stream(0)
    e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
    lib.ofl_event_create(0, ctypes.byref(e0))
    lib.ofl_event_create(0, ctypes.byref(e1))
    times = []
    for rep in range(3):
        X.enqueue_write(0, x)
        lib.ofl_event_record(e0, st.ptr)
        p.run([X, Y, n, steps], "heat", (n // 256, 1, 1), (256, 1, 1))
        lib.ofl_event_record(e1, st.ptr)
        ms = ctypes.c_float()
        _native.check(lib.ofl_event_elapsed_ms(e0, e1, ctypes.byref(ms)), "elapsed")
        times.append(ms.value)
    out = pinned_empty(n * 8, np.float64)
    (X if steps % 2 == 0 else Y).enqueue_read_into(0, out).get()
    ok = hashlib.sha256(memoryview(out).cast("B")).hexdigest() == ref["sha256"]
    env = {k: v for k, v in os.environ.items() if k.startswith("OFL_HEAT")}
    print(json.dumps({"env": env, "ms": [round(t, 3) for t in times], "best_ms": round(min(times), 3),
                      "bitexact_vs_reference": ok}), flush=True)
