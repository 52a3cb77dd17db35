"""The reference's own runtime, unmodified, driving the B200s: attach this
package's CUDA locality to an ``offloadrt.Runtime`` (the drop-in boundary,
INTEGRATION.md Option B) and run the reference's stencil kernel through the
reference's handles and when_all.

    PYTHONPATH=baseline/_ref python examples/reference_runtime_on_b200.py
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
from offloadrt import Runtime, when_all  # noqa: E402  (the reference package)
from offloadrt.bench import kernel_source  # noqa: E402

from paper_1810_11482_b200.offloadrt_backend import attach  # noqa: E402


def main(n: int = 1 << 20) -> bool:
    rt = Runtime(backend="host")                  # the reference runtime
    try:
        attach(rt)                                # B200s join as one more locality
        dev = rt.get_all_devices().get()[-1]      # a reference DeviceHandle on cuda0
        x = np.random.default_rng(0).random(n)
        X, Y = dev.create_buffer(n * 8).get(), dev.create_buffer(n * 8).get()
        prog = dev.create_program_with_source(kernel_source("stencil")).get()
        when_all([X.enqueue_write(0, x.tobytes()), prog.build("stencil")]).get()
        prog.run([X, Y, n], "stencil", ((n + 255) // 256, 1, 1), (256, 1, 1)).get()
        y = np.frombuffer(Y.enqueue_read(0, n * 8).get(), np.float64)
        expect = x.copy()
        expect[1:-1] = 0.5 * x[:-2] + x[1:-1] + 0.5 * x[2:]
        ok = np.array_equal(y, expect)
        print(f"reference runtime -> {dev.info.name}: stencil over {n} cells "
              f"{'matches' if ok else 'DIFFERS FROM'} numpy")
        return ok
    finally:
        rt.close()


if __name__ == "__main__":
    assert main()
