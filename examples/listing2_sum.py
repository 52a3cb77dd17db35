"""The paper's workflow listing (arXiv 1810.11482, PAPER.md "Workflow of
HPXCL") on this runtime: find the devices, create buffers and start the
writes, start the kernel build, gate the launch on all of them with one
when_all, run, read the result back.  Every call returns a future; nothing
blocks until the gate.

    python examples/listing2_sum.py          # on a machine with a B200
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_1810_11482_b200 import Runtime, when_all  # noqa: E402

KERNELS = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "paper_1810_11482_b200", "kernels")


def main(n: int = 1000) -> int:
    with Runtime() as rt:
        devices = rt.get_all_devices(10, 0).get()         # compute capability >= 10.0
        dev = devices[0]
        data = np.ones(n, dtype=np.uint32)

        futures = []
        inp = dev.create_buffer(n * 4).get()
        futures.append(inp.enqueue_write(0, data))
        res = dev.create_buffer(4).get()
        futures.append(res.enqueue_write(0, np.zeros(1, np.uint32)))
        prog = dev.create_program_with_file(os.path.join(KERNELS, "sum.k")).get()
        futures.append(prog.build("sum"))                 # compiles while the writes run

        when_all(futures).get()                           # the listing's wait_all
        prog.run([inp, res, n], "sum", (1, 1, 1), (32, 1, 1)).get()
        total = int(np.frombuffer(res.enqueue_read_sync(0, 4), np.uint32)[0])
        print(f"sum of {n} ones on {dev.info.name}: {total}")
        return total


if __name__ == "__main__":
    assert main() == 1000
