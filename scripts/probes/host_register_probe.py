"""Cost of page-locking pageable memory in place (cudaHostRegister) vs the
staged copy: would DMA-ing straight from a registered numpy array beat the
pinned staging ring for large pageable writes?"""
import time

import numpy as np
import torch

cr = torch.cuda.cudart()
n = 256 << 20
for trial in range(3):
    a = np.ones(n, np.uint8)  # pageable, faulted in
    t0 = time.perf_counter()
    r = cr.cudaHostRegister(a.ctypes.data, n, 0)
    t1 = time.perf_counter()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    src = torch.from_numpy(a)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    d.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    cr.cudaHostUnregister(a.ctypes.data)
    t4 = time.perf_counter()
    print(f"register {n / (t1 - t0) / 1e9:.1f} GB/s ({(t1 - t0) * 1e3:.1f} ms, rc={r}), "
          f"dma {n / (t3 - t2) / 1e9:.1f} GB/s, unregister {(t4 - t3) * 1e3:.1f} ms, "
          f"total {n / (t4 - t0 - (t2 - t1)) / 1e9:.1f} GB/s")
