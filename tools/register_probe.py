"""Can the drop-in path pin the caller's pageable array in place instead of
copying it through a staging buffer?  Time cudaHostRegister + one DMA +
cudaHostUnregister of a 168 MB numpy array against the staged copy rate."""
import time

import numpy as np
import torch

cr = torch.cuda.cudart()
for mb in (8, 32, 168):
    a = np.random.default_rng(0).normal(size=mb * (1 << 20) // 8)
    d = torch.empty(a.size, dtype=torch.float64, device="cuda")
    h = torch.from_numpy(a)
    for rep in range(3):
        t0 = time.perf_counter()
        r = cr.cudaHostRegister(a.__array_interface__["data"][0], a.nbytes, 0)
        t1 = time.perf_counter()
        d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        cr.cudaHostUnregister(a.__array_interface__["data"][0])
        t3 = time.perf_counter()
        print(f"{mb:4d} MB rep {rep}: register {1e3 * (t1 - t0):7.2f} ms  DMA {1e3 * (t2 - t1):7.2f} ms "
              f"({a.nbytes / (t2 - t1) / 1e9:5.1f} GB/s)  unregister {1e3 * (t3 - t2):6.2f} ms  rc={r}")
    t0 = time.perf_counter()
    d.copy_(h)
    torch.cuda.synchronize()
    print(f"{mb:4d} MB pageable torch copy {1e3 * (time.perf_counter() - t0):7.2f} ms")
