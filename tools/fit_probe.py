"""Time K1 (fit_gaussian) on the config-1 ensemble shape: M=20, C=2, 1024^2, fp32 and fp64."""
import sys
import torch
sys.path.insert(0, '.')
import __graft_entry__; __graft_entry__.build()
from paper_2510_01190_b200 import configs, device as dev

nx = ny = 1024
M = 20
m32 = configs.config1_members(nx, ny, M, 101)
m64 = m32.double()
w = torch.empty(256 << 20, dtype=torch.uint8, device='cuda'); r = torch.ones(256 << 20, dtype=torch.uint8, device='cuda')
for name, mem in (("fp32", m32), ("fp64", m64)):
    mu = torch.empty((2, nx * ny), dtype=mem.dtype, device='cuda'); sg = torch.empty_like(mu)
    ts = []
    for it in range(25):
        w.zero_(); r.sum()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); dev.fit_moments(mem, out=(mu, sg), check=False); b.record(); torch.cuda.synchronize()
        if it >= 5: ts.append(a.elapsed_time(b))
    ts.sort(); t = ts[len(ts) // 2]
    byts = mem.numel() * mem.element_size() + 2 * mu.numel() * mu.element_size()
    print(f"{name}: {t*1e3:.1f} us  {byts / t / 1e6:.0f} GB/s")
