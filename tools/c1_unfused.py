import sys, torch
sys.path.insert(0, '.')
import __graft_entry__; __graft_entry__.build()
from paper_2510_01190_b200 import configs, device as dev
nx = ny = 1024; M = 20
mem = configs.config1_members(nx, ny, M, 101)
w = torch.empty(256 << 20, dtype=torch.uint8, device='cuda'); r = torch.ones(256 << 20, dtype=torch.uint8, device='cuda')
mu = torch.empty((2, nx*ny), device='cuda'); sg = torch.empty_like(mu)
out = {k: torch.empty(nx*ny, device='cuda') for k in ('mu', 'sigma', 'p_src')}
def step_unfused():
    dev.fit_moments(mem, out=(mu, sg), check=False)
    dev.propagate2d(mu[0], mu[1], sg[0], sg[1], nx, ny, 1.0, 1.0, 0.0, outputs=('mu','sigma','p_src'), out=out, check=False)
def step_fused():
    dev.ensemble_divergence2d(mem, nx, ny, 1.0, 1.0, 0.0, outputs=('mu','sigma','p_src'), out=out, check=False)
def step_fit():
    dev.fit_moments(mem, out=(mu, sg), check=False)
for name, fn in (('fused', step_fused), ('unfused', step_unfused), ('fit only', step_fit)):
    ts = []
    for it in range(25):
        w.zero_(); r.sum()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        if it >= 5: ts.append(a.elapsed_time(b))
    ts.sort(); print(name, "median %.1f us" % (ts[len(ts)//2]*1e3))
