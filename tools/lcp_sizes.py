"""lcp2d fp64 over sizes (device-side time, validation word on)."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from paper_2510_01190_b200 import device as dev  # noqa: E402
from shape_sweep import timeit, PEAK, ERR  # noqa: E402

for nx, ny in ((1024, 1024), (2048, 2048), (4096, 4096), (1000, 700), (8192, 2048)):
    mu = torch.randn(nx * ny, device="cuda", dtype=torch.float64)
    sg = torch.rand(nx * ny, device="cuda", dtype=torch.float64)
    ms = timeit(lambda: dev.lcp2d(mu, sg, nx, ny, 0.0, check=ERR), reps=20)
    print(f"lcp2d fp64 {nx}x{ny}: {ms * 1e3:8.1f} us  {24 * (nx - 1) * (ny - 1) / ms / 1e6 / PEAK * 100:5.1f} % HBM")
