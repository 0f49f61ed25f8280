"""propagate2d fp64/fp32 over sizes: the 2D kernels' HBM fraction."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from paper_2510_01190_b200 import device as dev  # noqa: E402
from shape_sweep import timeit, PEAK, ERR  # noqa: E402

for dt, bpp in ((torch.float64, 64), (torch.float32, 32)):
    for nx, ny in ((128, 128), (512, 512), (1024, 1024), (2048, 2048), (4096, 4096), (1001, 999)):
        g = [torch.randn(nx * ny, device="cuda", dtype=dt) for _ in range(2)] + \
            [torch.rand(nx * ny, device="cuda", dtype=dt) for _ in range(2)]
        ms = timeit(lambda: dev.propagate2d(*g, nx, ny, 1.0, 1.0, 0.0, check=ERR))
        print(f"propagate2d {str(dt)[6:]} {nx}x{ny}: {ms * 1e3:8.1f} us  {bpp * nx * ny / ms / 1e6 / PEAK * 100:5.1f} % HBM")
