"""K6 on an unaligned shape (register-staged variant) for A/B timing."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from paper_2510_01190_b200 import device as dev  # noqa: E402
from shape_sweep import timeit, PEAK, ERR  # noqa: E402

for nx in (1023, 2047):
    ny, m = 1024, 20
    mem = torch.randn(m, 2, nx * ny, device="cuda")
    ms = timeit(lambda: dev.gradient_ensemble_divergence2d(mem, nx, ny, 1.0, 1.0, 0.0, check=ERR))
    print(f"K6 M=20 {nx}x{ny}: {ms * 1e3:.1f} us  {(160 + 16) * nx * ny / ms / 1e6 / PEAK * 100:.1f} % HBM")
