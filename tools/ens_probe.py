"""A few ensemble_divergence2d launches on an unaligned shape (ncu launch list)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_01190_b200 import device as dev  # noqa: E402

nx, ny, m = int(sys.argv[1]) if len(sys.argv) > 1 else 1023, 1024, 20
mem = torch.randn(m, 2, nx * ny, device="cuda")
err = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(3):
    dev.ensemble_divergence2d(mem, nx, ny, 1.0, 1.0, 0.0, check=err)
torch.cuda.synchronize()
