"""One propagate3d launch on an unaligned shape (the flat 1D-TMA K2) for ncu."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2510_01190_b200 import device as dev  # noqa: E402

nx, ny, nz = int(sys.argv[1]) if len(sys.argv) > 1 else 511, 512, 512
n = nx * ny * nz
f = [torch.randn(n, device="cuda") for _ in range(3)] + [torch.rand(n, device="cuda") * 0.3 + 0.05 for _ in range(3)]
out = {k: torch.empty(n, device="cuda") for k in dev.ALL_OUTPUTS}
err = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(4):
    dev.propagate3d(*f, nx, ny, nz, 1.0, 1.0, 1.0, 0.0, out=out, check=err)
torch.cuda.synchronize()
