"""Per-call host cost of the device API at small sizes (1000 back-to-back
calls, wall clock): the Python wrapper + ctypes + launch."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2510_01190_b200 import device as dev  # noqa: E402

nx = ny = 128
g = [torch.randn(nx * ny, device="cuda", dtype=torch.float64) for _ in range(2)] + \
    [torch.rand(nx * ny, device="cuda", dtype=torch.float64) for _ in range(2)]
err = torch.zeros(1, dtype=torch.int32, device="cuda")
outs = {k: torch.empty(nx * ny, device="cuda", dtype=torch.float64) for k in dev.ALL_OUTPUTS}
for label, kw in (("fresh outputs", {}), ("out= given", {"out": outs})):
    for _ in range(50):
        dev.propagate2d(*g, nx, ny, 1.0, 1.0, 0.0, check=err, **kw)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(1000):
        dev.propagate2d(*g, nx, ny, 1.0, 1.0, 0.0, check=err, **kw)
    torch.cuda.synchronize()
    print(f"propagate2d 128^2 fp64, {label}: {(time.perf_counter() - t) * 1e3:.1f} us per call")
