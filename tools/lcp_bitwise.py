"""Dump lcp2d / propagate_lcp2d outputs on a mixed field (sigma = 0 patches,
tiny sigma, exact zeros of theta - mu) with the library in DIVUQ_LIB_PATH
(A/B bitwise checks of LCP kernel rewrites)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2510_01190_b200 import device as dev  # noqa: E402

rng = np.random.default_rng(11)
out = {}
for nx, ny in ((1031, 517), (1032, 517)):   # register kernel / TMA kernel
    n = nx * ny
    mu = rng.normal(0, 1.5, n)
    sg = rng.uniform(0, 2, n)
    sg[rng.random(n) < 0.05] = 0.0
    sg[rng.random(n) < 0.01] = 1e-310
    mu[rng.random(n) < 0.02] = 0.25
    m, s = torch.from_numpy(mu).cuda(), torch.from_numpy(sg).cuda()
    for t in (0.0, 0.25, -1.0):
        out[f"{nx}_{t}"] = dev.lcp2d(m, s, nx, ny, t).cpu().numpy()
n = nx * ny
g = [torch.from_numpy(x).cuda() for x in (rng.normal(size=n), rng.normal(size=n),
                                          rng.uniform(0, 1, n), rng.uniform(0, 1, n))]
f = dev.propagate_lcp2d(*g, nx, ny, 0.7, 1.3, 0.1, moments=False)
out["fused"] = f["lcp"].cpu().numpy()
np.savez(sys.argv[1], **out)
