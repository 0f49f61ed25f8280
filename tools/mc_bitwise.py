"""Dump mc_divergence2d outputs for a config-2-like case with the library in
DIVUQ_LIB_PATH (A/B bitwise checks of MC kernel rewrites)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2510_01190_b200 import device as dev  # noqa: E402

rng = np.random.default_rng(7)
nx = ny = 256
n = nx * ny
a = [rng.normal(0, 2, n), rng.normal(0, 2, n), rng.uniform(0.0, 0.6, n), rng.uniform(0.0, 0.6, n)]
t = [torch.from_numpy(x).cuda() for x in a]
m, s = dev.mc_divergence2d(*t, nx, ny, 0.1, 0.2, 777, 1234)
np.savez(sys.argv[1], mean=m.cpu().numpy(), std=s.cpu().numpy())
