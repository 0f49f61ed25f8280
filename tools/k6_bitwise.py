"""Dump the fused Red Sea chain (K6) outputs on a few shapes with the library
in DIVUQ_LIB_PATH (A/B bitwise checks of gradfused rewrites)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2510_01190_b200 import device as dev  # noqa: E402

rng = np.random.default_rng(5)
out = {}
for m, nx, ny in ((20, 1024, 256), (7, 132, 37), (3, 129, 40), (2, 68, 17)):
    mem = torch.from_numpy(rng.normal(0, 3, (m, 2, nx * ny)).astype(np.float32)).cuda()
    o = dev.gradient_ensemble_divergence2d(mem, nx, ny, 0.5, 0.7, 0.05, moments=True)
    for k, v in o.items():
        out[f"{m}_{nx}_{ny}_{k}"] = v.cpu().numpy()
np.savez(sys.argv[1], **out)
