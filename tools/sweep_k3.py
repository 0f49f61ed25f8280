"""Time K3 (config-4 slab: 1024^2 x 128 planes, M=16, fp32) under launch knobs (env read per launch)."""
import itertools
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_01190_b200 import configs, device as dev  # noqa: E402

nx = ny = 1024
nzl = int(os.environ.get("K3_NZL", "128"))
mem = configs.config4_slab(0, nzl, nx, ny, 1024, 16, 104)
out = {k: torch.empty(nx * ny * nzl, device="cuda") for k in dev.ALL_OUTPUTS}
knobs = {}
for spec in os.environ.get("SWEEP", "DIVUQ_K3_SYNC_W=0,2").split(";"):
    k, v = spec.split("=")
    knobs[k] = v.split(",")
byts = 208 * nx * ny * nzl
for combo in itertools.product(*knobs.values()):
    for k, v in zip(knobs, combo):
        os.environ[k] = v
    reps = 1 if os.environ.get("NCU") else 10
    for _ in range(1 if reps == 1 else 2):
        dev.ensemble_divergence3d(mem, nx, ny, nzl, 1.0, 1.0, 1.0, 0.1, z0=0, nz_global=nzl,
                                  out=out, check=False)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        dev.ensemble_divergence3d(mem, nx, ny, nzl, 1.0, 1.0, 1.0, 0.1, z0=0, nz_global=nzl,
                                  out=out, check=False)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    print(dict(zip(knobs, combo)), f"{ms:.3f} ms  {byts / ms / 1e6:.0f} GB/s", flush=True)
