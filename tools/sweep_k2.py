"""Time K2 (config 3, 512^3 fp32) under different launch knobs (env vars read per launch)."""
import itertools
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_01190_b200 import configs, device as dev  # noqa: E402

n = 512
f = configs.config3_slab(0, n)
out = {k: torch.empty(n**3, device="cuda") for k in dev.ALL_OUTPUTS}
knobs = {}
for spec in os.environ.get("SWEEP", "DIVUQ_PHASE=0,1,2,4").split(";"):
    k, v = spec.split("=")
    knobs[k] = v.split(",")
for combo in itertools.product(*knobs.values()):
    for k, v in zip(knobs, combo):
        os.environ[k] = v
    reps = 1 if os.environ.get("NCU") else 20
    for _ in range(1 if reps == 1 else 3):
        dev.propagate3d(*f, n, n, n, out=out, check=False)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        dev.propagate3d(*f, n, n, n, out=out, check=False)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    print(dict(zip(knobs, combo)), f"{ms:.3f} ms  {40 * n**3 / ms / 1e6:.0f} GB/s", flush=True)
