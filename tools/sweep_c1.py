"""Time the 2D fused ensemble kernel (config 1) under launch knobs (env vars read per launch).
L2 is flushed before every launch, as in bench.py."""
import itertools
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_01190_b200 import configs, device as dev  # noqa: E402

nx = ny = int(os.environ.get("C1_N", "1024"))
M = int(os.environ.get("C1_M", "20"))
mem = configs.config1_members(nx, ny, M, 101)
out = {k: torch.empty(nx * ny, device="cuda") for k in ("mu", "sigma", "p_src")}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
drain = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
MODE = os.environ.get("FLUSH", "drain")
knobs = {}
for spec in os.environ.get("SWEEP", "DIVUQ_TMA_TY=0,8,10,12,14").split(";"):
    k, v = spec.split("=")
    knobs[k] = v.split(",")
byts = (M * 2 * 4 + 12) * nx * ny
for combo in itertools.product(*knobs.values()):
    for k, v in zip(knobs, combo):
        os.environ[k] = v
    ts = []
    for it in range(23):
        flush.zero_()
        if MODE == "drain":
            drain.sum(dtype=torch.int64)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        dev.ensemble_divergence2d(mem, nx, ny, 1.0, 1.0, 0.0, outputs=("mu", "sigma", "p_src"), out=out,
                                  check=False)
        e.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(s.elapsed_time(e))
    ms = sum(ts) / len(ts)
    print(dict(zip(knobs, combo)), f"{ms * 1e3:.1f} us  {byts / ms / 1e6:.0f} GB/s  min {min(ts) * 1e3:.1f} us",
          flush=True)
