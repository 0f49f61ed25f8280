"""Where a small host-entry call spends its time: torch.profiler (CUPTI) over
200 calls of divuq_host_propagate2d_f64 at 128^2 with pinned buffers (the
bench's config-0 e2e call), runtime API calls and GPU activities summed."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_2510_01190_b200._lib import lib  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 128
n = side * side
rng = np.random.default_rng(0)
arrs = [rng.normal(size=n), rng.normal(size=n), rng.uniform(0.1, 1, n), rng.uniform(0.1, 1, n)]
host_in = [torch.from_numpy(a).pin_memory() for a in arrs]
host_out = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(4)]


def call():
    st = lib.divuq_host_propagate2d_f64(*(t.data_ptr() for t in host_in), side, side, 1.0, 1.0, 0.0,
                                        *(t.data_ptr() for t in host_out), 0)
    assert st == 0


for _ in range(50):
    call()
t0 = time.perf_counter()
for _ in range(200):
    call()
print(f"{side}^2 pinned: {(time.perf_counter() - t0) / 200 * 1e6:.1f} us per call")
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(200):
        call()
print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=25))
