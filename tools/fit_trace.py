"""fit_gaussian 1024^2 x 20 drop-in (168 MB pageable in): wall time of the C
entry alone, then torch.profiler (CUPTI) over 5 calls: where the host waits."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import torch  # noqa: E402

from paper_2510_01190_b200._lib import lib  # noqa: E402

M, N = 20, 1024 * 1024
rng = np.random.default_rng(0)
stacked = rng.normal(size=(M, 2, N))
mu = np.empty((2, N))
sg = np.empty((2, N))
p = lambda a: a.__array_interface__["data"][0]  # noqa: E731


def call():
    assert lib.divuq_host_fit_gaussian_f64(p(stacked), M, 2, N, p(mu), p(sg), 0) == 0


call()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    call()
    ts.append(time.perf_counter() - t0)
print(f"C entry: best {min(ts) * 1e3:.2f} ms, all {[round(t * 1e3, 2) for t in ts]}")
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        call()
print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=8))
print(prof.key_averages().table(sort_by="self_cuda_time_total", row_limit=6))

# the same call through the drop-in API (types, output records)
import paper_2510_01190_b200 as d  # noqa: E402

g = d.UniformGrid2(1024, 1024)
ens = d.Ensemble2(g, tuple(d.VectorField2(g, stacked[k, 0], stacked[k, 1]) for k in range(M)))
d.fit_gaussian(ens)
for label, fn in (("drop-in fit_gaussian", lambda: d.fit_gaussian(ens)),
                  ("np.empty x2 + C entry", lambda: (np.empty((2, N)), np.empty((2, N)), call()))):
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    print(f"{label}: best {min(ts) * 1e3:.2f} ms, all {[round(t * 1e3, 2) for t in ts]}")
