"""Drop-in call latency across grid sizes (best of 7 after warm-up), to A/B
the small-call pinned bounce arena (run twice: DIVUQ_BOUNCE_MAX_KB=0 and the
default).  propagate_divergence (4 arrays in, 2 out), source_probability
(2 in, 1 out), lcp (2 in, cells out)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_01190_b200 as d  # noqa: E402


def best(fn, runs=7):
    fn()
    ts = []
    for _ in range(runs):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3


rng = np.random.default_rng(1)
print(f"DIVUQ_BOUNCE_MAX_KB={os.environ.get('DIVUQ_BOUNCE_MAX_KB', 'default')}")
for side in (68, 128, 256, 500, 724, 1024, 1448):
    n = side * side
    g = d.UniformGrid2(side, side)
    m = d.GaussianVectorField(g, rng.normal(size=n), rng.normal(size=n), rng.uniform(0.1, 1, n),
                              rng.uniform(0.1, 1, n))
    f = d.propagate_divergence(m)
    tp = best(lambda: d.propagate_divergence(m))
    ts = best(lambda: d.source_probability(f, 0.0))
    tl = best(lambda: d.lcp(f, 0.0))
    print(f"{side:5d}^2 ({n * 8 / 2**20:6.2f} MB/array): propagate {tp:7.3f} ms  P-map {ts:7.3f} ms  lcp {tl:7.3f} ms")
