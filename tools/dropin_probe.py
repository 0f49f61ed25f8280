"""Time the drop-in (numpy in / numpy out) API on the GPU box at the sizes the
SURVEY probed the reference at (SURVEY 8a / BASELINE.md 3), host copies included."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import paper_2510_01190_b200 as d  # noqa: E402


def best(fn, runs=5):
    fn()
    ts = []
    for _ in range(runs):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts)


rng = np.random.default_rng(1)
g = d.UniformGrid2(1024, 1024)
n = g.n_vertices
model = d.GaussianVectorField(g, rng.normal(0, 2, n), rng.normal(0, 2, n),
                              rng.uniform(0.05, 0.6, n), rng.uniform(0.05, 0.6, n))
members = tuple(d.VectorField2(g, rng.normal(size=n), rng.normal(size=n)) for _ in range(20))
ens = d.Ensemble2(g, members)
fld = d.propagate_divergence(model)
g2 = d.UniformGrid2(256, 256)
n2 = g2.n_vertices
model2 = d.GaussianVectorField(g2, rng.normal(0, 2, n2), rng.normal(0, 2, n2),
                               rng.uniform(0.05, 0.6, n2), rng.uniform(0.05, 0.6, n2))
rows = [
    ("propagate_divergence 1024^2 fp64", lambda: d.propagate_divergence(model), 189e-3),
    ("fit_gaussian 1024^2 x 20", lambda: d.fit_gaussian(ens), 408e-3),
    ("source_probability (tail map) 1024^2", lambda: d.source_probability(fld, 0.0), 89e-3),
    ("mc_divergence 256^2 N=2000 (Philox)", lambda: d.mc_divergence(model2, d.McConfig(2000, seed=5)), 8.67),
    ("mc_divergence 256^2 N=2000 (reference stream)",
     lambda: d.mc_divergence(model2, d.McConfig(2000, seed=5), stream="reference"), 8.67),
]
for name, fn, ref_s in rows:
    t = best(fn)
    print(f"{name:48s} {t * 1e3:9.2f} ms   reference probe {ref_s * 1e3:9.1f} ms   x{ref_s / t:8.1f}")
