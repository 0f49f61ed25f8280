"""Time the drop-in (numpy in / numpy out) API against the unmodified
reference (baseline/_ref) on the SAME box, same inputs, at the sizes SURVEY
8a probed (host copies included on our side; the reference serial and with
ParallelConfig(threads=os.cpu_count()) where it takes one).

    python tools/dropin_probe.py        # on the GPU box, after build()
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import divuq as ref  # noqa: E402  (the reference's own pip install)
from divuq.lcp import _tail_probs  # noqa: E402

import paper_2510_01190_b200 as d  # noqa: E402


def best(fn, runs=5):
    fn()
    ts = []
    for _ in range(runs):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts)


threads = os.cpu_count() or 1
rng = np.random.default_rng(1)
arrs = [rng.normal(0, 2, 1024 * 1024), rng.normal(0, 2, 1024 * 1024),
        rng.uniform(0.05, 0.6, 1024 * 1024), rng.uniform(0.05, 0.6, 1024 * 1024)]
mem = [(rng.normal(size=1024 * 1024), rng.normal(size=1024 * 1024)) for _ in range(20)]
a2 = [rng.normal(0, 2, 256 * 256), rng.normal(0, 2, 256 * 256),
      rng.uniform(0.05, 0.6, 256 * 256), rng.uniform(0.05, 0.6, 256 * 256)]
ours = {}
theirs = {}
for pkg, out in ((d, ours), (ref, theirs)):
    g = pkg.UniformGrid2(1024, 1024)
    out["model"] = pkg.GaussianVectorField(g, *arrs)
    out["ens"] = pkg.Ensemble2(g, tuple(pkg.VectorField2(g, u, v) for u, v in mem))
    out["fld"] = pkg.propagate_divergence(out["model"])
    out["model2"] = pkg.GaussianVectorField(pkg.UniformGrid2(256, 256), *a2)
    # the paper's own grid sizes: wind 68^2 x 15, Red Sea 500^2 x 20
    for k, side, m in (("wind", 68, 15), ("redsea", 500, 20)):
        gk = pkg.UniformGrid2(side, side)
        nk = side * side
        out[k] = pkg.GaussianVectorField(gk, *(a[:nk] for a in arrs))
        out[k + "_ens"] = pkg.Ensemble2(gk, tuple(pkg.VectorField2(gk, u[:nk], v[:nk]) for u, v in mem[:m]))
        out[k + "_fld"] = pkg.propagate_divergence(out[k])
pc = ref.ParallelConfig(threads=threads)
rows = [
    ("propagate_divergence 1024^2 fp64", lambda: d.propagate_divergence(ours["model"]),
     lambda: ref.propagate_divergence(theirs["model"]), lambda: ref.propagate_divergence(theirs["model"], pc)),
    ("fit_gaussian 1024^2 x 20", lambda: d.fit_gaussian(ours["ens"]), lambda: ref.fit_gaussian(theirs["ens"]),
     None),
    ("P(div > 0) map 1024^2", lambda: d.source_probability(ours["fld"], 0.0),
     lambda: _tail_probs(theirs["fld"].mu, theirs["fld"].sigma, 0.0), None),
    ("lcp 1024^2", lambda: d.lcp(ours["fld"], 0.0), lambda: ref.lcp(theirs["fld"], 0.0),
     lambda: ref.lcp(theirs["fld"], 0.0, pc)),
    ("propagate_divergence 500^2 (Red Sea grid)", lambda: d.propagate_divergence(ours["redsea"]),
     lambda: ref.propagate_divergence(theirs["redsea"]), lambda: ref.propagate_divergence(theirs["redsea"], pc)),
    ("fit_gaussian 500^2 x 20 (Red Sea ensemble)", lambda: d.fit_gaussian(ours["redsea_ens"]),
     lambda: ref.fit_gaussian(theirs["redsea_ens"]), None),
    ("lcp 500^2", lambda: d.lcp(ours["redsea_fld"], 0.0), lambda: ref.lcp(theirs["redsea_fld"], 0.0),
     lambda: ref.lcp(theirs["redsea_fld"], 0.0, pc)),
    ("propagate_divergence 68^2 (wind grid)", lambda: d.propagate_divergence(ours["wind"]),
     lambda: ref.propagate_divergence(theirs["wind"]), None),
    ("fit_gaussian 68^2 x 15 (wind ensemble)", lambda: d.fit_gaussian(ours["wind_ens"]),
     lambda: ref.fit_gaussian(theirs["wind_ens"]), None),
    ("lcp 68^2", lambda: d.lcp(ours["wind_fld"], 0.0), lambda: ref.lcp(theirs["wind_fld"], 0.0), None),
    ("mc_divergence 256^2 N=200 (reference stream)",
     lambda: d.mc_divergence(ours["model2"], d.McConfig(200, seed=5), stream="reference"),
     lambda: ref.mc_divergence(theirs["model2"], ref.McConfig(200, seed=5)), None),
]
print(f"host: {threads} cores; times are the best of 5 after one warm-up; "
      f"DIVUQ_ADOPT={os.environ.get('DIVUQ_ADOPT', '1')}")
for name, fo, fr, fp in rows:
    t = best(fo)
    tr = best(fr, runs=3)
    tp = best(fp, runs=3) if fp else None
    tb = min(tr, tp) if tp else tr
    print(f"{name:46s} ours {t * 1e3:9.2f} ms | reference serial {tr * 1e3:9.1f} ms"
          + (f", {threads} threads {tp * 1e3:9.1f} ms" if tp else "")
          + f" | x{tb / t:7.1f} vs the faster")
