"""CPU baselines of the hot path -- TEST INFRASTRUCTURE ONLY.

Only ``bench.py``'s ``cpu_baseline`` leg and ``--impl reference`` arm call
this, and both call the SAME ``cpu_leg`` (same sample, same threads):

* 2D configs 0-2: the UNMODIFIED reference itself -- its own pip install in
  ``baseline/_ref`` (made by ``__graft_entry__.build()``, shipped to the GPU
  box) -- through its public API, with ``ParallelConfig(threads=
  os.cpu_count())`` where the reference takes one (propagate_divergence,
  divergence.py:48-70; parallel.py:65-116), ``kind: "reference"``;
* 3D configs 3-4 (no reference code): the oracle restatement,
  parallelised the way the reference parallelises (static contiguous chunks
  of the index space on a thread pool, numpy releasing the GIL), fp64 like
  the reference (grid.py:23), ``kind: "port"``.
"""

from __future__ import annotations

import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import ref2d, ref3d


def _chunk_3d(fields, nx, ny, nz, z0, z1, dx, dy, dz, t):
    plane = nx * ny
    sl = [f[z0 * plane:z1 * plane] for f in fields]
    lo = (fields[2][(z0 - 1) * plane:z0 * plane], fields[5][(z0 - 1) * plane:z0 * plane]) if z0 else None
    hi = (fields[2][z1 * plane:(z1 + 1) * plane], fields[5][z1 * plane:(z1 + 1) * plane]) if z1 < nz else None
    mu, sg = ref3d.propagate3d_slab(sl, lo, hi, nx, ny, z0, nz, dx, dy, dz)
    p_src = ref2d.source_probability(mu, sg, t)
    p_snk = ref2d.sink_probability(mu, sg, t)
    return mu, sg, p_src, p_snk


def propagate3d_threaded(fields, nx, ny, nz, dx=1.0, dy=1.0, dz=1.0, t=0.0, threads=None,
                         planes_per_chunk=2):
    """mu, sigma, P(div>t), P(div<-t) for a whole (small) grid on all cores."""
    threads = threads or os.cpu_count() or 1
    bounds = list(range(0, nz, planes_per_chunk)) + [nz]
    with ThreadPoolExecutor(max_workers=threads) as pool:
        parts = list(pool.map(lambda ab: _chunk_3d(fields, nx, ny, nz, ab[0], ab[1], dx, dy, dz, t),
                              zip(bounds[:-1], bounds[1:])))
    return tuple(np.concatenate([p[q] for p in parts]) for q in range(4))


def propagate3d_thunk(nx, ny, nz_sample, threads=None, seed=0):
    """A callable running the threaded oracle once on an nx x ny x nz_sample
    sub-volume with config-3-like values."""
    threads = threads or os.cpu_count() or 1
    rng = np.random.default_rng(seed)
    n = nx * ny * nz_sample
    f = [rng.normal(size=n).astype(np.float32) for _ in range(3)] + \
        [rng.uniform(0.05, 0.3, n).astype(np.float32) for _ in range(3)]
    return lambda: propagate3d_threaded(f, nx, ny, nz_sample, threads=threads), n, threads


def ensemble3d_thunk(nx, ny, nz_sample, members, threads=None, seed=0):
    """A callable running fit_gaussian + 3D propagation + tails once."""
    threads = threads or os.cpu_count() or 1
    rng = np.random.default_rng(seed)
    n = nx * ny * nz_sample
    mem = rng.normal(0, 1, (members, 3, n)).astype(np.float32)

    def work():
        bounds = list(range(0, n, max(1, n // (4 * threads)))) + [n]
        with ThreadPoolExecutor(max_workers=threads) as pool:
            parts = list(pool.map(lambda ab: ref2d.fit_moments(mem[:, :, ab[0]:ab[1]]),
                                  zip(bounds[:-1], bounds[1:])))
        mu = np.concatenate([p[0] for p in parts], axis=1)
        sg = np.concatenate([p[1] for p in parts], axis=1)
        propagate3d_threaded(list(mu) + list(sg), nx, ny, nz_sample, t=0.1, threads=threads)

    return work, n, threads


def rate(thunk_n_threads, seconds=10.0):
    """(pts/s, threads, runs): one warm-up, then repeat for ~seconds."""
    thunk, n, threads = thunk_n_threads
    thunk()
    runs, t0 = 0, time.perf_counter()
    while True:
        thunk()
        runs += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return runs * n / el, threads, runs


def propagate2d_thunk(model, nx, ny, t):
    """Serial reference-order 2D propagation + both tails (config 0; the
    reference runs it serially when no ParallelConfig is given)."""
    mu_u, mu_v, s_u, s_v = model

    def work():
        mu, sg = ref2d.propagate2d(mu_u, mu_v, s_u, s_v, nx, ny, 1.0, 1.0)
        ref2d.source_probability(mu, sg, t)
        ref2d.sink_probability(mu, sg, t)

    return work, nx * ny, 1


def mc_thunk(model, nx, ny, n_samples):
    """The GPU's Philox estimator restated in numpy on `n_samples` samples
    (vertex-samples per call = nx*ny*n_samples)."""
    from . import philox

    mu_u, mu_v, s_u, s_v = model
    return (lambda: philox.mc_divergence(mu_u, mu_v, s_u, s_v, nx, ny, 1.0, 1.0, n_samples, 7),
            nx * ny * n_samples, 1)


# ---------------------------------------------------------------------------
# the unified CPU leg (both bench arms)
# ---------------------------------------------------------------------------

REF_ROOT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


def reference_package():
    """The unmodified reference ``divuq`` (baseline/_ref), or None if absent."""
    if not os.path.isdir(os.path.join(REF_ROOT, "divuq")):
        return None
    if REF_ROOT not in sys.path:
        sys.path.insert(0, REF_ROOT)
    import divuq

    return divuq


def _config1_members_host(nx, ny, m, seed):
    """Config-1 recipe on the host (24 sources/sinks + vortex, smooth sigma in
    [0.02, 0.5], iid normal perturbations): same shapes and value ranges as the
    device generator, for CPU timing only."""
    from paper_2510_01190_b200 import configs

    u, v, _, _ = configs.host_model2d(nx, ny, 24, seed)
    j, i = np.divmod(np.arange(nx * ny), nx)
    sig = 0.02 + 0.48 * (0.5 + 0.5 * np.sin(i / 37.0) * np.cos(j / 53.0))
    rng = np.random.default_rng(seed + 7)
    return [(u + sig * rng.standard_normal(nx * ny), v + sig * rng.standard_normal(nx * ny))
            for _ in range(m)]


def cpu_leg(cid, threads=None):
    """(thunk, units per call, unit, sample text, kind, extra) for config cid.

    The sample is fixed per config (not budget-derived), so the two bench
    arms time exactly the same work."""
    threads = threads or os.cpu_count() or 1
    ref = reference_package() if cid in (0, 1, 2) else None
    if cid in (0, 1, 2) and ref is None:
        raise RuntimeError("baseline/_ref (the reference install) is missing: run "
                           "__graft_entry__.build() where /root/reference exists")
    from paper_2510_01190_b200 import configs

    if cid == 0:
        mu_u, mu_v, s_u, s_v = configs.config0_model()
        g = ref.UniformGrid2(128, 128)
        model = ref.GaussianVectorField(g, mu_u, mu_v, s_u, s_v)
        pc = ref.ParallelConfig(threads=threads)
        from divuq.lcp import _tail_probs

        def work(par=True):
            f = ref.propagate_divergence(model, pc if par else None)
            _tail_probs(f.mu, f.sigma, 0.0)        # P(div <= 0), P(div > 0)
            _tail_probs(f.mu, f.sigma, -0.0)       # the sink map at -t

        return (work, g.n_vertices, "grid points/s",
                f"reference propagate_divergence(ParallelConfig(threads={threads})) + _tail_probs "
                "for P(div>0), P(div<0) on the full config-0 128^2 model", "reference")
    if cid == 1:
        nx, ny, m = 1024, 256, 20
        g = ref.UniformGrid2(nx, ny)
        ens = ref.Ensemble2(g, tuple(ref.VectorField2(g, a, b)
                                     for a, b in _config1_members_host(nx, ny, m, 101)))
        pc = ref.ParallelConfig(threads=threads)
        from divuq.lcp import _tail_probs

        def work(par=True):
            model = ref.fit_gaussian(ens)
            f = ref.propagate_divergence(model, pc if par else None)
            _tail_probs(f.mu, f.sigma, 0.0)

        return (work, g.n_vertices, "grid points/s",
                f"reference fit_gaussian (M=20) + propagate_divergence(ParallelConfig(threads="
                f"{threads})) + _tail_probs P(div>0), config-1 recipe on 1024x256 (a quarter of "
                "the 1024^2 grid)", "reference")
    if cid == 2:
        mu_u, mu_v, s_u, s_v = configs.config2_model()
        g = ref.UniformGrid2(256, 256)
        model = ref.GaussianVectorField(g, mu_u, mu_v, s_u, s_v)
        n = 100
        cfgm = ref.McConfig(n, seed=2024)

        def work(par=True):
            ref.mc_divergence(model, cfgm)

        return (work, g.n_vertices * n, "vertex-samples/s",
                "reference mc_divergence (numba RNG, numpy stencil, Welford) on the config-2 256^2 "
                f"model with N={n} samples (of 2000)", "reference")
    if cid == 3:
        work, n, _ = propagate3d_thunk(512, 512, 32, threads=threads)
        return (work, n, "grid points/s",
                f"oracle 3D propagation + P(div>0) + P(div<0), fp64, on a 512x512x32 sub-volume of "
                f"config 3, {threads} threads (no 3D reference code exists)", "port")
    work, n, _ = ensemble3d_thunk(1024, 1024, 2, 16, threads=threads)
    return (work, n, "grid points/s",
            f"oracle fit_gaussian (M=16) + 3D propagation + P(div>+-0.1), fp64, on 1024x1024x2 of "
            f"config 4, {threads} threads (no 3D reference code exists)", "port")


def time_leg(cid, seconds=10.0, threads=None):
    """The cpu_baseline dict of bench.py: one warm-up, then repeated calls for
    ~seconds (the reference's bench() protocol, parallel.py:119-129).  For the
    2D configs with a ParallelConfig seam (0, 1) both the threaded and the
    serial reference path are timed and the FASTER one is the baseline (at
    128^2 the reference's thread pool costs more than the work)."""
    threads = threads or os.cpu_count() or 1
    work, units, unit, sample, kind = cpu_leg(cid, threads)
    v, _, runs = rate((work, units, threads), seconds=seconds)
    out = {"value": v, "unit": unit, "cores": threads, "kind": kind,
           "sample": sample + f", {runs} timed runs after 1 warm-up"}
    if cid in (0, 1):   # the serial path too (ParallelConfig omitted)
        sv, _, sruns = rate((lambda: work(False), units, 1), seconds=min(seconds, 5.0))
        out["threaded_value"], out["serial_value"] = v, sv
        if sv > v:
            out.update(value=sv, cores=1,
                       sample=out["sample"] + f"; the serial path (config=None, {sruns} runs) is "
                              "faster and is the baseline value")
    return out
