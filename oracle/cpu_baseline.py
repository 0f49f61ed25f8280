"""Threaded CPU baseline of the hot path -- TEST INFRASTRUCTURE ONLY.

Only ``bench.py``'s ``cpu_baseline`` leg and ``--impl reference`` arm call
this.  It times the oracle restatement of the reference's algorithm (the
reference itself is pure Python and cannot travel to the GPU box, and there is
no 3D reference -- SURVEY F2), parallelised the way the reference parallelises:
static contiguous chunks of the index space on a ThreadPoolExecutor
(parallel.py:65-116), numpy releasing the GIL inside each chunk.  Arithmetic
is fp64 like the reference (grid.py:23), on the same fp32-exact inputs.
"""

from __future__ import annotations

import os
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
