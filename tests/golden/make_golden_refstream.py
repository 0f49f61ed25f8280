"""Golden vectors for the reference's own MC stream (splitmix64 + AS241).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_refstream.py

Imports ``divuq`` from /root/reference/pkg/src (read-only, nothing copied) and
writes ``mc_refstream.npz``: normal_stream values (rng.py:102-106) over edge and
random counters, mc_divergence estimates (mc.py:94-117), sample_divergence_1d
draws and mc_histogram_1d bins (mc.py:120-156), all produced by the reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
FIG1 = ((5.98, 0.96), (6.40, 0.38), (6.50, 0.94), (4.30, 0.65))   # test_mc.py:19


def main():
    sys.path.insert(0, REF_SRC)
    import divuq
    from divuq.mc import sample_divergence_1d
    from divuq.rng import normal_stream

    rng = np.random.default_rng(97)
    g = {}
    edge = np.array([0, 1, 2, 3, 2**32 - 1, 2**32, 2**63, 2**64 - 1], dtype=np.uint64)
    rand = rng.integers(0, 2**63, size=6000, dtype=np.uint64) * np.uint64(2)
    g["counters"] = np.concatenate([edge, rand])
    g["seeds"] = np.array([0, 5, 2**64 - 1], dtype=np.uint64)
    g["normals"] = np.stack([normal_stream(int(s), g["counters"]) for s in g["seeds"]])

    for name, (nx, ny, dx, dy, n, seed, zero) in {
        "a": (16, 12, 0.5, 0.75, 300, 5, False),
        "b": (7, 5, 1.0, 1.3, 513, 123, False),
        "c": (6, 4, 1.0, 1.0, 50, 9, True),
    }.items():
        grid = divuq.UniformGrid2(nx, ny, dx, dy)
        k = grid.n_vertices
        mu = rng.normal(0, 2, (2, k))
        sg = np.zeros((2, k)) if zero else rng.uniform(0.05, 0.6, (2, k))
        m = divuq.GaussianVectorField(grid, mu[0], mu[1], sg[0], sg[1])
        est = divuq.mc_divergence(m, divuq.McConfig(n, seed=seed))
        g[f"mc_{name}_grid"] = np.array([nx, ny, dx, dy, n, seed], dtype=np.float64)
        g[f"mc_{name}_model"] = np.concatenate([mu, sg])
        g[f"mc_{name}_mean"] = est.mean
        g[f"mc_{name}_std"] = est.std

    g["s1d_values"] = sample_divergence_1d(FIG1, (1.0, 1.0), divuq.McConfig(5000, seed=7))
    g["s1d_aniso"] = sample_divergence_1d(FIG1, (0.7, 1.9), divuq.McConfig(3000, seed=2**64 - 1))
    h = divuq.mc_histogram_1d(FIG1, (1.0, 1.0), divuq.McConfig(20000, seed=7), n_bins=50)
    g["hist_edges"], g["hist_counts"] = h.bin_edges, h.counts
    h = divuq.mc_histogram_1d(FIG1, (1.0, 2.0), divuq.McConfig(7777, seed=13), n_bins=7)
    g["hist2_edges"], g["hist2_counts"] = h.bin_edges, h.counts
    h = divuq.mc_histogram_1d(((1.0, 0.0), (2.0, 0.0), (3.0, 0.0), (4.0, 0.0)), (1.0, 1.0),
                              divuq.McConfig(500, seed=0), n_bins=10)
    g["hist0_edges"], g["hist0_counts"] = h.bin_edges, h.counts
    np.savez_compressed(os.path.join(OUT, "mc_refstream.npz"), **g)
    print("wrote mc_refstream.npz")


if __name__ == "__main__":
    main()
