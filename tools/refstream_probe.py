import numpy as np, sys
sys.path.insert(0, '.')
import __graft_entry__; __graft_entry__.build()
import paper_2510_01190_b200 as pkg
from oracle import refstream
golden = lambda n: np.load("tests/golden/" + n)
nb = ((0.0, 1.0), (0.0, 0.0), (0.0, 0.0), (0.0, 0.0))
for seed in (0, 5, 2**64-1):
    n = 1_000_000
    z = -pkg.sample_divergence_1d(nb, (0.5, 1.0), pkg.McConfig(n, seed=seed))
    ref = refstream.normal_stream(seed, np.arange(n, dtype=np.uint64) * np.uint64(4))
    d = z != ref
    print("seed", seed, "bitwise frac", 1 - d.mean(), "n diff", d.sum(), "max ulps", (np.abs(z-ref)/np.spacing(np.abs(ref)))[d].max() if d.any() else 0)
g = golden("mc_refstream.npz")
for c in "ab":
    nx, ny, dx, dy, n, seed = g[f"mc_{c}_grid"]; m = g[f"mc_{c}_model"]
    model = pkg.GaussianVectorField(pkg.UniformGrid2(int(nx), int(ny), dx, dy), m[0], m[1], m[2], m[3])
    est = pkg.mc_divergence(model, pkg.McConfig(int(n), seed=int(seed)), stream="reference")
    print(c, "mean bitwise", np.mean(est.mean == g[f"mc_{c}_mean"]), "std bitwise", np.mean(est.std == g[f"mc_{c}_std"]))
h = pkg.mc_histogram_1d(((5.98, 0.96), (6.40, 0.38), (6.50, 0.94), (4.30, 0.65)), (1.0, 1.0), pkg.McConfig(20000, seed=7), n_bins=50)
print("hist edges bitwise", np.array_equal(h.bin_edges, g["hist_edges"]), "counts", np.array_equal(h.counts, g["hist_counts"]))
