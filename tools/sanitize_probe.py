"""Small invocations of every kernel family: python tools/sanitize_probe.py.
Written for compute-sanitizer runs (memcheck / racecheck / synccheck); the GPU
pool has since closed compute-sanitizer, so it now runs plainly as an
every-kernel smoke (odd and aligned shapes, halos, slot merges) next to the
bounds/validation tests in tests/."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_2510_01190_b200 import device as dev  # noqa: E402
import paper_2510_01190_b200 as d  # noqa: E402

rng = np.random.default_rng(0)
cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
# K2 2D fp64 + 3D fp32 (TMA, pacer: 64+ planes)
nx, ny = 37, 21
a = [rng.normal(size=nx * ny), rng.normal(size=nx * ny), rng.uniform(0.1, 0.5, nx * ny), rng.uniform(0.1, 0.5, nx * ny)]
dev.propagate2d(*[cu(x) for x in a], nx, ny, 0.5, 0.7, 0.1)
nx, ny, nz = 128, 28, 70
f = [rng.normal(size=nx * ny * nz).astype(np.float32) for _ in range(3)] + \
    [rng.uniform(0.1, 0.4, nx * ny * nz).astype(np.float32) for _ in range(3)]
dev.propagate3d(*[cu(x) for x in f], nx, ny, nz, 1.0, 1.0, 1.0, 0.0)
# K3 3D tiled, 2D row march (+ tiled fallback with many members)
mem = rng.normal(0, 1, (5, 3, 128 * 20 * 9)).astype(np.float32)
dev.ensemble_divergence3d(cu(mem), 128, 20, 9, 1.0, 1.0, 1.0, 0.1)
for m, (nx, ny) in ((20, (192, 70)), (3, (68, 5)), (40, (64, 9))):
    mem2 = rng.normal(0, 1, (m, 2, nx * ny)).astype(np.float32)
    dev.ensemble_divergence2d(cu(mem2), nx, ny, 0.5, 0.5, 0.0, moments=True)
# K1 fp32 / fp64 (smem parking), strided
dev.fit_moments(cu(rng.normal(size=(20, 2, 4096)).astype(np.float32)))
dev.fit_moments(cu(rng.normal(size=(20, 2, 4096))))
# K4 both streams, LCP, gradient, histogram
nx, ny = 40, 24
t = [cu(x) for x in (rng.normal(size=nx * ny), rng.normal(size=nx * ny),
                     rng.uniform(0.1, 0.5, nx * ny), rng.uniform(0.1, 0.5, nx * ny))]
dev.mc_divergence2d(*t, nx, ny, 0.5, 0.7, 300, 3)
dev.mc_divergence2d(*t, nx, ny, 0.5, 0.7, 40, 3, stream="reference")
mu, sg = cu(rng.normal(size=130 * 70)), cu(rng.uniform(0.1, 1, 130 * 70))
dev.lcp2d(mu, sg, 130, 70, 0.0)
dev.gradient_ensemble2d(cu(rng.normal(size=(3, 2, 130 * 70))), 130, 70)
dev.lcp2d(cu(rng.normal(size=131 * 33)), cu(rng.uniform(0, 1, 131 * 33)), 131, 33, 0.2)   # register LCP
dev.tail_probs(mu, sg, 0.3)
g4 = [cu(x) for x in (rng.normal(size=130 * 70), rng.normal(size=130 * 70),
                      rng.uniform(0, 1, 130 * 70), rng.uniform(0, 1, 130 * 70))]
dev.propagate_lcp2d(*g4, 130, 70, 0.5, 0.7, 0.1, moments=True)               # fused LCP (round 2)
# K6 fused Red Sea chain (TMA: nx % 4 == 0; register-staged: odd nx), fp32 members
for nx6, ny6 in ((132, 37), (129, 37)):
    dev.gradient_ensemble_divergence2d(cu(rng.normal(size=(6, 2, nx6 * ny6)).astype(np.float32)),
                                       nx6, ny6, 0.5, 0.5, 0.0, moments=True)
# MC with more chunks than slots (Chan merge across a slot's chunks), then
# the device error_metrics reduction on its output
em, es = dev.mc_divergence2d(*t, nx, ny, 0.5, 0.7, 129 * 40, 5)
dev.error_metrics(em, es, t[0], t[2])
d.mc_histogram_1d(((1.0, 0.3), (2.0, 0.2), (0.5, 0.1), (1.5, 0.4)), (1.0, 1.0), d.McConfig(5000, seed=1), 17)
torch.cuda.synchronize()
print("sanitize probe: ok")
