import sys; sys.path.insert(0, ".")  # run from the repo root
import numpy as np
import paper_2510_01190_b200 as d
g = d.UniformGrid2(512, 512, 1.0, 1.0)
members = [d.VectorField2(g, np.random.randn(g.n_vertices), np.random.randn(g.n_vertices)) for _ in range(20)]
model = d.fit_gaussian(d.Ensemble2(g, members))
div = d.propagate_divergence(model)
p_src = d.source_probability(div, 0.0)
cells = d.lcp(div, 0.0)
est = d.mc_divergence(model, d.McConfig(n_samples=1000, seed=7))
print("readme snippet ok", div.mu.shape, p_src.shape, cells.probabilities.shape, est.mean.shape)
