"""Velocity-magnitude-gradient prologue (gaussian.py:48-66).

Golden vectors from the reference (tests/golden/gradient.npz).  The GPU's
hypot is within an ulp of glibc's (the reference suite itself compares hypot
to sqrt(u^2 + v^2) at rtol 1e-15, pkg/tests/test_gaussian.py:85-92); the
gradient stencil is the reference's expression, so gradients agree to a few
ulps.  The reference suite's gradient cases run on the GPU.
"""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def d():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build()
    import paper_2510_01190_b200

    return paper_2510_01190_b200


def _xy(g):
    return (np.arange(g.n_vertices) % g.nx) * g.dx, (np.arange(g.n_vertices) // g.nx) * g.dy


def test_gradient_ensemble_vs_reference_golden(d):
    gd = golden("gradient.npz")
    nx, ny, dx, dy = gd["grid"]
    g = d.UniformGrid2(int(nx), int(ny), float(dx), float(dy))
    mem = gd["members"]
    ens = d.Ensemble2(g, tuple(d.VectorField2(g, m[0], m[1]) for m in mem))
    out = d.gradient_ensemble(ens)
    got = np.stack([np.stack([m.u, m.v]) for m in out.members])
    ref = gd["out"]
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
    vm = d.velocity_magnitude(ens.members[0]).values
    assert np.allclose(vm, gd["vmag0"], rtol=1e-15, atol=0)


def test_velocity_magnitude_cases(d):
    g = d.UniformGrid2(2, 2)
    mag = d.velocity_magnitude(d.VectorField2(g, [3, 0, 1, 0], [4, 0, 1, 0]))
    assert mag.values[0] == 5.0 and mag.values[1] == 0.0
    rng = np.random.default_rng(1)
    u, v = rng.normal(size=4), rng.normal(size=4)
    got = d.velocity_magnitude(d.VectorField2(g, u, v)).values
    assert np.allclose(got, np.sqrt(u**2 + v**2), rtol=1e-15)


def test_gradient_affine_constant_and_quadratic(d):
    g = d.UniformGrid2(9, 7, 0.3, 0.7)
    x, y = _xy(g)
    grad = d.gradient(d.ScalarField2(g, 2.0 * x + 3.0 * y))
    assert np.allclose(grad.u, 2.0, rtol=0, atol=1e-13)
    assert np.allclose(grad.v, 3.0, rtol=0, atol=1e-13)
    const = d.gradient(d.ScalarField2(g, np.full(g.n_vertices, 5.0)))
    assert np.all(const.u == 0.0) and np.all(const.v == 0.0)
    g = d.UniformGrid2(101, 3, 0.01, 0.01)
    x, _ = _xy(g)
    grad = d.gradient(d.ScalarField2(g, x**2))
    i = np.arange(g.n_vertices) % g.nx
    inner = (i > 0) & (i < g.nx - 1)
    assert np.max(np.abs(grad.u[inner] - 2.0 * x[inner])) < 1e-3


def test_gradient_ensemble_identical_members_and_composition(d):
    g = d.UniformGrid2(8, 8)
    rng = np.random.default_rng(2)
    m = d.VectorField2(g, rng.normal(size=64), rng.normal(size=64))
    out = d.gradient_ensemble(d.Ensemble2(g, (m, m)))
    assert np.array_equal(out.members[0].u, out.members[1].u)
    g = d.UniformGrid2(10, 10)
    rng = np.random.default_rng(3)
    members = tuple(d.VectorField2(g, rng.normal(size=100), rng.normal(size=100)) for _ in range(3))
    out = d.gradient_ensemble(d.Ensemble2(g, members))
    for k, m in enumerate(members):
        direct = d.gradient(d.velocity_magnitude(m))
        assert np.array_equal(out.members[k].u, direct.u)
        assert np.array_equal(out.members[k].v, direct.v)


def test_vortex_magnitude_gradient_pipeline_to_divergence(d):
    # (u, v) = (-y, x) exp(-r^2): |f| grows away from the centre, so the
    # magnitude-gradient field diverges there (pkg/tests/test_gaussian.py:137-158)
    g = d.UniformGrid2(41, 41, 0.1, 0.1)
    x, y = _xy(g)
    r2 = (x - 2.0) ** 2 + (y - 2.0) ** 2
    m = d.VectorField2(g, -(y - 2.0) * np.exp(-r2), (x - 2.0) * np.exp(-r2))
    grad = d.gradient(d.velocity_magnitude(m))
    centre = g.vertex_index(20, 20)
    assert d.divergence_deterministic(grad).values[centre] > 0


@pytest.mark.parametrize("shape", [(2, 2, 1.0, 1.0), (3, 70, 0.5, 0.25), (33, 9, 0.1, 0.3),
                                   (65, 17, 1.0, 2.0), (130, 41, 0.01, 0.07)])
def test_gradient_ensemble_tiles_vs_oracle(d, shape):
    # tile edges (32 x 8) at every offset, 2-wide axes, partial tiles
    import torch

    from oracle import ref2d
    from paper_2510_01190_b200 import device

    nx, ny, dx, dy = shape
    rng = np.random.default_rng(nx * 1000 + ny)
    mem = rng.normal(size=(3, 2, nx * ny))
    want = ref2d.gradient_ensemble(mem, nx, ny, dx, dy)
    got = device.gradient_ensemble2d(torch.from_numpy(mem).cuda(), nx, ny, dx, dy).cpu().numpy()
    # GPU hypot within 1 ulp of glibc's: |d(gx)| <= (ulp(a) + ulp(b)) * c <= 4.4e-16 * max|f| / h
    fmax = np.hypot(mem[:, 0], mem[:, 1]).max()
    assert np.abs(got - want).max() <= 5e-16 * fmax / min(dx, dy)
    got32 = device.gradient_ensemble2d(torch.from_numpy(mem.astype(np.float32)).cuda(), nx, ny,
                                       dx, dy).cpu().numpy()
    want32 = ref2d.gradient_ensemble(mem.astype(np.float32), nx, ny, dx, dy)
    assert np.abs(got32 - want32).max() <= 1e-5 * np.abs(want32).max()


@pytest.mark.parametrize("shape", [(2, 2, 1.0, 1.0), (3, 70, 0.5, 0.25), (65, 17, 1.0, 2.0),
                                   (130, 41, 0.01, 0.07), (64, 16, 1.0, 1.0), (200, 33, 0.3, 0.3),
                                   (4, 3, 1.0, 1.0), (128, 300, 0.5, 0.5), (68, 2, 1.0, 1.0)])
@pytest.mark.parametrize("m,t", [(2, 0.0), (5, 0.3), (20, 0.0)])
def test_fused_gradient_ensemble_divergence(d, shape, m, t, monkeypatch):
    """K6 (velocity magnitude -> gradient -> moments -> divergence -> tails,
    one pass) == gradient_ensemble2d_f32 then ensemble_divergence2d_f32, bit
    for bit, at every tile offset; and within the fp32 bar of the fp64 oracle
    composition of the reference's functions."""
    import torch

    from oracle import ref2d
    from paper_2510_01190_b200 import device

    nx, ny, dx, dy = shape
    rng = np.random.default_rng(nx * 7 + ny * 3 + m)
    base = rng.normal(size=(1, 2, nx * ny))
    mem = (base + 0.2 * rng.normal(size=(m, 2, nx * ny))).astype(np.float32)
    gm = torch.from_numpy(mem).cuda()
    fused = device.gradient_ensemble_divergence2d(gm, nx, ny, dx, dy, t, moments=True)
    grad = device.gradient_ensemble2d(gm, nx, ny, dx, dy)
    comp = device.ensemble_divergence2d(grad, nx, ny, dx, dy, t, moments=True)
    for k in ("mu", "sigma", "p_src", "p_snk", "mom_mu", "mom_sigma"):
        assert torch.equal(fused[k], comp[k]), k
    # the opt-in strip march (nx % 4 == 0) and the tiled K6 are the same arithmetic
    monkeypatch.setenv("DIVUQ_GRADMARCH", "1")
    march = device.gradient_ensemble_divergence2d(gm, nx, ny, dx, dy, t, moments=True)
    monkeypatch.delenv("DIVUQ_GRADMARCH")
    for k in ("mu", "sigma", "p_src", "p_snk", "mom_mu", "mom_sigma"):
        assert torch.equal(fused[k], march[k]), k
    g64 = ref2d.gradient_ensemble(mem.astype(np.float64), nx, ny, dx, dy)
    mu_r, sg_r = ref2d.fit_moments(g64)
    dmu, dsg = ref2d.propagate2d(mu_r[0], mu_r[1], sg_r[0], sg_r[1], nx, ny, dx, dy)
    got_mu = fused["mu"].cpu().numpy()
    got_sg = fused["sigma"].cpu().numpy()
    assert np.abs(got_mu - dmu).max() <= 1e-5 * np.abs(dmu).max()
    assert np.abs(got_sg - dsg).max() <= 1e-5 * np.abs(dsg).max()
    ps_own = ref2d.source_probability(got_mu.astype(np.float64), got_sg.astype(np.float64), t)
    p = fused["p_src"].cpu().numpy()
    assert np.all(np.abs(p - ps_own) <= 1e-5 * ps_own + 1e-6)


def test_fused_gradient_ensemble_divergence_host_api_and_errors(d):
    import torch

    from paper_2510_01190_b200 import device

    g = d.UniformGrid2(96, 40, 0.5, 0.25)
    x, y = _xy(g)
    rng = np.random.default_rng(5)
    members = []
    for k in range(6):   # vortex ensemble with jittered centres (the Red Sea use case)
        cx, cy = 24 + rng.normal(0, 0.5), 5 + rng.normal(0, 0.3)
        r2 = (x - cx) ** 2 + (y - cy) ** 2
        members.append(d.VectorField2(g, -(y - cy) * np.exp(-r2 / 20), (x - cx) * np.exp(-r2 / 20)))
    ens = d.Ensemble2(g, members)
    res = d.gradient_ensemble_divergence(ens, 0.0)
    gm = torch.from_numpy(np.ascontiguousarray(ens.stacked(), dtype=np.float32)).cuda()
    o = device.gradient_ensemble_divergence2d(gm, g.nx, g.ny, g.dx, g.dy, 0.0, moments=True)
    assert np.array_equal(res.field.mu, o["mu"].cpu().numpy())
    assert np.array_equal(res.field.sigma, o["sigma"].cpu().numpy())
    assert np.array_equal(res.model.mu_u, o["mom_mu"][0].cpu().numpy())
    # the magnitude-gradient field diverges at the vortex core
    centre = int(np.argmin((x - 24) ** 2 + (y - 5) ** 2))
    assert res.field.mu[centre] > 0 and res.p_src[centre] > 0.5
    bad = gm.clone()
    bad[1, 0, 7] = float("nan")
    with pytest.raises(ValueError, match="non-finite"):
        device.gradient_ensemble_divergence2d(bad, g.nx, g.ny, g.dx, g.dy)
    with pytest.raises(ValueError):
        device.gradient_ensemble_divergence2d(gm[:1].contiguous(), g.nx, g.ny, g.dx, g.dy)
