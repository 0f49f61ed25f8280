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
