"""Level-crossing probability (lcp.py:71-100).

CPU part: the oracle restatement is pinned BITWISE to the reference's own
lcp() / cell_crossing_probability outputs (tests/golden/lcp.npz).
GPU part: the kernel vs those golden values at |dP| <= 1e-12 (the tails come
from a branch-free fitted fp64 erfc, max 3.8e-15 relative; not scipy's), plus the reference suite's own LCP
properties (pkg/tests/test_lcp.py): range, exact negation symmetry, sigma -> 0
indicator, finite extreme tails, the cell formula on a field.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import ref2d


def test_oracle_lcp_bitwise_vs_reference_golden():
    g = golden("lcp.npz")
    for gi in range(int(g["n_grids"])):
        nx, ny, iso = g[f"l{gi}_grid"]
        got = ref2d.lcp(g[f"l{gi}_mu"], g[f"l{gi}_sigma"], int(nx), int(ny), float(iso))
        assert np.array_equal(got, g[f"l{gi}_lcp"]), gi
    got = ref2d.cell_crossing_probability(g["cells_mu"], g["cells_sigma"], 0.3)
    assert np.array_equal(got, g["cells_lcp"])


@pytest.fixture(scope="module")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build()
    import paper_2510_01190_b200 as d

    return d


def _cell(d, mus, sigmas, theta):
    return float(d.cell_crossing_probability(np.array([mus], float), np.array([sigmas], float), theta)[0])


@pytest.mark.gpu
def test_lcp_gpu_vs_reference_golden(gpu):
    d = gpu
    g = golden("lcp.npz")
    for gi in range(int(g["n_grids"])):
        nx, ny, iso = g[f"l{gi}_grid"]
        grid = d.UniformGrid2(int(nx), int(ny))
        fld = d.GaussianScalarField(grid, g[f"l{gi}_mu"], g[f"l{gi}_sigma"])
        out = d.lcp(fld, float(iso))
        assert isinstance(out, d.LcpField) and out.probabilities.shape == (grid.n_cells,)
        assert np.abs(out.probabilities - g[f"l{gi}_lcp"]).max() <= 1e-12
    got = d.cell_crossing_probability(g["cells_mu"], g["cells_sigma"], 0.3)
    assert np.abs(got - g["cells_lcp"]).max() <= 1e-12


@pytest.mark.gpu
def test_lcp_reference_suite_properties(gpu, rng):
    d = gpu
    assert _cell(d, [1, 2, 3, 4], [0, 0, 0, 0], 0.5) == 0.0
    assert _cell(d, [-1, 2, 3, 4], [0, 0, 0, 0], 0.5) == 1.0
    assert abs(_cell(d, [0.7] * 4, [0.3] * 4, 0.7) - 0.875) <= 1e-15
    assert _cell(d, [1e8] * 4, [1e-8] * 4, 0.0) == 0.0
    assert _cell(d, [0.0, 0.0, 1e8, -1e8], [1e-8] * 4, 0.5) == 1.0
    # exact negation symmetry and range on random cells
    mus = rng.uniform(-100, 100, (5000, 4))
    sgs = rng.uniform(0.001, 10, (5000, 4))
    th = 0.37
    a = d.cell_crossing_probability(mus, sgs, th)
    b = d.cell_crossing_probability(-mus, sgs, -th)
    assert np.array_equal(a, b)
    assert np.all((a >= 0) & (a <= 1))
    # sigma -> 0: the deterministic crossing indicator
    mus = rng.normal(size=(500, 4))
    theta = 0.1
    crossing = ~(np.all(mus < theta, axis=1) | np.all(mus > theta, axis=1))
    assert np.array_equal(d.cell_crossing_probability(mus, np.zeros_like(mus), theta), crossing.astype(float))
    shrunk = d.cell_crossing_probability(mus, np.full_like(mus, 1e-300), theta)
    assert np.abs(shrunk - crossing).max() <= 1e-12
    # subnormal / tiny sigma and quotients that overflow: the reference's
    # "overflow allowed" division (lcp.py:62-65) -> the 0/1 limits, never NaN
    # (regression: the reciprocal-based quotient returned NaN; found by the
    # reference's own test_lcp.py through the drop-in hook)
    cases = [([0.0] * 4, [0.0, 0.0, 0.0, 5e-324], 0.0),
             ([0.0, 1.0, -1.0, 2.0], [5e-324, 1e-310, 2.2e-308, 1e-300], 0.5),
             ([1e300, -1e300, 1e300, -1e300], [1e-10, 1e-10, 1e-300, 1e-300], 0.0),
             ([3.0, 3.0, 3.0, 3.0], [1e-320, 1e-320, 1e-320, 1e-320], 3.0)]
    for mu4, s4, th in cases:
        got = d.cell_crossing_probability(np.array([mu4]), np.array([s4]), th)
        with np.errstate(over="ignore", divide="ignore", invalid="ignore"):
            want = ref2d.cell_crossing_probability(np.array([mu4]), np.array([s4]), th)
        assert np.all(np.isfinite(got)) and 0.0 <= got[0] <= 1.0, (mu4, s4, th, got)
        assert np.abs(got - want).max() <= 1e-12, (mu4, s4, th, got, want)


@pytest.mark.gpu
def test_lcp_field_matches_cell_formula_and_device_api(gpu, rng):
    d = gpu
    import torch

    from paper_2510_01190_b200 import device as dev

    for nx, ny in ((5, 4), (70, 33), (2, 2)):
        grid = d.UniformGrid2(nx, ny)
        mu = rng.normal(size=grid.n_vertices)
        sg = rng.uniform(0.05, 0.5, grid.n_vertices)
        out = d.lcp(d.GaussianScalarField(grid, mu, sg), -0.1)
        assert np.abs(out.probabilities - ref2d.lcp(mu, sg, nx, ny, -0.1)).max() <= 1e-12
        o32 = dev.lcp2d(torch.from_numpy(mu.astype(np.float32)).cuda(),
                        torch.from_numpy(sg.astype(np.float32)).cuda(), nx, ny, -0.1).cpu().numpy()
        ref32 = ref2d.lcp(mu.astype(np.float32), sg.astype(np.float32), nx, ny, -0.1)
        assert np.abs(o32 - ref32).max() <= 2e-5


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(4096, 64), (130, 67), (65, 33), (2, 2), (3, 5), (64, 16), (66, 18)])
def test_propagate_lcp_fused(gpu, rng, shape):
    """propagate -> lcp fused (8f next #1): bitwise equal to K2 then the LCP
    kernel, the divergence moments bitwise equal to the reference order, the
    LCP within 1e-12 of the oracle chain (pinned bitwise to the reference's
    lcp()); odd nx takes the two-kernel path with the same bits."""
    import torch

    from paper_2510_01190_b200 import device as dev

    d = gpu
    nx, ny = shape
    n = nx * ny
    a = [rng.normal(0, 2, n), rng.normal(0, 2, n), rng.uniform(0.05, 0.6, n), rng.uniform(0.05, 0.6, n)]
    t = [torch.from_numpy(x).cuda() for x in a]
    for iso in (0.0, -0.3):
        f = dev.propagate_lcp2d(*t, nx, ny, 0.7, 1.3, iso)
        k2 = dev.propagate2d(*t, nx, ny, 0.7, 1.3, 0.0, outputs=("mu", "sigma"))
        l2 = dev.lcp2d(k2["mu"], k2["sigma"], nx, ny, iso)
        assert torch.equal(f["mu"], k2["mu"]) and torch.equal(f["sigma"], k2["sigma"])
        assert torch.equal(f["lcp"], l2)
        mu, sg = ref2d.propagate2d(*a, nx, ny, 0.7, 1.3)
        assert np.array_equal(f["mu"].cpu().numpy(), mu)
        assert np.abs(f["lcp"].cpu().numpy() - ref2d.lcp(mu, sg, nx, ny, iso)).max() <= 1e-12
    # moments not requested: same LCP; reference-facing entry point
    g = dev.propagate_lcp2d(*t, nx, ny, 0.7, 1.3, 0.0, moments=False)
    assert torch.equal(g["lcp"], dev.propagate_lcp2d(*t, nx, ny, 0.7, 1.3, 0.0)["lcp"])
    grid = d.UniformGrid2(nx, ny, 0.7, 1.3)
    fld, lf = d.propagate_lcp(d.GaussianVectorField(grid, *a), 0.0)
    assert np.array_equal(fld.mu, mu) and np.array_equal(fld.sigma, sg)
    assert np.array_equal(lf.probabilities, g["lcp"].cpu().numpy())
    # validation: a negative sigma raises the reference's ValueError
    bad = [x.clone() for x in t]
    bad[2][n // 2] = -1.0
    with pytest.raises(ValueError):
        dev.propagate_lcp2d(*bad, nx, ny, 0.7, 1.3, 0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(1031, 517), (65, 33), (3, 70), (4095, 41)])
def test_lcp_flat_kernel_matches_register_kernel(gpu, rng, shape, monkeypatch):
    """Odd nx runs the 1D-tensor-map LCP kernel (row boxes at 16-byte-aligned
    starts); the register kernel is the same arithmetic, bit for bit."""
    import torch

    from paper_2510_01190_b200 import device as dev

    nx, ny = shape
    n = nx * ny
    mu = rng.normal(0, 1.5, n)
    sg = rng.uniform(0, 2, n)
    sg[rng.random(n) < 0.05] = 0.0
    mu[rng.random(n) < 0.02] = 0.25
    m, s = torch.from_numpy(mu).cuda(), torch.from_numpy(sg).cuda()
    for t in (0.0, 0.25):
        a = dev.lcp2d(m, s, nx, ny, t)
        monkeypatch.setenv("DIVUQ_NO_FLAT", "1")
        b = dev.lcp2d(m, s, nx, ny, t)
        monkeypatch.delenv("DIVUQ_NO_FLAT")
        assert torch.equal(a, b)
        assert np.abs(a.cpu().numpy() - ref2d.lcp(mu, sg, nx, ny, t)).max() <= 1e-12
