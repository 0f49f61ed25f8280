"""Pin the CPU oracle before trusting it (CPU-only; no GPU needed).

The 2D restatement must reproduce the reference's own outputs BITWISE on the
golden vectors in tests/golden (produced by make_golden.py running the
reference).  The 3D restatement is pinned by planar reduction to the 2D
reference plus exact invariants.  Philox is pinned by Random123's
known-answer vectors.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import philox, ref2d, ref3d


def test_propagate2d_bitwise_vs_reference_golden():
    g = golden("propagate2d.npz")
    for gi in range(int(g["n_grids"])):
        nx, ny, dx, dy = g[f"g{gi}_grid"]
        nx, ny = int(nx), int(ny)
        mu, sigma = ref2d.propagate2d(
            g[f"g{gi}_mu_u"], g[f"g{gi}_mu_v"], g[f"g{gi}_s_u"], g[f"g{gi}_s_v"], nx, ny, dx, dy
        )
        assert np.array_equal(mu, g[f"g{gi}_out_mu"]), gi
        assert np.array_equal(sigma, g[f"g{gi}_out_sigma"]), gi
        det = ref2d.divergence2d(g[f"g{gi}_mu_u"], g[f"g{gi}_mu_v"], nx, ny, dx, dy)
        assert np.array_equal(det, g[f"g{gi}_det"]), gi
        for t in (0.0, 0.3):
            assert np.array_equal(ref2d.source_probability(mu, sigma, t), g[f"g{gi}_t{t}_above"])
            assert np.array_equal(ref2d.sink_probability(mu, sigma, t), g[f"g{gi}_t{t}_below_neg"])


def test_fig1_golden():
    g = golden("fig1.npz")
    mu, sd = ref2d.stencil_distribution(tuple(map(tuple, g["neighbors"])), (1.0, 1.0))
    assert mu == float(g["mu"])
    assert sd == float(g["sigma"])
    assert sd == 0.7700811645534514  # pkg/tests/test_divergence.py:21
    assert abs(mu - (-0.89)) <= 1e-12


def test_tail_probs_bitwise_vs_reference_golden():
    g = golden("tail_probs.npz")
    for t in (0.0, 0.1, 0.3, -0.7):
        b, a = ref2d.tail_probs(g["mu"], g["sigma"], t)
        assert np.array_equal(b, g[f"t{t}_below"])
        assert np.array_equal(a, g[f"t{t}_above"])


def test_fit_gaussian_bitwise_vs_reference_golden():
    g = golden("fit_gaussian.npz")
    for ci in range(int(g["n_cases"])):
        mu, sd = ref2d.fit_gaussian(g[f"c{ci}_members"])
        assert np.array_equal(mu[0], g[f"c{ci}_mu_u"]), ci
        assert np.array_equal(mu[1], g[f"c{ci}_mu_v"]), ci
        assert np.array_equal(sd[0], g[f"c{ci}_s_u"]), ci
        assert np.array_equal(sd[1], g[f"c{ci}_s_v"]), ci
    mu, sd = ref2d.fit_gaussian(g["syn_members"])
    assert np.array_equal(mu[0], g["syn_mu_u"]) and np.array_equal(sd[1], g["syn_s_v"])
    dm, ds = ref2d.propagate2d(mu[0], mu[1], sd[0], sd[1], 24, 20, 1.0, 1.0)
    assert np.array_equal(dm, g["syn_div_mu"]) and np.array_equal(ds, g["syn_div_sigma"])


def test_ref3d_planar_reduces_to_2d_reference_bitwise(rng):
    g = golden("propagate2d.npz")
    for gi in (2, 3, 6):
        nx, ny, dx, dy = g[f"g{gi}_grid"]
        nx, ny = int(nx), int(ny)
        nz = 5
        t = lambda a: np.tile(a, nz)
        z = np.zeros(nx * ny * nz)
        mu, sd = ref3d.propagate3d(
            t(g[f"g{gi}_mu_u"]), t(g[f"g{gi}_mu_v"]), z,
            t(g[f"g{gi}_s_u"]), t(g[f"g{gi}_s_v"]), z, nx, ny, nz, dx, dy, 0.7,
        )
        for k in range(nz):
            sl = slice(k * nx * ny, (k + 1) * nx * ny)
            assert np.array_equal(mu[sl], g[f"g{gi}_out_mu"])
            assert np.array_equal(sd[sl], g[f"g{gi}_out_sigma"])


def test_ref3d_identity_and_rotation_fields():
    nx, ny, nz, dx, dy, dz = 11, 9, 7, 0.5, 0.25, 2.0
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    x, y, zc = (i * dx).ravel(), (j * dy).ravel(), (k * dz).ravel()
    d = ref3d.divergence3d(x, y, zc, nx, ny, nz, dx, dy, dz)
    assert np.all(d == 3.0)
    d = ref3d.divergence3d(-y, x, np.zeros_like(x), nx, ny, nz, dx, dy, dz)
    assert np.all(d == 0.0)


def test_ref3d_uniform_and_zero_sigma(rng):
    nx = ny = nz = 6
    n = nx * ny * nz
    s, h = 0.4, 0.5
    mu0 = np.zeros(n)
    _, sd = ref3d.propagate3d(mu0, mu0, mu0, *(np.full(n, s),) * 3, nx, ny, nz, h, h, h)
    interior = sd.reshape(nz, ny, nx)[1:-1, 1:-1, 1:-1]
    # six terms of (s/(2h))^2 -> sqrt(6)/2 * s/h
    assert np.allclose(interior, np.sqrt(6.0) / 2.0 * s / h, rtol=1e-15)
    u, v, w = rng.normal(size=(3, n))
    mu, sd = ref3d.propagate3d(u, v, w, mu0, mu0, mu0, nx, ny, nz, 1.0, 1.0, 1.0)
    assert np.all(sd == 0.0)
    assert np.array_equal(mu, ref3d.divergence3d(u, v, w, nx, ny, nz, 1.0, 1.0, 1.0))


def test_ref3d_slab_decomposition_bitwise(rng):
    nx, ny, nz = 7, 5, 13
    n = nx * ny * nz
    f = [rng.normal(size=n) for _ in range(3)] + [rng.uniform(0.1, 1, n) for _ in range(3)]
    mu, sd = ref3d.propagate3d(*f, nx, ny, nz, 0.3, 0.7, 1.1)
    plane = nx * ny
    for parts in (1, 2, 3, 4, 13):
        bounds = [nz * r // parts for r in range(parts + 1)]
        for r in range(parts):
            z0, z1 = bounds[r], bounds[r + 1]
            sl = [a[z0 * plane:z1 * plane] for a in f]
            lo = (f[2][(z0 - 1) * plane:z0 * plane], f[5][(z0 - 1) * plane:z0 * plane]) if z0 else None
            hi = (f[2][z1 * plane:(z1 + 1) * plane], f[5][z1 * plane:(z1 + 1) * plane]) if z1 < nz else None
            m, s = ref3d.propagate3d_slab(sl, lo, hi, nx, ny, z0, nz, 0.3, 0.7, 1.1)
            assert np.array_equal(m, mu[z0 * plane:z1 * plane])
            assert np.array_equal(s, sd[z0 * plane:z1 * plane])


@pytest.mark.parametrize(
    "ctr,key,expect",
    [  # Random123 kat_vectors, philox4x32_10
        ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
        ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
        ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
         (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
    ],
)
def test_philox_known_answers(ctr, key, expect):
    out = philox.philox4x32_10(*ctr, *key)
    assert tuple(int(x) for x in out) == expect


def test_philox_normals_are_standard():
    z_u, z_v = philox.normals(7, np.arange(200_000), 3)
    for z in (z_u, z_v):
        assert abs(z.mean()) < 5 / np.sqrt(2e5)
        assert abs(z.std() - 1.0) < 5 / np.sqrt(4e5)
    assert abs(np.corrcoef(z_u, z_v)[0, 1]) < 5 / np.sqrt(2e5)


def test_philox_mc_oracle_statistics_and_zero_sigma(rng):
    g = golden("mc_ref.npz")
    nx, ny, dx, dy = g["grid"]
    nx, ny = int(nx), int(ny)
    n = int(g["n_samples"])
    mean, std = philox.mc_divergence(g["mu_u"], g["mu_v"], g["s_u"], g["s_v"], nx, ny, dx, dy, n, 5)
    # statistical agreement with the analytic moments (4 sigma / sqrt(N))
    assert np.mean(np.abs(mean - g["an_mu"]) <= 4 * g["an_sigma"] / np.sqrt(n)) >= 0.99
    assert np.mean(np.abs(std - g["an_sigma"]) <= 4 * g["an_sigma"] / np.sqrt(2 * n)) >= 0.99
    # and with the reference's own (splitmix64 + AS241) estimate: both are
    # unbiased, so their difference is within 4*sqrt(2)*sigma/sqrt(N)
    assert np.mean(np.abs(mean - g["mean"]) <= 4 * np.sqrt(2) * g["an_sigma"] / np.sqrt(n)) >= 0.99
    # sigma == 0 -> exactly the deterministic divergence, std exactly 0 (test_mc.py:33-41)
    z = np.zeros(nx * ny)
    m0, s0 = philox.mc_divergence(g["mu_u"], g["mu_v"], z, z, nx, ny, dx, dy, 300, 9)
    assert np.array_equal(m0, ref2d.divergence2d(g["mu_u"], g["mu_v"], nx, ny, dx, dy))
    assert np.all(s0 == 0.0)


def test_gradient_oracle_pinned_to_reference():
    from oracle import ref2d

    gd = golden("gradient.npz")
    nx, ny, dx, dy = gd["grid"]
    out = ref2d.gradient_ensemble(gd["members"], int(nx), int(ny), float(dx), float(dy))
    assert np.array_equal(out, gd["out"])
    m0 = gd["members"][0]
    assert np.array_equal(ref2d.velocity_magnitude(m0[0], m0[1]), gd["vmag0"])


@pytest.mark.parametrize("name", ["ens_a", "ens_b", "ens_c", "ens_d"])
def test_divuq1_oracle_pinned_to_reference_files(name):
    import os

    from conftest import GOLDEN
    from oracle import divuq1

    path = os.path.join(GOLDEN, f"divuq1_{name}.duq")
    (nx, ny, dx, dy), planes = divuq1.read_members(path)
    raw = open(path, "rb").read()
    hdr = divuq1.header(nx, ny, dx, dy, planes.shape[0])
    assert raw == hdr + planes.astype("<f4").tobytes()


# --------------------------------------------------------------------------
# the reference's own MC stream (oracle/refstream.py) vs the reference itself
# --------------------------------------------------------------------------

def test_refstream_oracle_bitwise_vs_reference_golden():
    from oracle import refstream

    g = golden("mc_refstream.npz")
    for i, seed in enumerate(g["seeds"]):
        assert np.array_equal(refstream.normal_stream(int(seed), g["counters"]), g["normals"][i])
    for c in "abc":
        nx, ny, dx, dy, n, seed = g[f"mc_{c}_grid"]
        m = g[f"mc_{c}_model"]
        mean, std = refstream.mc_divergence(m[0], m[1], m[2], m[3], int(nx), int(ny), dx, dy,
                                            int(n), int(seed))
        assert np.array_equal(mean, g[f"mc_{c}_mean"]) and np.array_equal(std, g[f"mc_{c}_std"])
    fig1 = ((5.98, 0.96), (6.40, 0.38), (6.50, 0.94), (4.30, 0.65))
    assert np.array_equal(refstream.sample_divergence_1d(fig1, (1.0, 1.0), 5000, 7), g["s1d_values"])
    e, c = refstream.mc_histogram_1d(fig1, (1.0, 1.0), 20000, 7, 50)
    assert np.array_equal(e, g["hist_edges"]) and np.array_equal(c, g["hist_counts"])
    e, c = refstream.mc_histogram_1d(((1.0, 0.0), (2.0, 0.0), (3.0, 0.0), (4.0, 0.0)),
                                     (1.0, 1.0), 500, 0, 10)
    assert np.array_equal(e, g["hist0_edges"]) and np.array_equal(c, g["hist0_counts"])


def test_mc_histogram_type_invariants():
    import paper_2510_01190_b200 as d

    with pytest.raises(ValueError):
        d.McHistogram(np.array([0.0, 0.0, 1.0]), np.array([1, 1]), 2)
    with pytest.raises(ValueError):
        d.McHistogram(np.array([0.0, 1.0]), np.array([3]), 2)
    h = d.McHistogram(np.array([0.0, 1.0, 3.0]), np.array([1, 1]), 2)
    assert np.allclose(h.normalized_density(), [0.5, 0.25])
