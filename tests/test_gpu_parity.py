"""GPU parity: the sm_100a kernels against the pinned CPU oracle.

Bars (BASELINE.json north star):
* fp64 analytic mu / sigma / moments: BITWISE (reference op order, no FMA);
* fp64 probabilities: |dP| <= 1e-12 * P where P > 1e-300 (the GPU erfc is
  not scipy's cephes erfc; both keep ndtr's structure);
* fp32 fields: normwise max|d| / max|ref| <= 1e-5 against the fp64 oracle on
  the same fp32 inputs; fp32 probabilities |dP| <= 1e-5 * P + 1e-6.
"""

import numpy as np
import pytest

from conftest import golden, random_model_arrays

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import philox, ref2d, ref3d  # noqa: E402


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__

    __graft_entry__.build()
    from paper_2510_01190_b200 import device

    return device


def cu(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def host(t):
    return t.cpu().numpy()


def assert_p_close(got, ref, rtol=1e-12):
    got, ref = np.asarray(got), np.asarray(ref)
    m = ref > 1e-300
    assert np.all(np.abs(got[m] - ref[m]) <= rtol * ref[m]), np.max(np.abs(got[m] - ref[m]) / ref[m])
    # below the floor both must be (sub)normal-tiny
    assert np.all(got[~m] <= 1e-290)


def normwise(got, ref):
    return np.max(np.abs(np.asarray(got, np.float64) - ref)) / max(np.max(np.abs(ref)), 1e-300)


# --------------------------------------------------------------------------
# 2D analytic, fp64 -- bitwise against the reference's own outputs
# --------------------------------------------------------------------------

def test_propagate2d_f64_bitwise_vs_reference_golden(dev):
    g = golden("propagate2d.npz")
    for gi in range(int(g["n_grids"])):
        nx, ny, dx, dy = g[f"g{gi}_grid"]
        nx, ny = int(nx), int(ny)
        ins = [cu(g[f"g{gi}_{k}"]) for k in ("mu_u", "mu_v", "s_u", "s_v")]
        for t in (0.0, 0.3):
            o = dev.propagate2d(*ins, nx, ny, dx, dy, t)
            assert np.array_equal(host(o["mu"]), g[f"g{gi}_out_mu"]), gi
            assert np.array_equal(host(o["sigma"]), g[f"g{gi}_out_sigma"]), gi
            assert_p_close(host(o["p_src"]), g[f"g{gi}_t{t}_above"])
            assert_p_close(host(o["p_snk"]), g[f"g{gi}_t{t}_below_neg"])
        det = dev.propagate2d(ins[0], ins[1], None, None, nx, ny, dx, dy, outputs=("mu",))
        assert np.array_equal(host(det["mu"]), g[f"g{gi}_det"])


def test_dropin_api_bitwise_vs_reference_golden(dev):
    import paper_2510_01190_b200 as d

    g = golden("propagate2d.npz")
    for gi in range(int(g["n_grids"])):
        nx, ny, dx, dy = g[f"g{gi}_grid"]
        grid = d.UniformGrid2(int(nx), int(ny), float(dx), float(dy))
        model = d.GaussianVectorField(grid, *(g[f"g{gi}_{k}"] for k in ("mu_u", "mu_v", "s_u", "s_v")))
        out = d.propagate_divergence(model, d.ParallelConfig(threads=4))
        assert isinstance(out, d.GaussianScalarField)
        assert np.array_equal(out.mu, g[f"g{gi}_out_mu"])
        assert np.array_equal(out.sigma, g[f"g{gi}_out_sigma"])
        det = d.divergence_deterministic(model.mean_field())
        assert np.array_equal(det.values, g[f"g{gi}_det"])
        res = d.propagate_with_probabilities(model, 0.3)
        assert np.array_equal(res.field.mu, g[f"g{gi}_out_mu"])
        assert_p_close(res.p_src, g[f"g{gi}_t0.3_above"])
        assert_p_close(res.p_snk, g[f"g{gi}_t0.3_below_neg"])
        assert_p_close(d.source_probability(out, 0.3), g[f"g{gi}_t0.3_above"])
        assert_p_close(d.sink_probability(out, 0.3), g[f"g{gi}_t0.3_below_neg"])


def test_fig1_and_uniform_sigma(dev):
    import paper_2510_01190_b200 as d

    fig1 = golden("fig1.npz")
    g = d.UniformGrid2(3, 3)
    mu_u, mu_v, sg_u, sg_v = (np.zeros(9) for _ in range(4))
    nb = fig1["neighbors"]
    (mu_u[3], sg_u[3]), (mu_u[5], sg_u[5]) = nb[0], nb[1]
    (mu_v[1], sg_v[1]), (mu_v[7], sg_v[7]) = nb[2], nb[3]
    out = d.propagate_divergence(d.GaussianVectorField(g, mu_u, mu_v, sg_u, sg_v))
    assert abs(out.mu[4] - (-0.89)) <= 1e-12
    assert out.sigma[4] == float(fig1["sigma"])  # 0.7700811645534514
    # uniform sigma: interior sigma = s/h at rtol 1e-15 (test_divergence.py:117-124)
    s, h = 0.4, 0.5
    g = d.UniformGrid2(5, 5, h, h)
    out = d.propagate_divergence(d.GaussianVectorField(g, np.zeros(25), np.zeros(25),
                                                       np.full(25, s), np.full(25, s)))
    assert np.allclose(out.sigma.reshape(5, 5)[1:-1, 1:-1], s / h, rtol=1e-15)


def test_identity_rotation_and_zero_sigma(dev):
    for nx, ny, dx, dy in ((12, 9, 0.4, 1.7), (10, 11, 0.5, 0.25), (64, 33, 0.5, 0.25)):
        i = np.arange(nx * ny) % nx * dx
        j = np.arange(nx * ny) // nx * dy
        o = dev.propagate2d(cu(i), cu(j), None, None, nx, ny, dx, dy, outputs=("mu",))
        assert np.allclose(host(o["mu"]), 2.0, rtol=0, atol=1e-12)
        o = dev.propagate2d(cu(-j), cu(i), None, None, nx, ny, dx, dy, outputs=("mu",))
        assert np.all(host(o["mu"]) == 0.0)
    rng = np.random.default_rng(1)
    nx = ny = 9
    u, v = rng.normal(size=(2, 81))
    z = np.zeros(81)
    o = dev.propagate2d(cu(u), cu(v), cu(z), cu(z), nx, ny, 0.7, 0.2, 0.0)
    assert np.all(host(o["sigma"]) == 0.0)
    assert np.array_equal(host(o["mu"]), ref2d.divergence2d(u, v, nx, ny, 0.7, 0.2))
    # sigma == 0 tails are a step with mu == theta counted below (lcp.py:56-59)
    ps, pk = host(o["p_src"]), host(o["p_snk"])
    mu = host(o["mu"])
    assert np.array_equal(ps, np.where(mu <= 0.0, 0.0, 1.0))
    assert np.array_equal(pk, np.where(mu <= 0.0, 1.0, 0.0))


@pytest.mark.parametrize("shape", [(2, 2), (2, 9), (9, 2), (31, 17), (128, 128), (130, 66), (257, 3)])
def test_propagate2d_f64_shapes_and_vector_paths(dev, shape, rng):
    nx, ny = shape
    a = random_model_arrays(nx * ny, rng)
    o = dev.propagate2d(*(cu(x) for x in a), nx, ny, 0.6, 1.3, 0.1)
    mu, sg = ref2d.propagate2d(*a, nx, ny, 0.6, 1.3)
    assert np.array_equal(host(o["mu"]), mu)
    assert np.array_equal(host(o["sigma"]), sg)
    assert_p_close(host(o["p_src"]), ref2d.source_probability(mu, sg, 0.1))
    assert_p_close(host(o["p_snk"]), ref2d.sink_probability(mu, sg, 0.1))


@pytest.mark.parametrize("shape", [(2, 2), (31, 17), (128, 96), (1024, 64)])
def test_propagate2d_f32_tolerance(dev, shape, rng):
    nx, ny = shape
    a = [x.astype(np.float32) for x in random_model_arrays(nx * ny, rng)]
    o = dev.propagate2d(*(cu(x) for x in a), nx, ny, 1.0, 1.0, 0.0)
    mu, sg = ref2d.propagate2d(*a, nx, ny, 1.0, 1.0)
    assert normwise(host(o["mu"]), mu) <= 1e-5
    assert normwise(host(o["sigma"]), sg) <= 1e-5
    ps = ref2d.source_probability(mu, sg, 0.0)
    assert np.all(np.abs(host(o["p_src"]) - ps) <= 1e-5 * ps + 1e-6)


def test_tail_probs_golden(dev):
    g = golden("tail_probs.npz")
    mu, sg = cu(g["mu"]), cu(g["sigma"])
    for t in (0.0, 0.1, 0.3, -0.7):
        b, a = dev.tail_probs(mu, sg, t)
        assert_p_close(host(b), g[f"t{t}_below"])
        assert_p_close(host(a), g[f"t{t}_above"])
        deg = g["sigma"] == 0
        assert np.array_equal(host(b)[deg], g[f"t{t}_below"][deg])


def test_negation_symmetry_exact(dev, rng):
    # both tails evaluated directly (lcp.py:1-12): P_above(-mu, -theta) == P_below(mu, theta)
    mu = rng.normal(0, 3, 50000)
    sg = rng.uniform(0.001, 5, 50000)
    b, a = dev.tail_probs(cu(mu), cu(sg), 0.37)
    b2, a2 = dev.tail_probs(cu(-mu), cu(sg), -0.37)
    assert np.array_equal(host(b), host(a2)) and np.array_equal(host(a), host(b2))


# --------------------------------------------------------------------------
# ensemble moments (K1), fp64 bitwise
# --------------------------------------------------------------------------

def test_fit_gaussian_bitwise_vs_reference_golden(dev):
    import paper_2510_01190_b200 as d

    g = golden("fit_gaussian.npz")
    for ci in range(int(g["n_cases"])):
        mem = g[f"c{ci}_members"]
        mu, sg = dev.fit_moments(cu(mem))
        assert np.array_equal(host(mu)[0], g[f"c{ci}_mu_u"]) and np.array_equal(host(mu)[1], g[f"c{ci}_mu_v"])
        assert np.array_equal(host(sg)[0], g[f"c{ci}_s_u"]) and np.array_equal(host(sg)[1], g[f"c{ci}_s_v"])
    mem = g["syn_members"]
    m, _, n = mem.shape
    grid = d.UniformGrid2(24, 20)
    ens = d.Ensemble2(grid, tuple(d.VectorField2(grid, mem[k, 0], mem[k, 1]) for k in range(m)))
    model = d.fit_gaussian(ens)
    assert np.array_equal(model.mu_u, g["syn_mu_u"]) and np.array_equal(model.sigma_v, g["syn_s_v"])
    out = d.propagate_divergence(model)
    assert np.array_equal(out.mu, g["syn_div_mu"]) and np.array_equal(out.sigma, g["syn_div_sigma"])


@pytest.mark.parametrize("m", [2, 3, 16, 20, 33, 40])
def test_fit_moments_member_counts(dev, m, rng):
    mem = rng.normal(1.0, 0.5, (m, 3, 1001))
    mu, sg = dev.fit_moments(cu(mem))
    mu_r, sg_r = ref2d.fit_moments(mem)
    assert np.array_equal(host(mu), mu_r) and np.array_equal(host(sg), sg_r)
    mem32 = mem.astype(np.float32)
    mu, sg = dev.fit_moments(cu(mem32))
    mu_r, sg_r = ref2d.fit_moments(mem32)
    assert normwise(host(mu), mu_r) <= 1e-5 and normwise(host(sg), sg_r) <= 1e-5


# --------------------------------------------------------------------------
# 3D analytic
# --------------------------------------------------------------------------

def _model3d(nx, ny, nz, rng, dtype=np.float64):
    n = nx * ny * nz
    f = [rng.normal(size=n) for _ in range(3)] + [rng.uniform(0.05, 0.3, n) for _ in range(3)]
    return [x.astype(dtype) for x in f]


@pytest.mark.parametrize("shape", [(2, 2, 2), (7, 5, 13), (64, 8, 9), (130, 20, 6)])
def test_propagate3d_f64_bitwise(dev, shape, rng):
    nx, ny, nz = shape
    f = _model3d(nx, ny, nz, rng)
    o = dev.propagate3d(*(cu(x) for x in f), nx, ny, nz, 0.3, 0.7, 1.1, 0.05)
    mu, sg = ref3d.propagate3d(*f, nx, ny, nz, 0.3, 0.7, 1.1)
    assert np.array_equal(host(o["mu"]), mu)
    assert np.array_equal(host(o["sigma"]), sg)
    assert_p_close(host(o["p_src"]), ref2d.source_probability(mu, sg, 0.05))
    assert_p_close(host(o["p_snk"]), ref2d.sink_probability(mu, sg, 0.05))


@pytest.mark.parametrize("shape", [(32, 16, 40), (128, 24, 17), (33, 9, 5)])
def test_propagate3d_f32_tolerance(dev, shape, rng):
    nx, ny, nz = shape
    f = _model3d(nx, ny, nz, rng, np.float32)
    o = dev.propagate3d(*(cu(x) for x in f), nx, ny, nz, 1.0, 1.0, 1.0, 0.0)
    mu, sg = ref3d.propagate3d(*f, nx, ny, nz, 1.0, 1.0, 1.0)
    assert normwise(host(o["mu"]), mu) <= 1e-5
    assert normwise(host(o["sigma"]), sg) <= 1e-5
    ps = ref2d.source_probability(mu, sg, 0.0)
    pk = ref2d.sink_probability(mu, sg, 0.0)
    assert np.all(np.abs(host(o["p_src"]) - ps) <= 1e-5 * ps + 1e-6)
    assert np.all(np.abs(host(o["p_snk"]) - pk) <= 1e-5 * pk + 1e-6)


def test_propagate3d_identity_and_planar_reduction(dev):
    nx, ny, nz, dx, dy, dz = 40, 12, 9, 0.5, 0.25, 2.0
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    x, y, z = (i * dx).ravel(), (j * dy).ravel(), (k * dz).ravel()
    zero = np.zeros_like(x)
    o = dev.propagate3d(cu(x), cu(y), cu(z), cu(zero), cu(zero), cu(zero), nx, ny, nz, dx, dy, dz,
                        outputs=("mu",))
    assert np.all(host(o["mu"]) == 3.0)
    # z-invariant field with w = 0 reduces bitwise to the 2D reference
    g = golden("propagate2d.npz")
    gi = 6
    gnx, gny, gdx, gdy = g[f"g{gi}_grid"]
    gnx, gny = int(gnx), int(gny)
    tile = lambda a: np.tile(a, 4)
    z = np.zeros(gnx * gny * 4)
    o = dev.propagate3d(cu(tile(g[f"g{gi}_mu_u"])), cu(tile(g[f"g{gi}_mu_v"])), cu(z),
                        cu(tile(g[f"g{gi}_s_u"])), cu(tile(g[f"g{gi}_s_v"])), cu(z),
                        gnx, gny, 4, gdx, gdy, 0.9)
    for kk in range(4):
        sl = slice(kk * gnx * gny, (kk + 1) * gnx * gny)
        assert np.array_equal(host(o["mu"])[sl], g[f"g{gi}_out_mu"])
        assert np.array_equal(host(o["sigma"])[sl], g[f"g{gi}_out_sigma"])


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_propagate3d_slabs_and_k_ranges_bitwise(dev, dtype, rng):
    """z-slab decomposition with halo planes == whole-domain run, bit for bit
    (the multi-GPU correctness contract, emulated on one GPU)."""
    nx, ny, nz = 64, 10, 23
    plane = nx * ny
    f = _model3d(nx, ny, nz, rng, dtype)
    full = dev.propagate3d(*(cu(x) for x in f), nx, ny, nz, 0.5, 0.5, 0.5, 0.1)
    full = {k: host(v) for k, v in full.items()}
    for parts in (2, 3, 8):
        bounds = [nz * r // parts for r in range(parts + 1)]
        for r in range(parts):
            z0, z1 = bounds[r], bounds[r + 1]
            sl = [cu(x[z0 * plane:z1 * plane]) for x in f]
            lo = (cu(f[2][(z0 - 1) * plane:z0 * plane]), cu(f[5][(z0 - 1) * plane:z0 * plane])) if z0 else None
            hi = (cu(f[2][z1 * plane:(z1 + 1) * plane]), cu(f[5][z1 * plane:(z1 + 1) * plane])) if z1 < nz else None
            o = dev.propagate3d(*sl, nx, ny, z1 - z0, 0.5, 0.5, 0.5, 0.1, z0=z0, nz_global=nz,
                                halo_lo=lo, halo_hi=hi)
            for k in o:
                assert np.array_equal(host(o[k]), full[k][z0 * plane:z1 * plane]), (parts, r, k)
    # interior / edge split (the overlap schedule): two launches, same bits
    ins = [cu(x) for x in f]
    out = {k: torch.full((nx * ny * nz,), -7.0, dtype=ins[0].dtype, device="cuda") for k in full}
    dev.propagate3d(*ins, nx, ny, nz, 0.5, 0.5, 0.5, 0.1, k_range=(1, nz - 1), out=out)
    dev.propagate3d(*ins, nx, ny, nz, 0.5, 0.5, 0.5, 0.1, k_range=(0, 1), out=out)
    dev.propagate3d(*ins, nx, ny, nz, 0.5, 0.5, 0.5, 0.1, k_range=(nz - 1, nz), out=out)
    for k in out:
        assert np.array_equal(host(out[k]), full[k])


# --------------------------------------------------------------------------
# fused ensemble kernels (K3)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("m,shape", [(20, (256, 40)), (2, (33, 7)), (16, (128, 17)), (40, (64, 9)),
                                     # row-march edges: partial strips, both x edges in one
                                     # lane, 2-3 row runs, segment boundaries, many members
                                     (3, (4, 2)), (20, (68, 5)), (5, (100, 200)), (20, (132, 3)),
                                     (20, (1024, 64)), (30, (192, 130))])
def test_ensemble_divergence2d(dev, m, shape, rng, monkeypatch):
    nx, ny = shape
    n = nx * ny
    base = rng.normal(0, 1, (1, 2, n))
    mem = (base + rng.normal(0, 0.3, (m, 2, n))).astype(np.float32)
    o = dev.ensemble_divergence2d(cu(mem), nx, ny, 0.5, 0.5, 0.0, moments=True)
    mu_r, sg_r = ref2d.fit_moments(mem)
    assert normwise(host(o["mom_mu"]), mu_r) <= 1e-5
    assert normwise(host(o["mom_sigma"]), sg_r) <= 1e-5
    dmu, dsg = ref2d.propagate2d(mu_r[0], mu_r[1], sg_r[0], sg_r[1], nx, ny, 0.5, 0.5)
    assert normwise(host(o["mu"]), dmu) <= 1e-5
    assert normwise(host(o["sigma"]), dsg) <= 1e-5
    ps = ref2d.source_probability(dmu, dsg, 0.0)
    assert np.all(np.abs(host(o["p_src"]) - ps) <= 1e-5 * ps + 1e-6)
    # the fused moments are K1's, bit for bit
    mu_g, sg_g = dev.fit_moments(cu(mem))
    assert np.array_equal(host(o["mom_mu"]), host(mu_g))
    assert np.array_equal(host(o["mom_sigma"]), host(sg_g))
    # every fused path (row march, tiled K3, K1 triples + residual stencil)
    # differences the same (mu, r) pairs: identical maps
    for env in ("DIVUQ_NO_ROWMARCH", "DIVUQ_NO_TMA"):
        monkeypatch.setenv(env, "1")
        o2 = dev.ensemble_divergence2d(cu(mem), nx, ny, 0.5, 0.5, 0.0, moments=True)
        monkeypatch.delenv(env)
        for k in o:
            assert np.array_equal(host(o[k]), host(o2[k])), (env, k)


@pytest.mark.parametrize("m", [16, 5])
def test_ensemble_divergence3d_and_slabs(dev, m, rng, monkeypatch):
    nx, ny, nz = 64, 12, 14
    plane = nx * ny
    n = plane * nz
    mem = (rng.normal(0, 1, (1, 3, n)) + rng.normal(0, 0.3, (m, 3, n))).astype(np.float32)
    gm = cu(mem)
    full = dev.ensemble_divergence3d(gm, nx, ny, nz, 1.0, 1.0, 1.0, 0.1, moments=True)
    mu_r, sg_r = ref2d.fit_moments(mem)
    assert normwise(host(full["mom_mu"]), mu_r) <= 1e-5
    dmu, dsg = ref3d.propagate3d(*mu_r, *sg_r, nx, ny, nz, 1.0, 1.0, 1.0)
    assert normwise(host(full["mu"]), dmu) <= 1e-5
    assert normwise(host(full["sigma"]), dsg) <= 1e-5
    pk = ref2d.sink_probability(dmu, dsg, 0.1)
    assert np.all(np.abs(host(full["p_snk"]) - pk) <= 1e-5 * pk + 1e-6)
    # the fused moments are K1's; the fallback (K1 triples + residual stencil)
    # gives the same maps bit for bit
    mu_g, sg_g = dev.fit_moments(gm)
    assert np.array_equal(host(full["mom_mu"]), host(mu_g))
    monkeypatch.setenv("DIVUQ_NO_TMA", "1")
    o2 = dev.ensemble_divergence3d(gm, nx, ny, nz, 1.0, 1.0, 1.0, 0.1, moments=True)
    monkeypatch.delenv("DIVUQ_NO_TMA")
    for k in full:
        assert np.array_equal(host(full[k]), host(o2[k])), k
    # slabs with reduced w-moment halos == whole domain, bitwise
    for parts in (2, 3):
        bounds = [nz * r // parts for r in range(parts + 1)]
        for r in range(parts):
            z0, z1 = bounds[r], bounds[r + 1]
            sl = gm[:, :, z0 * plane:z1 * plane].contiguous()
            lo = dev.w_moments_plane(gm, nx, ny, nz, z0 - 1) if z0 else None
            hi = dev.w_moments_plane(gm, nx, ny, nz, z1) if z1 < nz else None
            o = dev.ensemble_divergence3d(sl, nx, ny, z1 - z0, 1.0, 1.0, 1.0, 0.1, z0=z0,
                                          nz_global=nz, halo_lo=lo, halo_hi=hi)
            for k in ("mu", "sigma", "p_src", "p_snk"):
                assert np.array_equal(host(o[k]), host(full[k])[z0 * plane:z1 * plane]), (parts, r, k)


@pytest.mark.parametrize("chunk", [1, 3, 5, 32])
def test_host_propagate3d_pipeline(dev, chunk, rng):
    """Host-buffer 3D propagation (3-stream z-chunk pipeline; halo planes read
    from the neighbour chunks in HBM) == the device K2 call, bitwise, for any
    chunking; the reference-facing wrapper returns the same maps."""
    import paper_2510_01190_b200 as d

    nx, ny, nz = 64, 9, 13
    n = nx * ny * nz
    f = [rng.normal(size=n).astype(np.float32) for _ in range(3)] + \
        [rng.uniform(0.05, 0.4, n).astype(np.float32) for _ in range(3)]
    whole = dev.propagate3d(*(cu(x) for x in f), nx, ny, nz, 1.0, 0.5, 2.0, 0.1)
    g = d.UniformGrid3(nx, ny, nz, 1.0, 0.5, 2.0)
    model = d.GaussianVectorField3(g, *f)
    r = d.propagate_with_probabilities3d(model, 0.1, chunk_planes=chunk)
    for k, a in (("mu", r.field.mu), ("sigma", r.field.sigma), ("p_src", r.p_src), ("p_snk", r.p_snk)):
        assert np.array_equal(a, host(whole[k])), (chunk, k)


@pytest.mark.parametrize("chunk", [0, 1, 3, 5])
def test_host_ensemble_divergence3d_pipeline(dev, chunk, rng):
    """Host-buffer 3D ensemble entry (3-stream z-chunk pipeline, halos fitted
    from the neighbour chunks in HBM) == the device fused kernel, bitwise, for
    any chunking and for slabs fed host ghost planes (strided views)."""
    import paper_2510_01190_b200 as d

    nx, ny, nz, m = 48, 10, 13, 6
    plane = nx * ny
    n = plane * nz
    mem = (rng.normal(0, 1, (1, 3, n)) + rng.normal(0, 0.3, (m, 3, n))).astype(np.float32)
    full = dev.ensemble_divergence3d(cu(mem), nx, ny, nz, 1.0, 0.5, 2.0, 0.1)
    g = d.UniformGrid3(nx, ny, nz, 1.0, 0.5, 2.0)
    r = d.ensemble_divergence3d(mem, g, 0.1, chunk_planes=chunk)
    got = {"mu": r.field.mu, "sigma": r.field.sigma, "p_src": r.p_src, "p_snk": r.p_snk}
    for k in ("mu", "sigma", "p_src", "p_snk"):
        assert np.array_equal(got[k], host(full[k])), (chunk, k)
    mu_r, sg_r = ref2d.fit_moments(mem)
    dmu, dsg = ref3d.propagate3d(*mu_r, *sg_r, nx, ny, nz, 1.0, 0.5, 2.0)
    assert normwise(got["mu"], dmu) <= 1e-5 and normwise(got["sigma"], dsg) <= 1e-5
    # z-slabs with host ghost planes, ghosts passed as strided views of mem
    bounds = [0, 4, 9, nz]
    for z0, z1 in zip(bounds[:-1], bounds[1:]):
        sl = np.ascontiguousarray(mem[:, :, z0 * plane:z1 * plane])
        lo = mem[:, 2, (z0 - 1) * plane:z0 * plane] if z0 else None
        hi = mem[:, 2, z1 * plane:(z1 + 1) * plane] if z1 < nz else None
        gs = d.UniformGrid3(nx, ny, z1 - z0, 1.0, 0.5, 2.0)
        rs = d.ensemble_divergence3d(sl, gs, 0.1, z0=z0, nz_global=nz, ghost_lo=lo, ghost_hi=hi,
                                     chunk_planes=chunk)
        for k, a in (("mu", rs.field.mu), ("sigma", rs.field.sigma), ("p_src", rs.p_src),
                     ("p_snk", rs.p_snk)):
            assert np.array_equal(a, host(full[k])[z0 * plane:z1 * plane]), (chunk, z0, k)
    with pytest.raises(ValueError):   # interior slab without its ghost planes
        d.ensemble_divergence3d(mem[:, :, plane:3 * plane], d.UniformGrid3(nx, ny, 2, 1.0, 0.5, 2.0),
                                z0=1, nz_global=nz)


# --------------------------------------------------------------------------
# Monte Carlo (K4)
# --------------------------------------------------------------------------

def _mc_model():
    g = golden("mc_ref.npz")
    nx, ny, dx, dy = g["grid"]
    return g, int(nx), int(ny), float(dx), float(dy)


def test_mc_matches_philox_oracle_same_stream(dev):
    g, nx, ny, dx, dy = _mc_model()
    ins = [cu(g[k]) for k in ("mu_u", "mu_v", "s_u", "s_v")]
    # 4396 and 12345: more 128-sample chunks than the 32 slots, so slots fold
    # several chunks with Chan's formula before the cross-slot merge
    for n in (2, 300, 513, 4396, 12345):
        mean, std = dev.mc_divergence2d(*ins, nx, ny, dx, dy, n, 77)
        om, os_ = philox.mc_divergence(g["mu_u"], g["mu_v"], g["s_u"], g["s_v"], nx, ny, dx, dy, n, 77)
        # same counters and merge order; only libdevice vs numpy log/sincos ulps differ
        assert np.allclose(host(mean), om, rtol=1e-11, atol=1e-11)
        assert np.allclose(host(std), os_, rtol=1e-9, atol=1e-11)


def test_mc_statistics_vs_analytic_and_reference(dev):
    g, nx, ny, dx, dy = _mc_model()
    n = int(g["n_samples"])
    ins = [cu(g[k]) for k in ("mu_u", "mu_v", "s_u", "s_v")]
    mean, std = dev.mc_divergence2d(*ins, nx, ny, dx, dy, n, 5)
    mean, std = host(mean), host(std)
    s = g["an_sigma"]
    # SURVEY 8d's MC gate: >= 99.9 % of vertices within 4 sigma / sqrt(N)
    assert np.mean(np.abs(mean - g["an_mu"]) <= 4 * s / np.sqrt(n)) >= 0.999
    assert np.mean(np.abs(std - s) <= 4 * s / np.sqrt(2 * n)) >= 0.999
    assert np.mean(np.abs(mean - g["mean"]) <= 4 * np.sqrt(2) * s / np.sqrt(n)) >= 0.99
    z = (mean - g["an_mu"]) / (s / np.sqrt(n))
    assert abs(z.mean()) < 0.5 and 0.5 < z.var() < 1.6


def test_mc_zero_sigma_exact_determinism_and_sharding(dev, rng):
    nx, ny = 37, 21
    u, v = rng.normal(size=(2, nx * ny))
    z = np.zeros(nx * ny)
    mean, std = dev.mc_divergence2d(cu(u), cu(v), cu(z), cu(z), nx, ny, 0.5, 0.7, 300, 9)
    assert np.array_equal(host(mean), ref2d.divergence2d(u, v, nx, ny, 0.5, 0.7))
    assert np.all(host(std) == 0.0)
    a = random_model_arrays(nx * ny, rng)
    ins = [cu(x) for x in a]
    m1, s1 = dev.mc_divergence2d(*ins, nx, ny, 0.5, 0.7, 700, 1234)
    m2, s2 = dev.mc_divergence2d(*ins, nx, ny, 0.5, 0.7, 700, 1234)
    m3, _ = dev.mc_divergence2d(*ins, nx, ny, 0.5, 0.7, 700, 1235)
    assert torch.equal(m1, m2) and torch.equal(s1, s2) and not torch.equal(m1, m3)
    # row sharding (multi-GPU partition) is bit-identical
    parts = []
    for r0, r1 in ((0, 5), (5, 6), (6, 21)):
        pm, ps = dev.mc_divergence2d(*ins, nx, ny, 0.5, 0.7, 700, 1234, rows=(r0, r1))
        parts.append((pm, ps))
    assert torch.equal(torch.cat([p[0] for p in parts]), m1)
    assert torch.equal(torch.cat([p[1] for p in parts]), s1)


def test_mc_dropin_fig1_error_scale(dev):
    import paper_2510_01190_b200 as d

    fig1 = golden("fig1.npz")
    g = d.UniformGrid2(3, 3)
    mu_u, mu_v, sg_u, sg_v = (np.zeros(9) for _ in range(4))
    nb = fig1["neighbors"]
    (mu_u[3], sg_u[3]), (mu_u[5], sg_u[5]) = nb[0], nb[1]
    (mu_v[1], sg_v[1]), (mu_v[7], sg_v[7]) = nb[2], nb[3]
    model = d.GaussianVectorField(g, mu_u, mu_v, sg_u, sg_v)
    an = d.propagate_divergence(model)
    errs = [abs(d.mc_divergence(model, d.McConfig(1000, seed=s)).mean[4] - an.mu[4]) for s in range(10)]
    assert 3e-3 <= np.mean(errs) <= 3e-2  # test_mc.py:161-179 bracket
    est = d.mc_divergence(model, d.McConfig(100_000, seed=21))
    assert abs(est.std[4] / an.sigma[4] - 1) < 0.02
    e_m, e_s, sse = d.error_metrics(est, an)
    assert e_m >= 0 and e_s >= 0 and sse >= 0
    with pytest.raises(ValueError):
        d.mc_divergence(model, d.McConfig(1))


@pytest.mark.parametrize("n", [1, 7, 1000, 65536, 3_000_001])
def test_error_metrics_on_device(dev, rng, n):
    """error_metrics (mc.py:159-175) as one device reduction: within 1e-13
    relative of the reference's numpy formula, deterministic run to run,
    and the drop-in keeps the reference's grid-mismatch ValueError."""
    import paper_2510_01190_b200 as d

    em, es, mu, sg = rng.normal(size=n), rng.uniform(0.5, 1.5, n), rng.normal(size=n), rng.uniform(0.5, 1.5, n)
    t = [cu(x) for x in (em, es, mu, sg)]
    got = dev.error_metrics(*t)
    again = dev.error_metrics(*t)
    assert torch.equal(got, again)
    dm, ds = em - mu, es - sg
    want = np.array([np.abs(dm).mean(), np.abs(ds).mean(), np.sum(dm**2) + np.sum(ds**2)])
    assert np.allclose(host(got), want, rtol=1e-13, atol=0)
    if n == 1000:
        g = d.UniformGrid2(40, 25)
        est = d.McDivergenceEstimate(g, em, es, 10)
        an = d.GaussianScalarField(g, mu, sg)
        assert np.allclose(d.error_metrics(est, an), want, rtol=1e-13, atol=0)
        with pytest.raises(ValueError):
            d.error_metrics(est, d.GaussianScalarField(d.UniformGrid2(25, 40), mu, sg))


# --------------------------------------------------------------------------
# validation word -> reference exceptions
# --------------------------------------------------------------------------

def test_device_validation_raises(dev, rng):
    nx, ny = 16, 8
    a = [x.copy() for x in random_model_arrays(nx * ny, rng)]
    a[0][5] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        dev.propagate2d(*(cu(x) for x in a), nx, ny)
    a = [x.copy() for x in random_model_arrays(nx * ny, rng)]
    a[3][7] = -0.1
    with pytest.raises(ValueError, match="non-negative"):
        dev.propagate2d(*(cu(x) for x in a), nx, ny)
    with pytest.raises(ValueError):
        dev.propagate2d(*(cu(x) for x in random_model_arrays(2, rng)), 1, 2)
    mem = rng.normal(size=(4, 3, 512)).astype(np.float32)
    mem[2, 2, 100] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        dev.ensemble_divergence3d(cu(mem), 16, 8, 4)
    with pytest.raises(ValueError):
        dev.fit_moments(cu(rng.normal(size=(1, 2, 10))))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_tma_pipeline_matches_register_kernel_bitwise(dev, dtype, rng, monkeypatch):
    """The TMA/mbarrier K2 and the register-prefetch K2 are the same arithmetic."""
    nx, ny, nz = 256, 40, 21
    f = _model3d(nx, ny, nz, rng, dtype)
    ins = [cu(x) for x in f]
    for t in (0.0, 0.25):
        a = dev.propagate3d(*ins, nx, ny, nz, 0.5, 1.5, 0.75, t)
        monkeypatch.setenv("DIVUQ_NO_TMA", "1")
        b = dev.propagate3d(*ins, nx, ny, nz, 0.5, 1.5, 0.75, t)
        monkeypatch.delenv("DIVUQ_NO_TMA")
        for k in a:
            assert torch.equal(a[k], b[k]), k


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("shape", [(131, 9, 7), (510, 17, 5), (3, 2, 4), (257, 30, 3), (65, 1 + 14, 6)])
def test_flat_tma_kernel_matches_generic_bitwise(dev, dtype, shape, rng, monkeypatch):
    """K2 on 1D tensor maps (k2flat.cuh: row pitch not a multiple of 16 bytes)
    == the generic register kernel bit for bit: whole domain, z-slabs with
    halo planes, k ranges, the deterministic (mean-only) variant."""
    nx, ny, nz = shape
    if dtype == np.float64 and nx % 2 == 0:
        nx += 1   # fp64 tiled maps take every even nx
    plane = nx * ny
    f = _model3d(nx, ny, nz, rng, dtype)
    ins = [cu(x) for x in f]

    def both(fn):
        a = fn()
        monkeypatch.setenv("DIVUQ_NO_FLAT", "1")
        b = fn()
        monkeypatch.delenv("DIVUQ_NO_FLAT")
        for k in a:
            assert torch.equal(a[k], b[k]), k
        return a

    for t in (0.0, 0.2):
        both(lambda: dev.propagate3d(*ins, nx, ny, nz, 0.5, 1.5, 0.75, t))
    both(lambda: dev.propagate3d(*ins, nx, ny, nz, 0.5, 1.5, 0.75, 0.0, outputs=("mu",)))
    if nz >= 4:
        z0, z1 = 1, nz - 1
        sl = [cu(x[z0 * plane:z1 * plane]) for x in f]
        lo = (cu(f[2][(z0 - 1) * plane:z0 * plane]), cu(f[5][(z0 - 1) * plane:z0 * plane]))
        hi = (cu(f[2][z1 * plane:(z1 + 1) * plane]), cu(f[5][z1 * plane:(z1 + 1) * plane]))
        full = dev.propagate3d(*ins, nx, ny, nz, 0.5, 1.5, 0.75, 0.1)
        o = both(lambda: dev.propagate3d(*sl, nx, ny, z1 - z0, 0.5, 1.5, 0.75, 0.1, z0=z0, nz_global=nz,
                                         halo_lo=lo, halo_hi=hi))
        for k in o:
            assert torch.equal(o[k], full[k][z0 * plane:z1 * plane]), k
    if dtype == np.float64:   # and the reference order, bit for bit
        o = dev.propagate3d(*ins, nx, ny, nz, 0.5, 1.5, 0.75, 0.0)
        mu, sg = ref3d.propagate3d(*f, nx, ny, nz, 0.5, 1.5, 0.75)
        assert np.array_equal(host(o["mu"]), mu) and np.array_equal(host(o["sigma"]), sg)


def test_flat_tma_kernel_unaligned_outputs_and_validation(dev, rng):
    """Aligned nx but outputs 4 bytes off a 16-byte boundary: the flat kernel
    (scalar stores) takes it; a negative sigma still raises."""
    nx, ny, nz = 128, 12, 6
    n = nx * ny * nz
    f = _model3d(nx, ny, nz, rng, np.float32)
    ins = [cu(x) for x in f]
    ref = dev.propagate3d(*ins, nx, ny, nz, 1.0, 1.0, 1.0, 0.0)
    buf = {k: torch.empty(n + 1, dtype=torch.float32, device="cuda") for k in ref}
    out = {k: v[1:] for k, v in buf.items()}
    dev.propagate3d(*ins, nx, ny, nz, 1.0, 1.0, 1.0, 0.0, out=out)
    for k in ref:
        assert torch.equal(out[k], ref[k]), k
    bad = [x.clone() for x in ins]
    bad[4][n // 3] = -0.5
    nx2 = 127
    with pytest.raises(ValueError):
        dev.propagate3d(*(x[: nx2 * ny * nz] for x in bad), nx2, ny, nz, 1.0, 1.0, 1.0, 0.0)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("shape", [(131, 9), (1023, 40), (3, 2), (257, 300), (3, 70001)])
def test_gather2d_matches_stencil_kernel_bitwise(dev, dtype, shape, rng, monkeypatch):
    """2D on unaligned rows runs the gather kernel (stencil.cuh); the
    z-marching register kernel is the same arithmetic, bit for bit: the
    analytic map (with and without sigma) and the fused-ensemble fallback's
    residual stencil."""
    nx, ny = shape
    n = nx * ny
    a = [rng.normal(0, 2, n), rng.normal(0, 2, n), rng.uniform(0.05, 0.6, n), rng.uniform(0.05, 0.6, n)]
    ins = [cu(x.astype(dtype)) for x in a]

    def both(fn):
        x = fn()
        monkeypatch.setenv("DIVUQ_NO_GATHER2D", "1")
        y = fn()
        monkeypatch.delenv("DIVUQ_NO_GATHER2D")
        for k in x:
            assert torch.equal(x[k], y[k]), k

    for t in (0.0, 0.3):
        both(lambda: dev.propagate2d(*ins, nx, ny, 0.7, 1.3, t))
    both(lambda: dev.propagate2d(*ins, nx, ny, 0.7, 1.3, 0.0, outputs=("mu",)))
    if dtype == np.float32 and nx % 4:
        mem = cu(rng.normal(size=(6, 2, n)).astype(np.float32))

        def fused():
            monkeypatch.setenv("DIVUQ_NO_ROWMARCH", "1")
            o = dev.ensemble_divergence2d(mem, nx, ny, 0.5, 0.5, 0.1, moments=True)
            monkeypatch.delenv("DIVUQ_NO_ROWMARCH")
            return o
        both(fused)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("shape", [(128, 40, 70), (127, 40, 70), (64, 16, 300)])
def test_zchunked_tma_kernels_bitwise(dev, dtype, shape, rng, monkeypatch):
    """Small planes (fewer tile columns than SMs): the TMA K2 / flat K2 / K3
    kernels split each column's z range into chunks that restart the
    z-march; the bits are the unchunked ones."""
    nx, ny, nz = shape
    f = _model3d(nx, ny, nz, rng, dtype)
    ins = [cu(x) for x in f]

    def both(fn):
        a = fn()
        monkeypatch.setenv("DIVUQ_NO_ZCHUNK", "1")
        b = fn()
        monkeypatch.delenv("DIVUQ_NO_ZCHUNK")
        for k in a:
            assert torch.equal(a[k], b[k]), k

    both(lambda: dev.propagate3d(*ins, nx, ny, nz, 0.5, 1.5, 0.75, 0.1))
    both(lambda: dev.propagate3d(*ins, nx, ny, nz, 0.5, 1.5, 0.75, 0.1, k_range=(3, nz - 2)))
    # a z-slab with halo planes, chunked: bitwise the whole-domain run's planes
    plane = nx * ny
    z0, z1 = 5, nz - 4
    full = dev.propagate3d(*ins, nx, ny, nz, 0.5, 1.5, 0.75, 0.1)
    sl = [cu(x[z0 * plane:z1 * plane]) for x in f]
    lo = (cu(f[2][(z0 - 1) * plane:z0 * plane]), cu(f[5][(z0 - 1) * plane:z0 * plane]))
    hi = (cu(f[2][z1 * plane:(z1 + 1) * plane]), cu(f[5][z1 * plane:(z1 + 1) * plane]))
    o = dev.propagate3d(*sl, nx, ny, z1 - z0, 0.5, 1.5, 0.75, 0.1, z0=z0, nz_global=nz, halo_lo=lo, halo_hi=hi)
    for k in o:
        assert torch.equal(o[k], full[k][z0 * plane:z1 * plane]), k
    if dtype == np.float32:
        mem = cu(rng.normal(size=(4, 3, nx * ny * nz)).astype(np.float32))
        both(lambda: dev.ensemble_divergence3d(mem, nx, ny, nz, 1.0, 1.0, 1.0, 0.1, moments=True))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("shape", [(640, 512), (1024, 600), (512, 1030)])
def test_tma2d_matches_register_kernels_bitwise(dev, dtype, shape, rng, monkeypatch):
    """Large 2D grids run the 3D TMA pipeline without w (K2Tma<T, *, false>);
    the register / gather kernels are the same arithmetic, bit for bit, and
    fp64 equals the reference order (oracle) bit for bit."""
    nx, ny = shape
    n = nx * ny
    a = [rng.normal(0, 2, n), rng.normal(0, 2, n), rng.uniform(0.05, 0.6, n), rng.uniform(0.05, 0.6, n)]
    ins = [cu(x.astype(dtype)) for x in a]

    def both(fn):
        x = fn()
        monkeypatch.setenv("DIVUQ_NO_TMA2D", "1")
        y = fn()
        monkeypatch.delenv("DIVUQ_NO_TMA2D")
        for k in x:
            assert torch.equal(x[k], y[k]), k
        return x

    for t in (0.0, 0.3):
        o = both(lambda: dev.propagate2d(*ins, nx, ny, 0.7, 1.3, t))
    both(lambda: dev.propagate2d(*ins, nx, ny, 0.7, 1.3, 0.0, outputs=("mu",)))
    if dtype == np.float64:
        mu, sg = ref2d.propagate2d(*a, nx, ny, 0.7, 1.3)
        assert np.array_equal(host(o["mu"]), mu) and np.array_equal(host(o["sigma"]), sg)
    bad = [x.clone() for x in ins]
    bad[3][n // 2] = -1.0
    with pytest.raises(ValueError):
        dev.propagate2d(*bad, nx, ny, 0.7, 1.3, 0.0)


@pytest.mark.parametrize("side", [68, 500, 1024])
def test_host_entry_staging_paths_bitwise(dev, side, rng):
    """The host-buffer entry points stage pageable spans through the pinned
    bounce arena (small calls) or the staged ring (large ones) and DMA pinned
    spans directly; any mix of pinned and pageable inputs/outputs, repeated
    calls on the warm arena, and the validation word read in the same sync
    give the device path's bits."""
    from paper_2510_01190_b200._lib import lib

    n = side * side
    mu_u, mu_v, s_u, s_v = random_model_arrays(n, rng)
    want = dev.propagate2d(cu(mu_u), cu(mu_v), cu(s_u), cu(s_v), side, side, 1.0, 1.0, 0.0)
    want = {k: host(v) for k, v in want.items()}
    pinned = [torch.from_numpy(a.copy()).pin_memory() for a in (mu_u, mu_v, s_u, s_v)]
    for mask in (0b0000, 0b0101, 0b1111):
        ins = [pinned[k].data_ptr() if mask >> k & 1 else a.__array_interface__["data"][0]
               for k, a in enumerate((mu_u, mu_v, s_u, s_v))]
        outs_np = [np.full(n, np.nan) for _ in range(4)]
        outs_pin = [torch.full((n,), float("nan"), dtype=torch.float64).pin_memory() for _ in range(4)]
        ptrs = [outs_pin[k].data_ptr() if mask >> k & 1 else outs_np[k].__array_interface__["data"][0]
                for k in range(4)]
        for _ in range(2):   # second call: warm arena / ring
            assert lib.divuq_host_propagate2d_f64(*ins, side, side, 1.0, 1.0, 0.0, *ptrs, 0) == 0
        got = [outs_pin[k].numpy() if mask >> k & 1 else outs_np[k] for k in range(4)]
        for k, key in enumerate(("mu", "sigma", "p_src", "p_snk")):
            assert np.array_equal(got[k], want[key]), (side, mask, key)
    bad = s_v.copy()
    bad[n // 2] = -1.0
    o = [np.empty(n) for _ in range(4)]
    st = lib.divuq_host_propagate2d_f64(*(a.__array_interface__["data"][0] for a in (mu_u, mu_v, s_u, bad)),
                                        side, side, 1.0, 1.0, 0.0,
                                        *(a.__array_interface__["data"][0] for a in o), 0)
    assert st != 0


def test_device_api_launches_on_torch_current_stream(dev, rng):
    """The device API enqueues on torch's current stream (raw-handle getter):
    same handle as the public object, inside a stream context too, and a
    launch on a side stream is ordered there."""
    assert dev._stream() == torch.cuda.current_stream().cuda_stream
    side = torch.cuda.Stream()
    n = 256 * 256
    arrs = [cu(a) for a in random_model_arrays(n, rng)]
    base = dev.propagate2d(*arrs, 256, 256, 1.0, 1.0, 0.0)
    with torch.cuda.stream(side):
        assert dev._stream() == side.cuda_stream
        side.wait_stream(torch.cuda.default_stream())
        o = dev.propagate2d(*arrs, 256, 256, 1.0, 1.0, 0.0, check=False)
    side.synchronize()
    for k in base:
        assert torch.equal(o[k], base[k])


def test_dropin_output_pool_never_hands_out_live_memory(dev, rng):
    """Large drop-in results are views of pooled pinned blocks (api._OutputPool):
    a block is reused only after every array (and view) of an earlier result
    is gone; results stay bitwise equal to fresh numpy outputs."""
    import paper_2510_01190_b200 as d
    from paper_2510_01190_b200 import api

    side = 1024
    g = d.UniformGrid2(side, side)
    model = d.GaussianVectorField(g, *random_model_arrays(side * side, rng))
    r1 = d.propagate_divergence(model)
    mu1, sg1 = r1.mu.copy(), r1.sigma.copy()
    assert r1.mu.base is not None and api._POOL._bytes > 0   # pooled, pinned
    r2 = d.propagate_divergence(model)
    assert not np.shares_memory(r1.mu, r2.mu) and not np.shares_memory(r1.sigma, r2.sigma)
    view = r2.mu[::3]
    keep = view.copy()
    del r2
    r3 = d.propagate_divergence(model)
    assert not np.shares_memory(view, r3.mu) and not np.shares_memory(view, r3.sigma)
    assert np.array_equal(view, keep)
    del view
    r4 = d.propagate_divergence(model)   # free blocks are reused from here on
    for r in (r1, r3, r4):
        assert np.array_equal(r.mu, mu1) and np.array_equal(r.sigma, sg1)
        assert not r.mu.flags.writeable
    p = d.source_probability(r4, 0.0)
    q = d.source_probability(r4, 0.0)
    assert not np.shares_memory(p, q) and np.array_equal(p, q)
    est = d.fit_gaussian(d.Ensemble2(g, tuple(d.VectorField2(g, *random_model_arrays(side * side, rng)[:2])
                                               for _ in range(3))))
    assert np.all(est.sigma_u >= 0) and not np.shares_memory(est.mu_u, r4.mu)


def test_dropin_calls_from_concurrent_threads(dev, rng):
    """Host entries from several Python threads at once (ctypes drops the
    GIL): per-thread streams and bounce arenas, the shared staging ring and
    host workers, the output pool's lock -- every result bitwise equal to the
    same call made alone."""
    import threading

    import paper_2510_01190_b200 as d

    models = []
    for side in (68, 500, 1024, 300):
        g = d.UniformGrid2(side, side)
        models.append(d.GaussianVectorField(g, *random_model_arrays(side * side, rng)))
    want = [(d.propagate_divergence(m), d.lcp(d.propagate_divergence(m), 0.0)) for m in models]
    want = [(f.mu.copy(), f.sigma.copy(), c.probabilities.copy()) for f, c in want]
    errors = []

    def worker(k):
        try:
            for _ in range(4):
                f = d.propagate_divergence(models[k])
                c = d.lcp(f, 0.0)
                mu, sg, pr = want[k]
                if not (np.array_equal(f.mu, mu) and np.array_equal(f.sigma, sg)
                        and np.array_equal(c.probabilities, pr)):
                    errors.append(k)
        except Exception as e:   # noqa: BLE001 -- surfaced below
            errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=(k % 4,)) for k in range(8)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("side", [64, 700])
def test_single_tail_dropins_equal_the_pair(dev, side, rng):
    """source/sink_probability compute and copy back only their own map: bitwise
    the matching half of tail_probs (lcp.py:48-68), sigma = 0 ties included."""
    import paper_2510_01190_b200 as d

    g = d.UniformGrid2(side, side)
    mu_u, mu_v, s_u, s_v = random_model_arrays(side * side, rng)
    s_u[::7] = 0.0
    s_v[::7] = 0.0
    f = d.propagate_divergence(d.GaussianVectorField(g, mu_u, mu_v, s_u, s_v))
    for t in (0.0, 0.25):
        below_neg, _ = d.tail_probs(f.mu, f.sigma, -t)
        _, above = d.tail_probs(f.mu, f.sigma, t)
        assert np.array_equal(d.source_probability(f, t), above)
        assert np.array_equal(d.sink_probability(f, t), below_neg)


def test_dropin_staging_knobs_off_give_the_same_bits(dev, rng, tmp_path):
    """With the output pool, the bounce arena, the copy kernel and the
    streaming stores all switched off (the driver's pageable copies and plain
    numpy outputs), the drop-in results are bitwise the defaults'."""
    import os
    import subprocess
    import sys

    import paper_2510_01190_b200 as d

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    side = 600
    arrs = random_model_arrays(side * side, rng)
    np.savez(tmp_path / "in.npz", *arrs)
    g = d.UniformGrid2(side, side)
    m = d.GaussianVectorField(g, *arrs)
    f = d.propagate_divergence(m)
    want = [f.mu, f.sigma, d.lcp(f, 0.0).probabilities, d.source_probability(f, 0.2)]
    script = (
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {root!r})\n"
        "import paper_2510_01190_b200 as d\n"
        f"z = np.load({str(tmp_path / 'in.npz')!r}); a = [z[k] for k in sorted(z.files)]\n"
        f"g = d.UniformGrid2({side}, {side}); f = d.propagate_divergence(d.GaussianVectorField(g, *a))\n"
        f"np.savez({str(tmp_path / 'out.npz')!r}, f.mu, f.sigma, d.lcp(f, 0.0).probabilities,"
        " d.source_probability(f, 0.2))\n")
    env = dict(os.environ, DIVUQ_OUT_POOL_MB="0", DIVUQ_BOUNCE_MAX_KB="0", DIVUQ_ZC_MAX_KB="0",
               DIVUQ_NT_COPY="0", DIVUQ_ADOPT="0")
    subprocess.run([sys.executable, "-c", script], env=env, check=True, timeout=300)
    z = np.load(tmp_path / "out.npz")
    got = [z[k] for k in sorted(z.files, key=lambda s: int(s.split("_")[1]))]
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
