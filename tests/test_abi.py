"""CPU-only checks of the C ABI boundary and the host-side mirror of the
reference interface (no kernel launches: this box has no GPU)."""

import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "divuq_b200.h")


@pytest.fixture(scope="module")
def pkg():
    import __graft_entry__

    __graft_entry__.build()
    import paper_2510_01190_b200

    return paper_2510_01190_b200


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(divuq_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol(pkg):
    syms = declared_symbols()
    assert len(syms) >= 20
    lib = pkg._lib.lib
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the ctypes table binds exactly the header's surface
    assert set(pkg._lib.SIGNATURES) == set(syms)


def test_abi_version_and_status_strings(pkg):
    lib = pkg._lib.lib
    assert lib.divuq_abi_version() == 2
    assert lib.divuq_status_string(-2).decode().startswith("grid must be")
    assert "non-finite" in lib.divuq_status_string(-10).decode()
    with pytest.raises(ValueError):
        pkg._lib.check(-11)


def test_argument_validation_before_any_launch(pkg):
    """Bad arguments are rejected on the host before touching the device."""
    lib = pkg._lib.lib
    assert lib.divuq_propagate2d_f64(None, None, None, None, 1, 5, 1.0, 1.0, 0.0,
                                     None, None, None, None, None, None) == -2
    assert lib.divuq_propagate2d_f64(None, None, None, None, 4, 4, 1.0, 0.0, 0.0,
                                     None, None, None, None, None, None) == -2
    assert lib.divuq_propagate2d_f64(None, None, None, None, 4, 4, 1.0, 1.0, 0.0,
                                     None, None, None, None, None, None) == -1
    assert lib.divuq_fit_gaussian_f64(1, 1, 2, 10, 1, 1, None, None) == -3
    assert lib.divuq_mc_divergence2d_f64(1, 1, 1, 1, 4, 4, 1.0, 1.0, 1, 0, 0, 4,
                                         1, 1, 1, None, None) == -4
    assert lib.divuq_mc_scratch_bytes(256, 0, 256, 2000) == 2 * 16 * 256 * 256 * 8  # 16 chunks of 128


def test_reference_type_validation(pkg):
    d = pkg
    with pytest.raises(ValueError):
        d.UniformGrid2(1, 5)
    with pytest.raises(ValueError):
        d.UniformGrid2(3, 3, 0.0, 1.0)
    with pytest.raises(ValueError):
        d.UniformGrid3(3, 3, 1)
    g = d.UniformGrid2(3, 2)
    assert g.vertex_index(2, 1) == 5 and g.vertex_ij(5) == (2, 1)
    with pytest.raises(IndexError):
        g.vertex_index(3, 0)
    with pytest.raises(ValueError):
        d.VectorField2(g, [np.nan] * 6, np.zeros(6))
    with pytest.raises(ValueError):
        d.GaussianVectorField(g, np.zeros(6), np.zeros(6), -np.ones(6), np.zeros(6))
    m = d.VectorField2(g, np.zeros(6), np.zeros(6))
    with pytest.raises(ValueError):
        d.Ensemble2(g, (m,))
    with pytest.raises(ValueError):
        d.McConfig(0)
    with pytest.raises(ValueError):
        d.McConfig(10, seed=2**64)
    with pytest.raises(ValueError):
        d.ParallelConfig(threads=0)
    ens = d.Ensemble2(g, (m, m, m))
    assert ens.stacked().shape == (3, 2, 6)
    # fields are frozen copies (grid.py:28-29)
    src = np.arange(6.0)
    f = d.ScalarField2(g, src)
    src[0] = 99.0
    assert f.values[0] == 0.0 and not f.values.flags.writeable


def test_stencil_distribution_fig1_host(pkg):
    from conftest import golden

    fig1 = golden("fig1.npz")
    mu, sd = pkg.stencil_distribution(tuple(map(tuple, fig1["neighbors"])), (1.0, 1.0))
    assert abs(mu + 0.89) <= 1e-12 and sd == 0.7700811645534514


def test_adopted_output_records_match_the_constructor(pkg):
    """api.py builds its output records with types.adopt (no defensive copy,
    reductions instead of scans): same fields and read-only arrays as the
    constructor, and for every invalid value the constructor's own error."""
    from paper_2510_01190_b200 import types as T

    g = T.UniformGrid2(5, 4)
    rng = np.random.default_rng(3)
    mu, sg = rng.normal(size=20), rng.uniform(0, 1, 20)
    a = T.adopt(T.GaussianScalarField, g, mu.copy(), sg.copy())
    b = T.GaussianScalarField(g, mu, sg)
    assert type(a) is type(b) and a.grid == b.grid
    assert np.array_equal(a.mu, b.mu) and np.array_equal(a.sigma, b.sigma)
    assert not a.mu.flags.writeable and not a.sigma.flags.writeable
    m = mu.copy()
    assert T.adopt(T.ScalarField2, g, m).values is m          # no copy
    # finite values whose sum overflows: proven by the constructor instead
    big = np.full(20, 1e308)
    assert np.array_equal(T.adopt(T.ScalarField2, g, big.copy()).values, big)
    cases = [
        (T.GaussianScalarField, lambda: (g, np.where(np.arange(20) == 7, np.nan, mu), sg.copy())),
        (T.GaussianScalarField, lambda: (g, mu.copy(), np.where(np.arange(20) == 3, np.inf, sg))),
        (T.GaussianScalarField, lambda: (g, mu.copy(), np.where(np.arange(20) == 3, -0.5, sg))),
        (T.GaussianScalarField, lambda: (g, mu.copy(), np.where(np.arange(20) == 3, np.nan, sg))),
        (T.GaussianVectorField, lambda: (g, mu.copy(), mu.copy(), sg.copy(), -sg)),
        (T.LcpField, lambda: (g, 0.0, np.where(np.arange(12) == 2, 1.5, 0.5))),
        (T.LcpField, lambda: (g, 0.0, np.where(np.arange(12) == 2, np.nan, 0.5))),
        (T.McDivergenceEstimate, lambda: (g, mu.copy(), np.full(20, -np.inf), 10)),
        (T.McDivergenceEstimate, lambda: (g, mu.copy(), sg.copy(), 1)),
        (T.ScalarField2, lambda: (g, np.zeros(19))),
    ]
    for cls, args in cases:
        with pytest.raises(ValueError) as want:
            cls(*args())
        with pytest.raises(ValueError) as got:
            T.adopt(cls, *args())
        assert str(got.value) == str(want.value), cls.__name__
    # 3D records keep the float dtype of mu
    g3 = T.UniformGrid3(3, 2, 2)
    f32 = rng.uniform(0, 1, 12).astype(np.float32)
    r = T.adopt(T.GaussianScalarField3, g3, f32.copy(), f32.copy())
    assert r.mu.dtype == np.float32 and np.array_equal(r.sigma, f32)
