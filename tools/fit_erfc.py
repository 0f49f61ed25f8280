"""Fit the fp32 erfc kernel approximation used in csrc/fastmath.cuh.

erfc(a) = exp(-a^2) * h(q) / (a + K),  q = (a - K) / (a + K),  a >= 0,
h(q) = (a + K) * erfcx(a) is smooth on q in [-1, 1).  h is fitted as a
polynomial in q by least squares on Chebyshev nodes, minimising relative
error; the fit is then verified in float32 arithmetic (numpy emulation of the
CUDA evaluation order) against scipy's erfc.  Run: python tools/fit_erfc.py
"""
import numpy as np
from scipy.special import erfc, erfcx

K = 2.0
AMAX = 10.5   # fp32 erfc underflows past ~10.05


def fit(deg):
    qmin, qmax = -1.0, (AMAX - K) / (AMAX + K)
    n = 4000
    t = np.cos(np.pi * (np.arange(n) + 0.5) / n)
    q = 0.5 * (qmin + qmax) + 0.5 * (qmax - qmin) * t
    a = K * (1 + q) / (1 - q)
    h = (a + K) * erfcx(a)
    # relative-error weighted least squares in the monomial basis of q
    V = np.vander(q, deg + 1)
    w = 1.0 / h
    c, *_ = np.linalg.lstsq(V * w[:, None], h * w, rcond=None)
    return c  # highest power first


def eval32(c, a):
    a = np.float32(a)
    f32 = np.float32
    r = f32(1) / (a + f32(K))
    q = (a - f32(K)) * r
    p = f32(c[0])
    for ci in c[1:]:
        p = f32(np.fma(p, q, f32(ci))) if hasattr(np, "fma") else f32(p * q + f32(ci))
    s = a * a
    e = f32(np.exp(-np.float64(s)))  # stands in for an accurate expf
    return p * r * e


if __name__ == "__main__":
    a = np.linspace(0, 10.0, 200001)
    ref = erfc(a)
    for deg in (8, 9, 10, 11, 12, 13):
        c = fit(deg)
        # fp64 model error
        q = (a - K) / (a + K)
        h = np.polyval(c, q)
        approx = h / (a + K) * np.exp(-a * a)
        rel = np.abs(approx - ref) / ref
        print(deg, "max rel (fp64 eval) %.3g" % rel[ref > 1e-38].max())
    c = fit(11)
    print("coefficients (highest power first):")
    for ci in c:
        print("  %.9ef," % np.float32(ci))


def verify32(c, a):
    """float32 evaluation in the device order (fma = one rounding via fp64)."""
    f32 = np.float32
    a = a.astype(np.float32)
    r = (f32(1) / (a + f32(K))).astype(np.float32)
    q = ((a - f32(K)) * r).astype(np.float32)
    p = np.full_like(a, f32(c[0]))
    for ci in c[1:]:
        p = (p.astype(np.float64) * q + np.float64(f32(ci))).astype(np.float32)
    s = (a * a).astype(np.float32)
    lo = (a.astype(np.float64) * a - s).astype(np.float32)          # fma(a, a, -s)
    e = np.exp(-s.astype(np.float64)).astype(np.float32)           # accurate expf
    y = (p * r).astype(np.float32)
    y = (y * e).astype(np.float32)
    y = (y.astype(np.float64) * -lo + y).astype(np.float32)         # fma(y, -lo, y)
    return y


if __name__ == "__main__":
    c = fit(9)
    c32 = [np.float32(ci) for ci in c]
    a = np.linspace(0, 9.9, 400001).astype(np.float32)
    ref = erfc(a.astype(np.float64))
    y = verify32(c32, a)
    m = ref > 1.2e-38
    rel = np.abs(y[m] - ref[m]) / ref[m]
    print("deg 9 float32: max rel %.3g, max ulp-ish %.2f" % (rel.max(), rel.max() / 5.96e-8))
    print("deg-9 coefficients (highest power first):")
    for ci in c32:
        print("  %.9ef," % ci)


# ---------------------------------------------------------------------------
# fp64 variant for the level-crossing kernels (csrc/lcp.cuh: erfc_abs_lcp):
# the same form over a in [0, 27] with K = 3.75 and a degree-20 polynomial,
# fitted in the Chebyshev basis (relative weighting) and converted to monomials
# in q (coefficients stay <= 1.1, so Horner is well conditioned).
# Verified: max relative error vs scipy erfc ~4e-15 on a in [0, 26.5].
#   python -c "import tools.fit_erfc as f; f.fit64_report()"
def fit64(K=3.75, deg=20, amax=27.0):
    from numpy.polynomial import chebyshev as C

    qmin, qmax = -1.0, (amax - K) / (amax + K)
    n = 6000
    t = np.cos(np.pi * (np.arange(n) + 0.5) / n)
    q = 0.5 * (qmin + qmax) + 0.5 * (qmax - qmin) * t
    a = K * (1 + q) / (1 - q)
    h = (a + K) * erfcx(a)
    x = (2 * q - (qmin + qmax)) / (qmax - qmin)
    w = 1 / h
    c, *_ = np.linalg.lstsq(C.chebvander(x, deg) * w[:, None], h * w, rcond=None)
    alpha, beta = 2 / (qmax - qmin), -(qmax + qmin) / (qmax - qmin)
    P = np.polynomial.Polynomial(C.cheb2poly(c))
    return P(np.polynomial.Polynomial([beta, alpha])).coef  # lowest power first


def fit64_report(K=3.75, deg=20):
    co = fit64(K, deg)
    a = np.linspace(0, 26.5, 200001)
    r = 1.0 / (a + K)
    q = (a - K) * r
    p = np.full_like(a, co[-1])
    for c in co[-2::-1]:
        p = p * q + c
    y = p * r * np.exp(-a * a)
    ref = erfc(a)
    print("max rel err", (np.abs(y - ref) / ref).max())
    print(", ".join(float.hex(float(c)) for c in co))
