"""The reference's own MC stream (splitmix64 + AS241) -- TEST INFRASTRUCTURE ONLY.

numpy restatement of ``/root/reference/pkg/src/divuq/rng.py`` and of the parts
of ``mc.py`` that consume it, used to check the GPU's reference-stream mode
(``mc_divergence(..., stream="reference")``, ``sample_divergence_1d``,
``mc_histogram_1d``).  Pinned bitwise against vectors the reference itself
produced (``tests/golden/make_golden_refstream.py``).

Stream contract (rng.py:23-34, 37-75, 86-92):
    z       = splitmix64(seed + counter * 0x9E3779B97F4A7C15)   (mod 2^64)
    u       = ((z >> 11) + 0.5) * 2^-53                          # in (0, 1)
    normal  = AS241 / PPND16 inverse normal CDF of u, every product and sum
              rounded separately (numba without fastmath does not contract)
Counters (mc.py:80-91): u of sample s at vertex v uses (2s) n + v, v uses
(2s+1) n + v, n = grid vertices.  sample_divergence_1d (mc.py:142-156): the
four neighbour draws of sample k use counters 4k, 4k+1, 4k+2, 4k+3.
"""

from __future__ import annotations

import numpy as np

from .ref2d import divergence2d

_U = np.uint64
GOLDEN = _U(0x9E3779B97F4A7C15)

# AS241 PPND16 coefficients (Wichura 1988, Appl. Statist. 37:477-484), the
# published table the reference evaluates (rng.py:40-73)
_A = (3.3871328727963666080e0, 1.3314166789178437745e2, 1.9715909503065514427e3,
      1.3731693765509461125e4, 4.5921953931549871457e4, 6.7265770927008700853e4,
      3.3430575583588128105e4, 2.5090809287301226727e3)
_B = (1.0, 4.2313330701600911252e1, 6.8718700749205790830e2, 5.3941960214247511077e3,
      2.1213794301586595867e4, 3.9307895800092710610e4, 2.8729085735721942674e4,
      5.2264952788528545610e3)
_C = (1.42343711074968357734e0, 4.63033784615654529590e0, 5.76949722146069140550e0,
      3.64784832476320460504e0, 1.27045825245236838258e0, 2.41780725177450611770e-1,
      2.27238449892691845833e-2, 7.74545014278341407640e-4)
_D = (1.0, 2.05319162663775882187e0, 1.67638483018380384940e0, 6.89767334985100004550e-1,
      1.48103976427480074590e-1, 1.51986665636164571966e-2, 5.47593808499534494600e-4,
      1.05075007164441684324e-9)
_E = (6.65790464350110377720e0, 5.46378491116411436990e0, 1.78482653991729133580e0,
      2.96560571828504891230e-1, 2.65321895265761230930e-2, 1.24266094738807843860e-3,
      2.71155556874348757815e-5, 2.01033439929228813265e-7)
_F = (1.0, 5.99832206555887937690e-1, 1.36929880922735805310e-1, 1.48753612908506148525e-2,
      7.86869131145613259100e-4, 1.84631831751005468180e-5, 1.42151175831644588870e-7,
      2.04426310338993978564e-15)


def _horner(coef, r):
    """((c7 r + c6) r + ...) r + c0, each product/sum rounded (no fma)."""
    acc = coef[7] * r
    for c in coef[6:0:-1]:
        acc = (acc + c) * r
    return acc + coef[0]


def mix(x):
    """splitmix64 finaliser of x (uint64 arrays, wrapping), rng.py:23-28."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=_U) + GOLDEN
        z = (z ^ (z >> _U(30))) * _U(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> _U(27))) * _U(0x94D049BB133111EB)
        return z ^ (z >> _U(31))


def to_uniform(z):
    return ((np.asarray(z, dtype=_U) >> _U(11)).astype(np.float64) + 0.5) * (2.0 ** -53)


def inv_normal_cdf(p):
    """AS241 for p in (0, 1), vectorised with the reference's branch order."""
    p = np.asarray(p, dtype=np.float64)
    q = p - 0.5
    out = np.empty_like(p)
    cen = np.abs(q) <= 0.425
    if cen.any():
        qc = q[cen]
        r = 0.180625 - qc * qc
        out[cen] = qc * _horner(_A, r) / _horner(_B, r)
    tail = ~cen
    if tail.any():
        qt = q[tail]
        r = np.where(qt < 0.0, p[tail], 1.0 - p[tail])
        r = np.sqrt(-np.log(r))
        lo = r <= 5.0
        x = np.empty_like(r)
        rl = r[lo] - 1.6
        x[lo] = _horner(_C, rl) / _horner(_D, rl)
        rh = r[~lo] - 5.0
        x[~lo] = _horner(_E, rh) / _horner(_F, rh)
        out[tail] = np.where(qt < 0.0, -x, x)
    return out


def normal_stream(seed: int, counters):
    c = np.asarray(counters, dtype=_U)
    with np.errstate(over="ignore"):
        x = _U(seed & 0xFFFFFFFFFFFFFFFF) + c * GOLDEN
    return inv_normal_cdf(to_uniform(mix(x)))


def mc_divergence(mu_u, mu_v, s_u, s_v, nx, ny, dx, dy, n_samples, seed, block=64):
    """(mean, std) exactly as mc.py:94-117 computes them."""
    if n_samples < 2:
        raise ValueError("mc_divergence needs n_samples >= 2")
    n = nx * ny
    vertex = np.arange(n, dtype=_U)
    mean = np.zeros(n)
    m2 = np.zeros(n)
    count = 0
    for start in range(0, n_samples, block):
        s = np.arange(start, min(start + block, n_samples), dtype=_U)[:, None]
        zu = normal_stream(seed, (s * _U(2)) * _U(n) + vertex)
        zv = normal_stream(seed, (s * _U(2) + _U(1)) * _U(n) + vertex)
        div = divergence2d(mu_u + s_u * zu, mu_v + s_v * zv, nx, ny, dx, dy)
        for row in div:
            count += 1
            delta = row - mean
            mean += delta / count
            m2 += delta * (row - mean)
    return mean, np.sqrt(m2 / (count - 1))


def sample_divergence_1d(neighbors, spacing, n_samples, seed):
    """mc.py:142-156: raw single-vertex samples."""
    (mu_um, s_um), (mu_up, s_up), (mu_vm, s_vm), (mu_vp, s_vp) = neighbors
    dx, dy = spacing
    c = np.arange(n_samples, dtype=_U) * _U(4)
    um = mu_um + s_um * normal_stream(seed, c)
    up = mu_up + s_up * normal_stream(seed, c + _U(1))
    vm = mu_vm + s_vm * normal_stream(seed, c + _U(2))
    vp = mu_vp + s_vp * normal_stream(seed, c + _U(3))
    return (up - um) / (2.0 * dx) + (vp - vm) / (2.0 * dy)


def mc_histogram_1d(neighbors, spacing, n_samples, seed, n_bins):
    """mc.py:120-139: (edges, counts) of the sampled single-vertex divergence."""
    values = sample_divergence_1d(neighbors, spacing, n_samples, seed)
    lo, hi = float(values.min()), float(values.max())
    if lo == hi:
        return np.array([lo - 0.5, hi + 0.5]), np.array([values.size])
    counts, edges = np.histogram(values, bins=n_bins, range=(lo, hi))
    return edges, counts
