"""numpy restatement of the reference's 2D hot path -- TEST INFRASTRUCTURE ONLY.

See ``oracle/__init__.py`` for who may import this.  Every function cites the
reference lines it restates (paths relative to ``/root/reference/pkg/src/divuq``).
The restatement works on (ny, nx) views instead of the reference's flat index
arithmetic, but evaluates every floating-point expression in the reference's
exact order, so results are bit-identical (pinned by ``tests/test_oracle.py``
against vectors the reference itself produced).
"""

from __future__ import annotations

import numpy as np
from scipy.special import ndtr  # the reference's own CDF (lcp.py:19)


def axis_rule(n: int, h: float):
    """Per-position (lo, hi, coeff) along one axis of length n.

    Restates ``axis_stencil`` (stencils.py:17-51): lo = clip(a-1), hi =
    clip(a+1), coeff = 1/(2h) strictly inside, 1/h on the two end vertices
    (the clamped neighbour is the vertex itself, stencils.py:46-50).
    """
    a = np.arange(n)
    lo = np.clip(a - 1, 0, n - 1)
    hi = np.clip(a + 1, 0, n - 1)
    coeff = np.where((a > 0) & (a < n - 1), 1.0 / (2.0 * h), 1.0 / h)
    return lo, hi, coeff


def _x_terms(f2, dx):
    lo, hi, c = axis_rule(f2.shape[-1], dx)
    return f2[..., hi] * c, f2[..., lo] * c


def _y_terms(f2, dy):
    lo, hi, c = axis_rule(f2.shape[-2], dy)
    c = c[:, None]
    return f2[..., hi, :] * c, f2[..., lo, :] * c


def divergence2d(u, v, nx: int, ny: int, dx: float, dy: float) -> np.ndarray:
    """du/dx + dv/dy, flat row-major (stencils.py:54-66).

    Evaluated as ``((u_hi*cx - u_lo*cx) + v_hi*cy) - v_lo*cy`` -- the reference's
    left-to-right association, each product rounded separately.  Accepts
    batched (B, n) inputs like the reference (stencils.py:58-59).
    """
    u = np.asarray(u, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    batch = u.shape[:-1]
    u2 = u.reshape(batch + (ny, nx))
    v2 = v.reshape(batch + (ny, nx))
    xh, xl = _x_terms(u2, dx)
    yh, yl = _y_terms(v2, dy)
    return (((xh - xl) + yh) - yl).reshape(batch + (nx * ny,))


def divergence_variance2d(su, sv, nx: int, ny: int, dx: float, dy: float) -> np.ndarray:
    """Sum of (sigma*c)^2 over the four stencil terms (stencils.py:69-84).

    Order: u_hi, u_lo, v_hi, v_lo; the square is of the rounded product.
    """
    su2 = np.asarray(su, dtype=np.float64).reshape(ny, nx)
    sv2 = np.asarray(sv, dtype=np.float64).reshape(ny, nx)
    xh, xl = _x_terms(su2, dx)
    yh, yl = _y_terms(sv2, dy)
    return (((xh * xh + xl * xl) + yh * yh) + yl * yl).ravel()


def propagate2d(mu_u, mu_v, s_u, s_v, nx, ny, dx, dy):
    """(mu_div, sigma_div) -- ``propagate_divergence`` (divergence.py:48-70)."""
    mu = divergence2d(mu_u, mu_v, nx, ny, dx, dy)
    var = divergence_variance2d(s_u, s_v, nx, ny, dx, dy)
    return mu, np.sqrt(var)


def stencil_distribution(neighbors, spacing):
    """Single interior vertex, Fig. 1 (divergence.py:73-85)."""
    (mu_um, s_um), (mu_up, s_up), (mu_vm, s_vm), (mu_vp, s_vp) = neighbors
    dx, dy = spacing
    cx, cy = 1.0 / (2.0 * dx), 1.0 / (2.0 * dy)
    mu = mu_up * cx - mu_um * cx + mu_vp * cy - mu_vm * cy
    a, b, c, d = s_up * cx, s_um * cx, s_vp * cy, s_vm * cy
    return float(mu), float(np.sqrt(a * a + b * b + c * c + d * d))


def fit_moments(members: np.ndarray):
    """Per-point mean / ddof=1 std over axis 0 (gaussian.py:35-45).

    numpy's axis-0 reduction is a sequential sum over members; ``mean`` divides
    by M; ``std(ddof=1)`` is two-pass: sum of squared deviations from that mean,
    divided by M-1, then sqrt.  Restated as explicit loops in that order.
    ``members`` has shape (M, ...); results have shape (...).
    """
    x = np.asarray(members, dtype=np.float64)
    m = x.shape[0]
    s = x[0].copy()
    for k in range(1, m):
        s = s + x[k]
    mu = s / m
    d = x[0] - mu
    q = d * d
    for k in range(1, m):
        d = x[k] - mu
        q = q + d * d
    return mu, np.sqrt(q / (m - 1))


def fit_gaussian(members_mcn: np.ndarray):
    """(M, C, N) member-major ensemble -> mu (C, N), sigma (C, N)."""
    return fit_moments(members_mcn)


def tail_probs(mu, sigma, theta: float):
    """(P[X <= theta], P[X > theta]) per vertex (lcp.py:48-68).

    sigma == 0 is a step with mu == theta counted as below; otherwise
    t = (theta - mu)/sigma (overflow to +-inf allowed) and both tails are
    evaluated directly with ndtr, never as 1 - p.
    """
    mu = np.asarray(mu, dtype=np.float64)
    sigma = np.asarray(sigma, dtype=np.float64)
    below = np.empty_like(mu)
    above = np.empty_like(mu)
    deg = sigma == 0
    below[deg] = np.where(mu[deg] <= theta, 1.0, 0.0)
    above[deg] = 1.0 - below[deg]
    ok = ~deg
    with np.errstate(over="ignore"):
        t = (theta - mu[ok]) / sigma[ok]
    below[ok] = ndtr(t)
    above[ok] = ndtr(-t)
    return below, above


def source_probability(mu, sigma, t: float):
    """P(div > t): the 'above' tail at isovalue t."""
    return tail_probs(mu, sigma, t)[1]


def sink_probability(mu, sigma, t: float):
    """P(div < -t) (P(div <= -t) on the sigma == 0 tie, lcp.py:58)."""
    return tail_probs(mu, sigma, -t)[0]


def error_metrics(est_mean, est_std, mu, sigma):
    """(e_m, e_sigma, sse) (mc.py:159-175)."""
    dm = np.asarray(est_mean) - np.asarray(mu)
    ds = np.asarray(est_std) - np.asarray(sigma)
    return (
        float(np.abs(dm).mean()),
        float(np.abs(ds).mean()),
        float(np.sum(dm**2) + np.sum(ds**2)),
    )


def cell_crossing_probability(mu, sigma, isovalue):
    """LCP for stacked cells (..., 4) (lcp.py:71-77): sequential products of
    the four corners' tails, 1 - (prod below + prod above), clipped."""
    below, above = tail_probs(np.asarray(mu, float), np.asarray(sigma, float), isovalue)
    pb = below[..., 0] * below[..., 1] * below[..., 2] * below[..., 3]
    pa = above[..., 0] * above[..., 1] * above[..., 2] * above[..., 3]
    return np.clip(1.0 - (pb + pa), 0.0, 1.0)


def lcp(mu, sigma, nx, ny, isovalue):
    """Per-cell LCP, cell index cj*(nx-1)+ci (lcp.py:80-100)."""
    ci, cj = np.meshgrid(np.arange(nx - 1), np.arange(ny - 1))
    v00 = (cj * nx + ci).ravel()
    corners = np.stack([v00, v00 + 1, v00 + nx, v00 + nx + 1], axis=-1)
    mu = np.asarray(mu, float)
    sigma = np.asarray(sigma, float)
    return cell_crossing_probability(mu[corners], sigma[corners], isovalue)


def velocity_magnitude(u, v):
    """hypot(u, v) per vertex (gaussian.py:48-50)."""
    return np.hypot(np.asarray(u, float), np.asarray(v, float))


def gradient2d(values, nx, ny, dx, dy):
    """(gx, gy) = (f[hx]*cx - f[lx]*cx, f[hy]*cy - f[ly]*cy) (gaussian.py:53-58,
    stencils.py:87-96), the divergence's per-axis rule (axis_rule)."""
    f2 = np.asarray(values, float).reshape(ny, nx)
    xh, xl = _x_terms(f2, dx)
    yh, yl = _y_terms(f2, dy)
    return (xh - xl).ravel(), (yh - yl).ravel()


def gradient_ensemble(members, nx, ny, dx, dy):
    """(M, 2, N) members -> (M, 2, N) gradients of |(u, v)| (gaussian.py:61-66)."""
    members = np.asarray(members, float)
    out = np.empty_like(members)
    for k, m in enumerate(members):
        out[k, 0], out[k, 1] = gradient2d(velocity_magnitude(m[0], m[1]), nx, ny, dx, dy)
    return out
