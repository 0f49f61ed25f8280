"""divuq/_b200.py -- the B200 backend hook for the reference package.

This is the file INTEGRATION.md tells a ``divuq`` maintainer to drop into
``divuq/`` (as ``_b200.py``), plus ONE line at the end of
``divuq/__init__.py``::

    from . import _b200; _b200.install()

It binds ``libdivuq_b200.so`` with plain ctypes (numpy buffers, no torch) and
routes the reference's hot-path functions through the C ABI declared in
``include/divuq_b200.h``.  The reference's dataclasses still validate every
input first (grid.py:21-30, divergence.py:34-35, gaussian.py:28-29), the
signatures, return types and exceptions stay the reference's, and the
routed functions return what the reference returns:

  ==========================================  ==================================  =========================
  reference function                          C entry point                       parity
  ==========================================  ==================================  =========================
  divergence.propagate_divergence :48-70      divuq_host_propagate2d_f64          bitwise
  divergence.divergence_deterministic :41-45  divuq_host_propagate2d_f64 (s=0)    bitwise
  gaussian.fit_gaussian :35-45                divuq_host_fit_gaussian_f64         bitwise
  gaussian.velocity_magnitude :48-50          divuq_host_velocity_magnitude_f64   <= 1 ulp (GPU hypot)
  gaussian.gradient :53-58                    divuq_host_gradient2d_f64           bitwise
  lcp._tail_probs :48-68                      divuq_host_tail_probs_f64           <= 1e-13 rel
  lcp.cell_crossing_probability :71-77        divuq_host_cell_crossing_f64        <= 1e-12 abs
  lcp.lcp :80-100                             divuq_host_lcp2d_f64                <= 1e-12 abs
  mc.mc_divergence :94-117                    divuq_host_mc_divergence2d_ref_f64  draw for draw
  mc.sample_divergence_1d :142-156            divuq_host_mc_histogram1d_f64       draw for draw
  mc.mc_histogram_1d :120-139                 divuq_host_mc_histogram1d_f64       draw for draw
  ==========================================  ==================================  =========================

``DIVUQ_B200_LIB`` names the library (default: ``libdivuq_b200.so`` on the
loader path); when it cannot be loaded ``install()`` leaves the reference
untouched.  ``DIVUQ_B200_TRACE=<path>`` appends one line per routed call
(the boundary test uses it to prove the GPU path ran).  ``install()`` warms
the device up (CUDA context, library pools) at import so the first routed
call is not charged for it; ``DIVUQ_B200_LAZY=1`` defers that to first use.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_LIB = os.environ.get("DIVUQ_B200_LIB", "libdivuq_b200.so")
try:
    _lib = ctypes.CDLL(_LIB)
except OSError:
    _lib = None

_p, _i64, _u64, _f64, _int = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double,
                              ctypes.c_int)
_ARGS = {
    "divuq_host_propagate2d_f64": [_p] * 4 + [_i64, _i64, _f64, _f64, _f64] + [_p] * 4 + [_int],
    "divuq_host_fit_gaussian_f64": [_p, _i64, _i64, _i64, _p, _p, _int],
    "divuq_host_tail_probs_f64": [_p, _p, _i64, _f64, _p, _p, _int],
    "divuq_host_lcp2d_f64": [_p, _p, _i64, _i64, _f64, _p, _int],
    "divuq_host_cell_crossing_f64": [_p, _p, _i64, _f64, _p, _int],
    "divuq_host_velocity_magnitude_f64": [_p, _p, _i64, _p, _int],
    "divuq_host_gradient2d_f64": [_p, _i64, _i64, _f64, _f64, _p, _int],
    "divuq_host_mc_divergence2d_ref_f64": [_p] * 4 + [_i64, _i64, _f64, _f64, _i64, _u64, _p, _p,
                                                      _int],
    "divuq_host_mc_histogram1d_f64": [_p, _f64, _f64, _i64, _u64, _i64, _p, _p, _p, _p, _int],
}
if _lib is not None:
    for _name, _a in _ARGS.items():
        getattr(_lib, _name).argtypes = _a
        getattr(_lib, _name).restype = _int
    _lib.divuq_status_string.argtypes = [_int]
    _lib.divuq_status_string.restype = ctypes.c_char_p

_DEVICE = int(os.environ.get("DIVUQ_B200_DEVICE", "0"))
_TRACE = os.environ.get("DIVUQ_B200_TRACE")


def _trace(name: str) -> None:
    if _TRACE:
        with open(_TRACE, "a") as fh:
            fh.write(name + "\n")


def _check(status: int) -> None:
    if status < 0:
        raise ValueError(_lib.divuq_status_string(status).decode())
    if status > 0:
        raise RuntimeError(f"CUDA error {status}: {_lib.divuq_status_string(status).decode()}")


def _ptr(a):
    return None if a is None else a.ctypes.data


def _f64c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def install() -> bool:
    """Route the reference's hot-path functions through the B200 library.
    Returns False (and changes nothing) when the library is unavailable."""
    if _lib is None:
        return False
    import importlib

    import divuq
    # submodules by name: the package re-exports a FUNCTION called lcp that
    # shadows the lcp submodule as a package attribute (__init__.py:33)
    divergence, gaussian, lcp, mc = (importlib.import_module(f"divuq.{m}")
                                     for m in ("divergence", "gaussian", "lcp", "mc"))
    from divuq.divergence import GaussianScalarField
    from divuq.gaussian import GaussianVectorField
    from divuq.grid import ScalarField2, VectorField2
    from divuq.lcp import LcpField
    from divuq.mc import McDivergenceEstimate, McHistogram

    def propagate_divergence(model, config=None):
        _trace("propagate_divergence")
        g = model.grid
        n = g.n_vertices
        mu, sg = np.empty(n), np.empty(n)
        _check(_lib.divuq_host_propagate2d_f64(
            _ptr(model.mu_u), _ptr(model.mu_v), _ptr(model.sigma_u), _ptr(model.sigma_v), g.nx,
            g.ny, float(g.dx), float(g.dy), 0.0, _ptr(mu), _ptr(sg), None, None, _DEVICE))
        return GaussianScalarField(g, mu, sg)

    def divergence_deterministic(fld):
        _trace("divergence_deterministic")
        g = fld.grid
        out = np.empty(g.n_vertices)
        _check(_lib.divuq_host_propagate2d_f64(
            _ptr(fld.u), _ptr(fld.v), None, None, g.nx, g.ny, float(g.dx), float(g.dy), 0.0,
            _ptr(out), None, None, None, _DEVICE))
        return ScalarField2(g, out)

    def fit_gaussian(ensemble):
        _trace("fit_gaussian")
        stacked = np.stack([np.stack([m.u, m.v]) for m in ensemble.members])   # (M, 2, N)
        m, c, n = stacked.shape
        mu, sd = np.empty((c, n)), np.empty((c, n))
        _check(_lib.divuq_host_fit_gaussian_f64(_ptr(stacked), m, c, n, _ptr(mu), _ptr(sd),
                                                _DEVICE))
        return GaussianVectorField(ensemble.grid, mu[0], mu[1], sd[0], sd[1])

    def velocity_magnitude(member):
        _trace("velocity_magnitude")
        g = member.grid
        out = np.empty(g.n_vertices)
        _check(_lib.divuq_host_velocity_magnitude_f64(_ptr(member.u), _ptr(member.v),
                                                      g.n_vertices, _ptr(out), _DEVICE))
        return ScalarField2(g, out)

    def gradient(fld):
        _trace("gradient")
        g = fld.grid
        out = np.empty((2, g.n_vertices))
        _check(_lib.divuq_host_gradient2d_f64(_ptr(fld.values), g.nx, g.ny, float(g.dx),
                                              float(g.dy), _ptr(out), _DEVICE))
        return VectorField2(g, out[0], out[1])

    def _tail_probs(mu, sigma, isovalue):
        _trace("_tail_probs")
        mu, sigma = _f64c(mu), _f64c(sigma)
        below, above = np.empty_like(mu), np.empty_like(mu)
        if mu.size:
            _check(_lib.divuq_host_tail_probs_f64(_ptr(mu), _ptr(sigma), mu.size, float(isovalue),
                                                  _ptr(below), _ptr(above), _DEVICE))
        return below, above

    def cell_crossing_probability(mu, sigma, isovalue):
        _trace("cell_crossing_probability")
        mu, sigma = _f64c(mu), _f64c(sigma)
        if mu.shape != sigma.shape or mu.ndim < 1 or mu.shape[-1] != 4:
            raise ValueError("mu and sigma must have shape (..., 4)")
        out = np.empty(mu.shape[:-1])
        n = out.size
        if n:
            _check(_lib.divuq_host_cell_crossing_f64(_ptr(mu), _ptr(sigma), n, float(isovalue),
                                                     _ptr(out), _DEVICE))
        return out

    def lcp_(fld, isovalue, config=None):
        _trace("lcp")
        g = fld.grid
        out = np.empty(g.n_cells)
        _check(_lib.divuq_host_lcp2d_f64(_ptr(fld.mu), _ptr(fld.sigma), g.nx, g.ny,
                                         float(isovalue), _ptr(out), _DEVICE))
        return LcpField(g, isovalue, out)

    def mc_divergence(model, config):
        _trace("mc_divergence")
        if config.n_samples < 2:
            raise ValueError("mc_divergence needs n_samples >= 2")
        g = model.grid
        n = g.n_vertices
        mean, std = np.empty(n), np.empty(n)
        _check(_lib.divuq_host_mc_divergence2d_ref_f64(
            _ptr(model.mu_u), _ptr(model.mu_v), _ptr(model.sigma_u), _ptr(model.sigma_v), g.nx,
            g.ny, float(g.dx), float(g.dy), int(config.n_samples), int(config.seed), _ptr(mean),
            _ptr(std), _DEVICE))
        return McDivergenceEstimate(g, mean, std, config.n_samples)

    def _neighbors8(neighbors):
        nb = np.asarray([float(x) for pair in neighbors for x in pair], dtype=np.float64)
        if nb.size != 8:
            raise ValueError("neighbors: four (mu, sigma) pairs")
        if np.any(nb[1::2] < 0):
            raise ValueError("sigmas must be non-negative")
        return nb

    def sample_divergence_1d(neighbors, spacing, config):
        _trace("sample_divergence_1d")
        nb = _neighbors8(neighbors)
        dx, dy = spacing
        values = np.empty(config.n_samples)
        edges, counts, used = np.empty(2), np.empty(1, dtype=np.int64), np.zeros(1, dtype=np.int64)
        _check(_lib.divuq_host_mc_histogram1d_f64(
            _ptr(nb), float(dx), float(dy), int(config.n_samples), int(config.seed), 1, _ptr(edges),
            _ptr(counts), _ptr(used), _ptr(values), _DEVICE))
        return values

    def mc_histogram_1d(neighbors, spacing, config, n_bins):
        _trace("mc_histogram_1d")
        if n_bins < 1:
            raise ValueError("n_bins must be >= 1")
        nb = _neighbors8(neighbors)
        dx, dy = spacing
        edges = np.empty(n_bins + 1)
        counts = np.empty(n_bins, dtype=np.int64)
        used = np.zeros(1, dtype=np.int64)
        _check(_lib.divuq_host_mc_histogram1d_f64(
            _ptr(nb), float(dx), float(dy), int(config.n_samples), int(config.seed), int(n_bins),
            _ptr(edges), _ptr(counts), _ptr(used), None, _DEVICE))
        k = int(used[0])
        return McHistogram(edges[: k + 1].copy(), counts[:k].copy(), int(config.n_samples))

    routes = [
        (divergence, "propagate_divergence", propagate_divergence),
        (divergence, "divergence_deterministic", divergence_deterministic),
        (gaussian, "fit_gaussian", fit_gaussian),
        (gaussian, "velocity_magnitude", velocity_magnitude),
        (gaussian, "gradient", gradient),
        (lcp, "_tail_probs", _tail_probs),
        (lcp, "cell_crossing_probability", cell_crossing_probability),
        (lcp, "lcp", lcp_),
        (mc, "mc_divergence", mc_divergence),
        (mc, "sample_divergence_1d", sample_divergence_1d),
        (mc, "mc_histogram_1d", mc_histogram_1d),
    ]
    for module, name, fn in routes:
        fn.__name__ = name
        fn.__doc__ = getattr(module, name).__doc__
        setattr(module, name, fn)            # callers inside the package
        if hasattr(divuq, name):
            setattr(divuq, name, fn)         # the public re-export (__init__.py:9-45)
    if os.environ.get("DIVUQ_B200_LAZY", "0") != "1":
        # create the CUDA context and stage the library's pools now, at import,
        # not inside the first routed call (~1-3 s once per process)
        one, zero = np.ones(1), np.zeros(1)
        b_, a_ = np.empty(1), np.empty(1)
        _lib.divuq_host_tail_probs_f64(_ptr(zero), _ptr(one), 1, 0.0, _ptr(b_), _ptr(a_), _DEVICE)
    return True
