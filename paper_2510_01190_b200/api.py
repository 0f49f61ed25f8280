"""Drop-in replacements for the reference's public hot-path functions.

Same names, signatures, return types and exceptions as
/root/reference/pkg/src/divuq (re-exported by its __init__.py:9-96).  Each
function hands host (numpy) buffers to a ``divuq_host_*`` entry point of the
C ABI (include/divuq_b200.h), which stages them into HBM, runs the sm_100a
kernel and copies the result back -- the "reference-facing" path the e2e
benchmark times.  There is no CPU fallback: without the CUDA library the
package does not import.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np

from ._lib import check as _check
from ._lib import lib
from .types import (
    Ensemble2,
    GaussianScalarField,
    GaussianScalarField3,
    GaussianVectorField,
    GaussianVectorField3,
    LcpField,
    McConfig,
    McDivergenceEstimate,
    McHistogram,
    ParallelConfig,
    ScalarField2,
    UniformGrid3,
    VectorField2,
    adopt,
)

_DEVICE = 0


from . import _pool  # noqa: E402  (pinned host blocks for results, _pool.py)

_POOL = _pool.POOL
_out = _pool.empty


def set_device(ordinal: int) -> None:
    """CUDA device used by the host-buffer entry points (default 0)."""
    global _DEVICE
    _DEVICE = int(ordinal)


def _p(a):
    return None if a is None else a.__array_interface__["data"][0]


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def fit_gaussian(ensemble: Ensemble2) -> GaussianVectorField:
    """Sample mean and ddof=1 std per vertex/component (gaussian.py:35-45).

    Bit-identical to the reference (sequential member sum, two-pass variance).
    """
    stacked = _c64(ensemble.stacked())  # (M, 2, N)
    m, c, n = stacked.shape
    mu = _out((c, n))
    sg = _out((c, n))
    _check(lib.divuq_host_fit_gaussian_f64(_p(stacked), m, c, n, _p(mu), _p(sg), _DEVICE))
    return adopt(GaussianVectorField, ensemble.grid, mu[0], mu[1], sg[0], sg[1])


def propagate_divergence(model, config: ParallelConfig | None = None):
    """Divergence distribution of an independent-Gaussian model (divergence.py:48-70).

    2D (``GaussianVectorField``) results are bit-identical to the reference;
    ``config`` is accepted and ignored (one launch covers every vertex, and the
    output is the same for any setting -- the reference's own contract,
    parallel.py:1-6).  A ``GaussianVectorField3`` runs the 3D restatement.
    """
    if isinstance(model, GaussianVectorField3):
        res = propagate_with_probabilities3d(model, 0.0, probabilities=False)
        return res.field
    return propagate_with_probabilities(model, 0.0, probabilities=False).field


class Propagation(NamedTuple):
    field: object          # GaussianScalarField / GaussianScalarField3
    p_src: np.ndarray | None   # P(div > t)
    p_snk: np.ndarray | None   # P(div < -t)


def propagate_with_probabilities(model: GaussianVectorField, t: float = 0.0, *,
                                 probabilities: bool = True) -> Propagation:
    """Fused hot path: mu_div, sigma_div and the source/sink maps in one pass.

    p_src = P(div > t) and p_snk = P(div < -t) with the reference's
    ``_tail_probs`` semantics (lcp.py:48-68), computed in the same kernel.
    """
    g = model.grid
    n = g.n_vertices
    mu = _out(n)
    sg = _out(n)
    ps = _out(n) if probabilities else None
    pk = _out(n) if probabilities else None
    _check(lib.divuq_host_propagate2d_f64(
        _p(model.mu_u), _p(model.mu_v), _p(model.sigma_u), _p(model.sigma_v), g.nx, g.ny,
        float(g.dx), float(g.dy), float(t), _p(mu), _p(sg), _p(ps), _p(pk), _DEVICE))
    return Propagation(adopt(GaussianScalarField, g, mu, sg), ps, pk)


def propagate_with_probabilities3d(model: GaussianVectorField3, t: float = 0.0, *,
                                   probabilities: bool = True, chunk_planes: int = 16) -> Propagation:
    """3D twin (fp32 models use the pipelined host entry point; fp64 models
    are staged through torch and run the fp64 kernel)."""
    g = model.grid
    n = g.n_vertices
    dt = model.dtype
    ins = [model.mu_u, model.mu_v, model.mu_w, model.sigma_u, model.sigma_v, model.sigma_w]
    mu = np.empty(n, dtype=dt)
    sg = np.empty(n, dtype=dt)
    ps = np.empty(n, dtype=dt) if probabilities else None
    pk = np.empty(n, dtype=dt) if probabilities else None
    if dt == np.float32:
        _check(lib.divuq_host_propagate3d_f32(
            *(_p(a) for a in ins), g.nx, g.ny, g.nz, float(g.dx), float(g.dy), float(g.dz),
            float(t), _p(mu), _p(sg), _p(ps), _p(pk), int(chunk_planes), _DEVICE))
    else:
        import torch

        from . import device as dev

        with torch.cuda.device(_DEVICE):
            tens = [torch.from_numpy(np.array(a)).cuda() for a in ins]
            outs = ("mu", "sigma", "p_src", "p_snk") if probabilities else ("mu", "sigma")
            o = dev.propagate3d(*tens, g.nx, g.ny, g.nz, g.dx, g.dy, g.dz, t, outputs=outs)
            mu[:] = o["mu"].cpu().numpy()
            sg[:] = o["sigma"].cpu().numpy()
            if probabilities:
                ps[:] = o["p_src"].cpu().numpy()
                pk[:] = o["p_snk"].cpu().numpy()
    return Propagation(adopt(GaussianScalarField3, g, mu, sg), ps, pk)


def divergence_deterministic(fld: VectorField2) -> ScalarField2:
    """du/dx + dv/dy with the one-sided boundary rule (divergence.py:41-45)."""
    g = fld.grid
    out = np.empty(g.n_vertices)
    _check(lib.divuq_host_propagate2d_f64(
        _p(fld.u), _p(fld.v), None, None, g.nx, g.ny, float(g.dx), float(g.dy), 0.0, _p(out),
        None, None, None, _DEVICE))
    return adopt(ScalarField2, g, out)


def stencil_distribution(neighbors, spacing: tuple[float, float]) -> tuple[float, float]:
    """Single interior vertex (divergence.py:73-85): four scalars, host-side by
    design -- a kernel launch would cost more than the math."""
    (mu_um, s_um), (mu_up, s_up), (mu_vm, s_vm), (mu_vp, s_vp) = neighbors
    dx, dy = spacing
    cx, cy = 1.0 / (2.0 * dx), 1.0 / (2.0 * dy)
    mu = mu_up * cx - mu_um * cx + mu_vp * cy - mu_vm * cy
    var = (s_up * cx) ** 2 + (s_um * cx) ** 2 + (s_vp * cy) ** 2 + (s_vm * cy) ** 2
    return float(mu), float(np.sqrt(var))


def tail_probs(mu, sigma, isovalue: float):
    """(P[X <= theta], P[X > theta]) per vertex (lcp.py:48-68), on the GPU."""
    mu = _c64(mu)
    sigma = _c64(sigma)
    if mu.shape != sigma.shape:
        raise ValueError("mu and sigma must have the same shape")
    below = _out(mu.shape, mu.dtype)
    above = _out(mu.shape, mu.dtype)
    _check(lib.divuq_host_tail_probs_f64(_p(mu), _p(sigma), mu.size, float(isovalue), _p(below),
                                         _p(above), _DEVICE))
    return below, above


def _one_tail(mu, sigma, isovalue: float, above: bool) -> np.ndarray:
    """One of tail_probs' two maps: only that map is computed and copied back."""
    mu = _c64(mu)
    sigma = _c64(sigma)
    if mu.shape != sigma.shape:
        raise ValueError("mu and sigma must have the same shape")
    out = _out(mu.shape, mu.dtype)
    _check(lib.divuq_host_tail_probs_f64(_p(mu), _p(sigma), mu.size, float(isovalue),
                                         None if above else _p(out), _p(out) if above else None,
                                         _DEVICE))
    return out


def source_probability(fld: GaussianScalarField, t: float = 0.0) -> np.ndarray:
    """P(div > t) per vertex: the reference's 'above' tail at isovalue t."""
    return _one_tail(fld.mu, fld.sigma, t, above=True)


def sink_probability(fld: GaussianScalarField, t: float = 0.0) -> np.ndarray:
    """P(div < -t) per vertex (P(div <= -t) on the sigma == 0 tie, lcp.py:56-59)."""
    return _one_tail(fld.mu, fld.sigma, -t, above=False)


def mc_divergence(model: GaussianVectorField, config: McConfig, *,
                  stream: str = "philox") -> McDivergenceEstimate:
    """Per-vertex empirical divergence mean/std (mc.py:94-117).

    ``stream="philox"`` (default, the north star's kernel): Philox4x32-10 +
    Box-Muller draws, statistically equivalent to the reference; deterministic
    in (model, seed, n) and invariant to launch shape.
    ``stream="reference"``: the reference's own splitmix64 + AS241 stream,
    counters and single-pass Welford, so the estimate reproduces the
    reference's ``mc_divergence`` draw for draw (golden-tested).
    """
    if config.n_samples < 2:
        raise ValueError("mc_divergence needs n_samples >= 2")
    if stream not in ("philox", "reference"):
        raise ValueError("stream must be 'philox' or 'reference'")
    g = model.grid
    n = g.n_vertices
    mean = _out(n)
    std = _out(n)
    fn = (lib.divuq_host_mc_divergence2d_f64 if stream == "philox"
          else lib.divuq_host_mc_divergence2d_ref_f64)
    _check(fn(
        _p(model.mu_u), _p(model.mu_v), _p(model.sigma_u), _p(model.sigma_v), g.nx, g.ny,
        float(g.dx), float(g.dy), int(config.n_samples), int(config.seed), _p(mean), _p(std),
        _DEVICE))
    return adopt(McDivergenceEstimate, g, mean, std, config.n_samples)


def _neighbors8(neighbors) -> np.ndarray:
    nb = np.ascontiguousarray(np.asarray(neighbors, dtype=np.float64).reshape(4, 2)).ravel()
    if np.any(nb[1::2] < 0):
        raise ValueError("sigmas must be non-negative")   # mc.py:147-149
    return nb


def sample_divergence_1d(neighbors, spacing: tuple[float, float], config: McConfig) -> np.ndarray:
    """Raw single-vertex divergence samples (mc.py:142-156), reference stream.

    neighbors: four (mu, sigma) pairs in stencil order -- u at i-1, u at i+1,
    v at j-1, v at j+1.  Draw k uses counters 4k..4k+3 of the reference's
    splitmix64 + AS241 stream, so the samples equal the reference's.
    """
    nb = _neighbors8(neighbors)
    dx, dy = spacing
    n = int(config.n_samples)
    values = np.empty(n)
    edges = np.empty(2)
    counts = np.empty(1, dtype=np.int64)
    used = np.zeros(1, dtype=np.int64)
    _check(lib.divuq_host_mc_histogram1d_f64(
        _p(nb), float(dx), float(dy), n, int(config.seed), 1, _p(edges), _p(counts), _p(used),
        _p(values), _DEVICE))
    return values


def mc_histogram_1d(neighbors, spacing: tuple[float, float], config: McConfig,
                    n_bins: int) -> McHistogram:
    """Histogram of sampled single-vertex divergence (mc.py:120-139).

    Samples, [min, max] and np.histogram's uniform-bin rule all run on the
    GPU; all-identical draws give the reference's one-bin histogram.
    """
    if n_bins < 1:
        raise ValueError("n_bins must be >= 1")
    nb = _neighbors8(neighbors)
    dx, dy = spacing
    edges = np.empty(n_bins + 1)
    counts = np.empty(n_bins, dtype=np.int64)
    used = np.zeros(1, dtype=np.int64)
    _check(lib.divuq_host_mc_histogram1d_f64(
        _p(nb), float(dx), float(dy), int(config.n_samples), int(config.seed), int(n_bins),
        _p(edges), _p(counts), _p(used), None, _DEVICE))
    k = int(used[0])
    return McHistogram(edges[: k + 1].copy(), counts[:k].copy(), int(config.n_samples))


def error_metrics(estimate: McDivergenceEstimate, analytic: GaussianScalarField):
    """(e_m, e_sigma, sse) between estimate and model (mc.py:159-175), one
    device reduction (divuq_host_error_metrics_f64); within ~1e-15 relative of
    numpy's pairwise sums."""
    if estimate.grid != analytic.grid:
        raise ValueError("estimate and analytic fields are on different grids")
    out = np.empty(3)
    _check(lib.divuq_host_error_metrics_f64(_p(estimate.mean), _p(estimate.std), _p(analytic.mu),
                                            _p(analytic.sigma), estimate.grid.n_vertices, _p(out),
                                            _DEVICE))
    return float(out[0]), float(out[1]), float(out[2])


class EnsembleDivergence(NamedTuple):
    model: GaussianVectorField      # fitted moments (fp32-rounded, returned as fp64)
    field: GaussianScalarField
    p_src: np.ndarray
    p_snk: np.ndarray


def ensemble_divergence(ensemble: Ensemble2, t: float = 0.0) -> EnsembleDivergence:
    """Fused fp32 pipeline fit_gaussian -> propagate_divergence -> tail maps
    (BASELINE config 1): one pass over the members on the GPU."""
    g = ensemble.grid
    stacked = np.ascontiguousarray(ensemble.stacked(), dtype=np.float32)
    m = stacked.shape[0]
    n = g.n_vertices
    o = [np.empty(n, dtype=np.float32) for _ in range(4)]
    mom_mu = np.empty((2, n), dtype=np.float32)
    mom_sg = np.empty((2, n), dtype=np.float32)
    _check(lib.divuq_host_ensemble_divergence2d_f32(
        _p(stacked), m, g.nx, g.ny, float(g.dx), float(g.dy), float(t), *(_p(a) for a in o),
        _p(mom_mu), _p(mom_sg), _DEVICE))
    model = GaussianVectorField(g, mom_mu[0], mom_mu[1], mom_sg[0], mom_sg[1])
    return EnsembleDivergence(model, GaussianScalarField(g, o[0], o[1]), o[2].astype(np.float64),
                              o[3].astype(np.float64))


def _wplanes(a, m, plane):
    """(M, plane) fp32 w-component planes -> (array, member stride in floats);
    a row-strided view (e.g. members[:, 2, k*plane:(k+1)*plane]) is passed
    without a copy."""
    a = np.asarray(a)
    if a.shape != (m, plane):
        raise ValueError(f"ghost planes must have shape ({m}, {plane})")
    if a.dtype != np.float32 or a.strides[1] != 4 or a.strides[0] % 4:
        a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.strides[0] // 4


def ensemble_divergence3d(members, grid: UniformGrid3, t: float = 0.0, *, z0: int = 0,
                          nz_global: int | None = None, ghost_lo=None, ghost_hi=None,
                          chunk_planes: int = 0) -> Propagation:
    """Fused fp32 3D ensemble pipeline (BASELINE config 4) from host buffers.

    members: (M, 3, nx*ny*nz) with grid the slab's grid (nz planes), covering
    global planes [z0, z0+nz) of nz_global (default: the slab is the whole
    volume).  ghost_lo / ghost_hi: (M, nx*ny) w-component member planes at
    global z0-1 / z0+nz, required when those planes exist.  The member data
    crosses PCIe once in a 3-stream z-chunk pipeline."""
    g = grid
    plane = g.nx * g.ny
    mem = np.asarray(members)
    if mem.ndim != 3 or mem.shape[1:] != (3, g.n_vertices):
        raise ValueError(f"members must have shape (M, 3, {g.n_vertices})")
    mem = np.ascontiguousarray(mem, dtype=np.float32)
    m = mem.shape[0]
    nzg = g.nz if nz_global is None else int(nz_global)
    lo, lo_s = _wplanes(ghost_lo, m, plane) if ghost_lo is not None else (None, plane)
    hi, hi_s = _wplanes(ghost_hi, m, plane) if ghost_hi is not None else (None, plane)
    if lo is not None and hi is not None and lo_s != hi_s:
        lo = np.ascontiguousarray(lo)
        hi = np.ascontiguousarray(hi)
        lo_s = hi_s = plane
    stride = lo_s if lo is not None else hi_s
    o = [np.empty(g.n_vertices, dtype=np.float32) for _ in range(4)]
    _check(lib.divuq_host_ensemble_divergence3d_f32(
        _p(mem), m, g.nx, g.ny, g.nz, int(z0), nzg, _p(lo), _p(hi), stride, float(g.dx),
        float(g.dy), float(g.dz), float(t), *(_p(a) for a in o), int(chunk_planes), _DEVICE))
    return Propagation(adopt(GaussianScalarField3, g, o[0], o[1]), o[2], o[3])


def gradient_ensemble_divergence(ensemble: Ensemble2, t: float = 0.0) -> EnsembleDivergence:
    """The Red Sea pipeline in one fp32 pass: gradient_ensemble (velocity
    magnitude gradient per member) -> fit_gaussian -> propagate_divergence ->
    tail maps.  ``model`` of the result is the gradient ensemble's Gaussian fit."""
    g = ensemble.grid
    stacked = np.ascontiguousarray(ensemble.stacked(), dtype=np.float32)
    m = stacked.shape[0]
    n = g.n_vertices
    o = [np.empty(n, dtype=np.float32) for _ in range(4)]
    mom_mu = np.empty((2, n), dtype=np.float32)
    mom_sg = np.empty((2, n), dtype=np.float32)
    _check(lib.divuq_host_gradient_ensemble_divergence2d_f32(
        _p(stacked), m, g.nx, g.ny, float(g.dx), float(g.dy), float(t), *(_p(a) for a in o),
        _p(mom_mu), _p(mom_sg), _DEVICE))
    model = GaussianVectorField(g, mom_mu[0], mom_mu[1], mom_sg[0], mom_sg[1])
    return EnsembleDivergence(model, GaussianScalarField(g, o[0], o[1]), o[2].astype(np.float64),
                              o[3].astype(np.float64))


def velocity_magnitude(member: VectorField2) -> ScalarField2:
    """hypot(u, v) per vertex (gaussian.py:48-50)."""
    g = member.grid
    out = np.empty(g.n_vertices)
    _check(lib.divuq_host_velocity_magnitude_f64(_p(member.u), _p(member.v), g.n_vertices, _p(out),
                                                 _DEVICE))
    return adopt(ScalarField2, g, out)


def gradient(fld: ScalarField2) -> VectorField2:
    """Central-difference gradient, one-sided on the boundary (gaussian.py:53-58)."""
    g = fld.grid
    out = np.empty((2, g.n_vertices))
    _check(lib.divuq_host_gradient2d_f64(_p(fld.values), g.nx, g.ny, float(g.dx), float(g.dy),
                                         _p(out), _DEVICE))
    return adopt(VectorField2, g, out[0], out[1])


def gradient_ensemble(ensemble: Ensemble2) -> Ensemble2:
    """Each member through velocity_magnitude then gradient (gaussian.py:61-66),
    fused on the GPU: the magnitude field is never materialised."""
    g = ensemble.grid
    stacked = _c64(ensemble.stacked())
    out = np.empty_like(stacked)
    _check(lib.divuq_host_gradient_ensemble2d_f64(_p(stacked), stacked.shape[0], g.nx, g.ny,
                                                  float(g.dx), float(g.dy), _p(out), _DEVICE))
    return Ensemble2(g, tuple(adopt(VectorField2, g, o[0], o[1]) for o in out))


def cell_crossing_probability(mu, sigma, isovalue: float) -> np.ndarray:
    """LCP for stacked cells: mu, sigma of shape (..., 4) (lcp.py:71-77)."""
    mu = _c64(mu)
    sigma = _c64(sigma)
    if mu.shape != sigma.shape or mu.shape[-1:] != (4,):
        raise ValueError("mu and sigma must have the same shape (..., 4)")
    out = np.empty(mu.shape[:-1])
    _check(lib.divuq_host_cell_crossing_f64(_p(mu), _p(sigma), out.size, float(isovalue), _p(out),
                                            _DEVICE))
    return out


def propagate_lcp(model, isovalue: float) -> tuple[GaussianScalarField, LcpField]:
    """propagate_divergence(model) then lcp(field, isovalue) in one fused pass
    (divergence.py:48-70 + lcp.py:80-100): both results bitwise equal to the
    two-call chain (and so to the reference's), without staging the
    divergence field through host memory in between."""
    g = model.grid
    n = g.n_vertices
    mu, sg, out = _out(n), _out(n), _out(g.n_cells)
    _check(lib.divuq_host_propagate_lcp2d_f64(
        _p(model.mu_u), _p(model.mu_v), _p(model.sigma_u), _p(model.sigma_v), g.nx, g.ny,
        float(g.dx), float(g.dy), float(isovalue), _p(mu), _p(sg), _p(out), _DEVICE))
    return adopt(GaussianScalarField, g, mu, sg), adopt(LcpField, g, isovalue, out)


def lcp(fld: GaussianScalarField, isovalue: float, config: ParallelConfig | None = None) -> LcpField:
    """Crossing probability of the isovalue for every grid cell (lcp.py:80-100)."""
    g = fld.grid
    out = _out(g.n_cells)
    _check(lib.divuq_host_lcp2d_f64(_p(fld.mu), _p(fld.sigma), g.nx, g.ny, float(isovalue), _p(out),
                                    _DEVICE))
    return adopt(LcpField, g, isovalue, out)
