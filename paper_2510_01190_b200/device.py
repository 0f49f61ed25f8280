"""Device-resident API: torch CUDA tensors in, torch CUDA tensors out.

This is the path the benchmark times (inputs already in HBM).  Every call is
one or two launches of the hand-written sm_100a kernels in libdivuq_b200.so,
enqueued on torch's current stream.  PyTorch only provides the memory and
the stream.  ``check=True`` synchronises and raises ``ValueError`` when the
kernels' validation word reports non-finite inputs or negative sigmas (the
reference's construction-time checks, grid.py:26-27 / divergence.py:34-35).
"""

from __future__ import annotations

import torch

from . import _lib
from ._lib import check as _check
from ._lib import lib

_FP = {torch.float64: "f64", torch.float32: "f32"}


def _ptr(t):
    """Device address of a tensor; an int is taken as a raw device address
    (e.g. a neighbour's peer-mapped halo plane, peer.py)."""
    if t is None or isinstance(t, int):
        return t
    return t.data_ptr()


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream():
    """torch's current stream on the current device, as a raw handle (the
    private getter costs ~0.3 us against ~3.3 us for the public object)."""
    if _raw_stream is not None:
        return _raw_stream(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


def _req(t, name, dtype=None, numel=None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name}: expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name}: expected a contiguous tensor")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name}: expected {numel} values, got {t.numel()}")
    return t


def raise_for_bits(bits: int) -> None:
    """The reference's exceptions for the kernels' validation bits
    (grid.py:26-27 non-finite; divergence.py:34-35 / gaussian.py:28-29 sigma < 0)."""
    if bits & 1:
        raise ValueError("non-finite values are not allowed")
    if bits & 2:
        raise ValueError("sigma must be non-negative")


class _ErrWord:
    """Device int32 validation word.  ``check=True``: a fresh word, read (one
    sync) and raised after the call; ``check=<int32 CUDA tensor>``: the
    kernels OR their bits into the caller's word and nothing is read back --
    the caller checks once after many calls (``raise_for_bits``);
    ``check=False``: no validation."""

    def __init__(self, device, enabled):
        if isinstance(enabled, torch.Tensor):
            if enabled.dtype != torch.int32 or not enabled.is_cuda or enabled.numel() < 1:
                raise TypeError("check: an int32 CUDA tensor (the validation word)")
            self.t, self.deferred = enabled, True
        else:
            self.t = torch.zeros(1, dtype=torch.int32, device=device) if enabled else None
            self.deferred = False

    @property
    def ptr(self):
        return _ptr(self.t)

    def raise_if_set(self):
        if self.t is None or self.deferred:
            return
        raise_for_bits(int(self.t.item()))


def _outs(like, n, names, out):
    out = dict(out or {})
    for k in names:
        if k not in out:
            out[k] = torch.empty(n, dtype=like.dtype, device=like.device)
        else:
            _req(out[k], k, like.dtype, n)
    return out


ALL_OUTPUTS = ("mu", "sigma", "p_src", "p_snk")


def propagate2d(mu_u, mu_v, s_u, s_v, nx, ny, dx=1.0, dy=1.0, t=0.0, *,
                outputs=ALL_OUTPUTS, out=None, check=True):
    """K2 2D: divergence mean, sigma, P(div>t), P(div<-t) (divergence.py:48-70, lcp.py:48-68).

    ``s_u``/``s_v`` may be None when ``outputs == ("mu",)`` (the reference's
    divergence_deterministic, divergence.py:41-45).  Returns a dict.
    """
    dt = mu_u.dtype
    n = nx * ny
    for name, x in (("mu_u", mu_u), ("mu_v", mu_v)):
        _req(x, name, dt, n)
    need_sigma = any(k != "mu" for k in outputs)
    if need_sigma:
        for name, x in (("s_u", s_u), ("s_v", s_v)):
            _req(x, name, dt, n)
    o = _outs(mu_u, n, outputs, out)
    err = _ErrWord(mu_u.device, check)
    fn = getattr(lib, f"divuq_propagate2d_{_FP[dt]}")
    _check(fn(_ptr(mu_u), _ptr(mu_v), _ptr(s_u) if need_sigma else None,
              _ptr(s_v) if need_sigma else None, nx, ny, float(dx), float(dy), float(t),
              _ptr(o.get("mu")), _ptr(o.get("sigma")), _ptr(o.get("p_src")), _ptr(o.get("p_snk")),
              err.ptr, _stream()))
    err.raise_if_set()
    return o


def propagate3d(mu_u, mu_v, mu_w, s_u, s_v, s_w, nx, ny, nz_local, dx=1.0, dy=1.0, dz=1.0,
                t=0.0, *, z0=0, nz_global=None, halo_lo=None, halo_hi=None, k_range=None,
                outputs=ALL_OUTPUTS, out=None, check=True):
    """K2 3D on a z-slab: planes [z0, z0+nz_local) of a grid of nz_global planes.

    ``halo_lo`` / ``halo_hi`` = (mu_w, s_w) planes at global z0-1 / z0+nz_local,
    needed only when those planes exist.  ``k_range`` = (kb, ke) local planes
    to compute (default all); outputs are slab-sized and only those planes are
    written.
    """
    dt = mu_u.dtype
    nzg = nz_local if nz_global is None else nz_global
    n = nx * ny * nz_local
    fields = {"mu_u": mu_u, "mu_v": mu_v, "mu_w": mu_w, "s_u": s_u, "s_v": s_v, "s_w": s_w}
    for name, x in fields.items():
        _req(x, name, dt, n)
    plane = nx * ny
    hl = halo_lo or (None, None)
    hh = halo_hi or (None, None)
    for h in (*hl, *hh):
        if h is not None and not isinstance(h, int):
            _req(h, "halo", dt, plane)
    kb, ke = (0, nz_local) if k_range is None else k_range
    o = _outs(mu_u, n, outputs, out)
    err = _ErrWord(mu_u.device, check)
    fn = getattr(lib, f"divuq_propagate3d_{_FP[dt]}")
    _check(fn(*(_ptr(x) for x in fields.values()), _ptr(hl[0]), _ptr(hl[1]), _ptr(hh[0]),
              _ptr(hh[1]), nx, ny, nz_local, z0, nzg, kb, ke, float(dx), float(dy), float(dz),
              float(t), _ptr(o.get("mu")), _ptr(o.get("sigma")), _ptr(o.get("p_src")),
              _ptr(o.get("p_snk")), err.ptr, _stream()))
    err.raise_if_set()
    return o


def tail_probs(mu, sigma, theta, *, check=True):
    """(P[X <= theta], P[X > theta]) elementwise (lcp.py:48-68)."""
    dt = mu.dtype
    _req(mu, "mu", dt)
    _req(sigma, "sigma", dt, mu.numel())
    below = torch.empty_like(mu)
    above = torch.empty_like(mu)
    err = _ErrWord(mu.device, check)
    fn = getattr(lib, f"divuq_tail_probs_{_FP[dt]}")
    _check(fn(_ptr(mu), _ptr(sigma), mu.numel(), float(theta), _ptr(below), _ptr(above), err.ptr,
              _stream()))
    err.raise_if_set()
    return below, above


def lcp2d(mu, sigma, nx, ny, isovalue, *, check=True):
    """Per-cell level-crossing probability ((ny-1)*(nx-1),) (lcp.py:80-100)."""
    dt = mu.dtype
    _req(mu, "mu", dt, nx * ny)
    _req(sigma, "sigma", dt, nx * ny)
    out = torch.empty((nx - 1) * (ny - 1), dtype=dt, device=mu.device)
    err = _ErrWord(mu.device, check)
    fn = getattr(lib, f"divuq_lcp2d_{_FP[dt]}")
    _check(fn(_ptr(mu), _ptr(sigma), nx, ny, float(isovalue), _ptr(out), err.ptr, _stream()))
    err.raise_if_set()
    return out


def propagate_lcp2d(mu_u, mu_v, s_u, s_v, nx, ny, dx=1.0, dy=1.0, isovalue=0.0, *,
                    moments=True, out=None, check=True):
    """propagate_divergence -> lcp fused (one pass, fp64): dict with "lcp"
    ((ny-1)*(nx-1),) and, if ``moments``, the divergence "mu", "sigma" (N,).
    Bitwise equal to propagate2d followed by lcp2d."""
    n = nx * ny
    for name, x in (("mu_u", mu_u), ("mu_v", mu_v), ("s_u", s_u), ("s_v", s_v)):
        _req(x, name, torch.float64, n)
    o = dict(out or {})
    o.setdefault("lcp", torch.empty((nx - 1) * (ny - 1), dtype=torch.float64, device=mu_u.device))
    if moments:
        o.setdefault("mu", torch.empty(n, dtype=torch.float64, device=mu_u.device))
        o.setdefault("sigma", torch.empty(n, dtype=torch.float64, device=mu_u.device))
    err = _ErrWord(mu_u.device, check)
    _check(lib.divuq_propagate_lcp2d_f64(
        _ptr(mu_u), _ptr(mu_v), _ptr(s_u), _ptr(s_v), nx, ny, float(dx), float(dy), float(isovalue),
        _ptr(o.get("mu")), _ptr(o.get("sigma")), _ptr(o["lcp"]), err.ptr, _stream()))
    err.raise_if_set()
    return o


def gradient_ensemble2d(members, nx, ny, dx=1.0, dy=1.0, *, out=None, check=True):
    """(M, 2, nx*ny) members -> (M, 2, nx*ny) gradients of |(u, v)| (gaussian.py:61-66)."""
    _req(members, "members")
    if members.dim() != 3 or members.shape[1:] != (2, nx * ny):
        raise ValueError("members must have shape (M, 2, nx*ny)")
    out = torch.empty_like(members) if out is None else _req(out, "out", members.dtype, members.numel())
    err = _ErrWord(members.device, check)
    fn = getattr(lib, f"divuq_gradient_ensemble2d_{_FP[members.dtype]}")
    _check(fn(_ptr(members), members.shape[0], nx, ny, float(dx), float(dy), _ptr(out), err.ptr,
              _stream()))
    err.raise_if_set()
    return out


def fit_moments(members, *, out=None, check=True):
    """K1: (M, C, N) members -> mu (C, N), sigma (C, N) (gaussian.py:35-45)."""
    _req(members, "members")
    if members.dim() != 3:
        raise ValueError("members must have shape (M, C, N)")
    m, c, n = members.shape
    mu, sg = out if out is not None else (
        torch.empty((c, n), dtype=members.dtype, device=members.device),
        torch.empty((c, n), dtype=members.dtype, device=members.device))
    err = _ErrWord(members.device, check)
    fn = getattr(lib, f"divuq_fit_gaussian_{_FP[members.dtype]}")
    _check(fn(_ptr(members), m, c, n, _ptr(mu), _ptr(sg), err.ptr, _stream()))
    err.raise_if_set()
    return mu, sg


def ensemble_divergence2d(members, nx, ny, dx=1.0, dy=1.0, t=0.0, *, moments=False,
                          outputs=ALL_OUTPUTS, out=None, check=True):
    """K3 2D fused: (M, 2, nx*ny) fp32 members -> outputs (+ moments (2, N) if asked)."""
    _req(members, "members", torch.float32)
    m = members.shape[0]
    if members.shape[1:] != (2, nx * ny):
        raise ValueError("members must have shape (M, 2, nx*ny)")
    n = nx * ny
    o = _outs(members, n, outputs, out)
    if moments:
        o.setdefault("mom_mu", torch.empty((2, n), dtype=members.dtype, device=members.device))
        o.setdefault("mom_sigma", torch.empty((2, n), dtype=members.dtype, device=members.device))
    err = _ErrWord(members.device, check)
    _check(lib.divuq_ensemble_divergence2d_f32(
        _ptr(members), m, nx, ny, float(dx), float(dy), float(t), _ptr(o.get("mu")),
        _ptr(o.get("sigma")), _ptr(o.get("p_src")), _ptr(o.get("p_snk")), _ptr(o.get("mom_mu")),
        _ptr(o.get("mom_sigma")), err.ptr, _stream()))
    err.raise_if_set()
    return o


def gradient_ensemble_divergence2d(members, nx, ny, dx=1.0, dy=1.0, t=0.0, *, moments=False,
                                   outputs=ALL_OUTPUTS, out=None, check=True):
    """K6 fused Red Sea pipeline: (M, 2, nx*ny) fp32 velocity members ->
    |v| -> gradient -> moments -> divergence -> tails in one pass (moments:
    the gradient ensemble's (2, N) mu / sigma)."""
    _req(members, "members", torch.float32)
    m = members.shape[0]
    if members.shape[1:] != (2, nx * ny):
        raise ValueError("members must have shape (M, 2, nx*ny)")
    n = nx * ny
    o = _outs(members, n, outputs, out)
    if moments:
        o.setdefault("mom_mu", torch.empty((2, n), dtype=members.dtype, device=members.device))
        o.setdefault("mom_sigma", torch.empty((2, n), dtype=members.dtype, device=members.device))
    err = _ErrWord(members.device, check)
    _check(lib.divuq_gradient_ensemble_divergence2d_f32(
        _ptr(members), m, nx, ny, float(dx), float(dy), float(t), _ptr(o.get("mu")),
        _ptr(o.get("sigma")), _ptr(o.get("p_src")), _ptr(o.get("p_snk")), _ptr(o.get("mom_mu")),
        _ptr(o.get("mom_sigma")), err.ptr, _stream()))
    err.raise_if_set()
    return o


def ensemble_divergence3d(members, nx, ny, nz_local, dx=1.0, dy=1.0, dz=1.0, t=0.0, *, z0=0,
                          nz_global=None, halo_lo=None, halo_hi=None, k_range=None,
                          moments=False, outputs=ALL_OUTPUTS, out=None, check=True):
    """K3 3D fused on a z-slab: (M, 3, nx*ny*nz_local) fp32 members.

    Halos are REDUCED w moments (mu_w, s_w, r_w) of the planes just outside
    the slab (see ``w_moments_plane``; r_w, the means' rounding residuals,
    may be omitted and then reads as 0)."""
    _req(members, "members", torch.float32)
    m = members.shape[0]
    n = nx * ny * nz_local
    if members.shape[1:] != (3, n):
        raise ValueError("members must have shape (M, 3, nx*ny*nz_local)")
    nzg = nz_local if nz_global is None else nz_global
    kb, ke = (0, nz_local) if k_range is None else k_range
    hl = tuple(halo_lo or ()) + (None,) * (3 - len(halo_lo or ()))
    hh = tuple(halo_hi or ()) + (None,) * (3 - len(halo_hi or ()))
    for h in hl + hh:
        if h is not None:
            _req(h, "halo", torch.float32, nx * ny)
    o = _outs(members, n, outputs, out)
    if moments:
        o.setdefault("mom_mu", torch.empty((3, n), dtype=members.dtype, device=members.device))
        o.setdefault("mom_sigma", torch.empty((3, n), dtype=members.dtype, device=members.device))
    err = _ErrWord(members.device, check)
    _check(lib.divuq_ensemble_divergence3d_f32(
        _ptr(members), m, _ptr(hl[0]), _ptr(hl[1]), _ptr(hl[2]), _ptr(hh[0]), _ptr(hh[1]),
        _ptr(hh[2]), nx, ny, nz_local,
        z0, nzg, kb, ke, float(dx), float(dy), float(dz), float(t), _ptr(o.get("mu")),
        _ptr(o.get("sigma")), _ptr(o.get("p_src")), _ptr(o.get("p_snk")), _ptr(o.get("mom_mu")),
        _ptr(o.get("mom_sigma")), err.ptr, _stream()))
    err.raise_if_set()
    return o


def w_moments_plane(members, nx, ny, nz_local, k, *, out=None, check=True):
    """(mu_w, s_w, r_w) of local plane k of a 3D member slab -- the reduced halo
    a z-slab neighbour needs.  Same K1 arithmetic as the fused kernel, so the
    sharded result stays bit-identical to the single-GPU one.  Read in place
    (member-strided), no gather copy."""
    _req(members, "members", torch.float32)
    m = members.shape[0]
    plane = nx * ny
    if members.numel() != m * 3 * plane * nz_local:
        raise ValueError("members: expected (M, 3, nx*ny*nz_local)")
    return w_moments_plane_ptr(members.data_ptr(), m, nx, ny, nz_local, k, device=members.device,
                               out=out, check=check)


def w_moments_plane_ptr(members_ptr: int, m, nx, ny, nz_local, k, *, device, out=None, check=True):
    """``w_moments_plane`` on a raw (M, 3, nx*ny*nz_local) fp32 slab address --
    typically a neighbour's slab mapped through peer memory (peer.py): the
    fit kernel then reads the neighbour's member planes over NVLink."""
    plane = nx * ny
    n = plane * nz_local
    if not (0 <= k < nz_local):
        raise ValueError("plane index outside the slab")
    mu, sg, r = out if out is not None else tuple(
        torch.empty(plane, dtype=torch.float32, device=device) for _ in range(3))
    err = _ErrWord(device, check)
    base = int(members_ptr) + (2 * n + k * plane) * 4   # component w, plane k, member 0
    _check(lib.divuq_fit_gaussian_strided_f32(base, m, 3 * n, plane, _ptr(mu), _ptr(sg), _ptr(r),
                                              err.ptr, _stream()))
    err.raise_if_set()
    return mu, sg, r


_EM_SCRATCH = {}


def error_metrics(est_mean, est_std, mu, sigma):
    """error_metrics (mc.py:159-175) on the device, one launch: a (3,) fp64
    CUDA tensor (e_m, e_sigma, sse); nothing is read back."""
    n = est_mean.numel()
    for name, x in (("est_mean", est_mean), ("est_std", est_std), ("mu", mu), ("sigma", sigma)):
        _req(x, name, torch.float64, n)
    dev = est_mean.device
    key = (dev.index, torch.cuda.current_stream(dev).cuda_stream)
    if key not in _EM_SCRATCH:   # zeroed once; the kernel leaves its ticket at 0
        _EM_SCRATCH[key] = torch.zeros(lib.divuq_error_metrics_scratch_bytes(), dtype=torch.uint8,
                                       device=dev)
    out = torch.empty(3, dtype=torch.float64, device=dev)
    _check(lib.divuq_error_metrics_f64(_ptr(est_mean), _ptr(est_std), _ptr(mu), _ptr(sigma), n,
                                       _ptr(out), _ptr(_EM_SCRATCH[key]), _stream()))
    return out


def mc_divergence2d(mu_u, mu_v, s_u, s_v, nx, ny, dx, dy, n_samples, seed, *, rows=None,
                    out=None, check=True, stream="philox"):
    """K4: Monte Carlo estimate for rows [r0, r1) (default all).

    stream="philox": the north star's Philox4x32-10 + Box-Muller kernel;
    stream="reference": the reference's splitmix64 + AS241 stream and
    single-pass Welford (draw-for-draw parity with mc.py:94-117).
    """
    if stream not in ("philox", "reference"):
        raise ValueError("stream must be 'philox' or 'reference'")
    n = nx * ny
    for name, x in (("mu_u", mu_u), ("mu_v", mu_v), ("s_u", s_u), ("s_v", s_v)):
        _req(x, name, torch.float64, n)
    if n_samples < 2:
        raise ValueError("mc_divergence needs n_samples >= 2")
    if not (0 <= int(seed) < 2**64):
        raise ValueError("seed must fit in 64 unsigned bits")
    r0, r1 = (0, ny) if rows is None else rows
    nv = (r1 - r0) * nx
    mean, std = out if out is not None else (
        torch.empty(nv, dtype=torch.float64, device=mu_u.device),
        torch.empty(nv, dtype=torch.float64, device=mu_u.device))
    err = _ErrWord(mu_u.device, check)
    if stream == "reference":
        _check(lib.divuq_mc_divergence2d_ref_f64(
            _ptr(mu_u), _ptr(mu_v), _ptr(s_u), _ptr(s_v), nx, ny, float(dx), float(dy),
            n_samples, int(seed), r0, r1, _ptr(mean), _ptr(std), err.ptr, _stream()))
        err.raise_if_set()
        return mean, std
    scratch = torch.empty(max(1, lib.divuq_mc_scratch_bytes(nx, r0, r1, n_samples)),
                          dtype=torch.uint8, device=mu_u.device)
    _check(lib.divuq_mc_divergence2d_f64(
        _ptr(mu_u), _ptr(mu_v), _ptr(s_u), _ptr(s_v), nx, ny, float(dx), float(dy), n_samples,
        int(seed), r0, r1, _ptr(mean), _ptr(std), _ptr(scratch), err.ptr, _stream()))
    err.raise_if_set()
    return mean, std


__all__ = [
    "ALL_OUTPUTS", "propagate2d", "propagate3d", "tail_probs", "lcp2d", "propagate_lcp2d",
    "fit_moments",
    "ensemble_divergence2d", "ensemble_divergence3d", "gradient_ensemble_divergence2d",
    "w_moments_plane", "w_moments_plane_ptr",
    "mc_divergence2d", "error_metrics",
]
_ = _lib  # re-export guard
