"""3D restatement of the reference stencil -- TEST INFRASTRUCTURE ONLY.

The reference is 2D only.  This restates its
per-axis rule (stencils.py:46-51) for a third axis with stride nx*ny, keeping
the reference's evaluation order extended by z-terms last:

    mu  = ((((u_hi*cx - u_lo*cx) + v_hi*cy) - v_lo*cy) + w_hi*cz) - w_lo*cz
    var = (u_hi c)^2 + (u_lo c)^2 + (v_hi c)^2 + (v_lo c)^2 + (w_hi c)^2 + (w_lo c)^2

Layout: flat index (k*ny + j)*nx + i (pkg/README.md:101-103).
Parity status: pinned only by (a) bitwise reduction to the 2D reference on a
z-invariant field with w = 0 (tests/test_oracle.py) and (b) the identity,
rotation, uniform-sigma and zero-sigma invariants -- no reference 3D code or
golden vectors exist.

A z-slab helper evaluates the stencil of planes [z0, z1) of a global grid given
only those planes plus one ghost plane of (mu_w, sigma_w) on each side; it is
the CPU model of the multi-GPU halo exchange.
"""

from __future__ import annotations

import numpy as np

from .ref2d import axis_rule


def _terms(f3, axis: int, h: float):
    """(f[hi]*c, f[lo]*c) along ``axis`` of a (nz, ny, nx) array."""
    n = f3.shape[axis]
    lo, hi, c = axis_rule(n, h)
    shape = [1, 1, 1]
    shape[axis] = n
    c = c.reshape(shape)
    return np.take(f3, hi, axis=axis) * c, np.take(f3, lo, axis=axis) * c


def divergence3d(u, v, w, nx, ny, nz, dx, dy, dz):
    u3 = np.asarray(u, dtype=np.float64).reshape(nz, ny, nx)
    v3 = np.asarray(v, dtype=np.float64).reshape(nz, ny, nx)
    w3 = np.asarray(w, dtype=np.float64).reshape(nz, ny, nx)
    xh, xl = _terms(u3, 2, dx)
    yh, yl = _terms(v3, 1, dy)
    zh, zl = _terms(w3, 0, dz)
    return (((((xh - xl) + yh) - yl) + zh) - zl).ravel()


def divergence_variance3d(su, sv, sw, nx, ny, nz, dx, dy, dz):
    su3 = np.asarray(su, dtype=np.float64).reshape(nz, ny, nx)
    sv3 = np.asarray(sv, dtype=np.float64).reshape(nz, ny, nx)
    sw3 = np.asarray(sw, dtype=np.float64).reshape(nz, ny, nx)
    xh, xl = _terms(su3, 2, dx)
    yh, yl = _terms(sv3, 1, dy)
    zh, zl = _terms(sw3, 0, dz)
    return (((((xh * xh + xl * xl) + yh * yh) + yl * yl) + zh * zh) + zl * zl).ravel()


def propagate3d(mu_u, mu_v, mu_w, s_u, s_v, s_w, nx, ny, nz, dx, dy, dz):
    mu = divergence3d(mu_u, mu_v, mu_w, nx, ny, nz, dx, dy, dz)
    var = divergence_variance3d(s_u, s_v, s_w, nx, ny, nz, dx, dy, dz)
    return mu, np.sqrt(var)


def propagate3d_slab(fields, ghost_lo, ghost_hi, nx, ny, z0, nz_global, dx, dy, dz):
    """Stencil of global planes [z0, z0+nzl) from slab data plus w ghosts.

    ``fields`` = (mu_u, mu_v, mu_w, s_u, s_v, s_w) of the slab, each of shape
    (nzl*ny*nx,).  ``ghost_lo`` / ``ghost_hi`` are (mu_w, s_w) planes at global
    z0-1 and z0+nzl (ignored -- may be None -- at the global faces, where the
    one-sided rule uses the vertex itself).  Bit-identical to slicing
    ``propagate3d`` of the whole grid (tests/test_shard.py).
    """
    mu_u, mu_v, mu_w, s_u, s_v, s_w = (np.asarray(f, np.float64) for f in fields)
    nzl = mu_u.size // (nx * ny)
    plane = nx * ny
    # x/y terms are slab-local (no halo); z terms come from a ghost-padded column
    u3 = mu_u.reshape(nzl, ny, nx)
    v3 = mu_v.reshape(nzl, ny, nx)
    su3 = s_u.reshape(nzl, ny, nx)
    sv3 = s_v.reshape(nzl, ny, nx)
    xh, xl = _terms(u3, 2, dx)
    yh, yl = _terms(v3, 1, dy)
    sxh, sxl = _terms(su3, 2, dx)
    syh, syl = _terms(sv3, 1, dy)
    w_pad = [mu_w.reshape(nzl, ny, nx)]
    sw_pad = [s_w.reshape(nzl, ny, nx)]
    has_lo = z0 > 0
    has_hi = z0 + nzl < nz_global
    if has_lo:
        w_pad.insert(0, np.asarray(ghost_lo[0], np.float64).reshape(1, ny, nx))
        sw_pad.insert(0, np.asarray(ghost_lo[1], np.float64).reshape(1, ny, nx))
    if has_hi:
        w_pad.append(np.asarray(ghost_hi[0], np.float64).reshape(1, ny, nx))
        sw_pad.append(np.asarray(ghost_hi[1], np.float64).reshape(1, ny, nx))
    wp = np.concatenate(w_pad, axis=0)
    swp = np.concatenate(sw_pad, axis=0)
    kg = np.arange(z0, z0 + nzl)  # global plane ids
    lo_g = np.clip(kg - 1, 0, nz_global - 1)
    hi_g = np.clip(kg + 1, 0, nz_global - 1)
    cz = np.where((kg > 0) & (kg < nz_global - 1), 1.0 / (2.0 * dz), 1.0 / dz)[:, None, None]
    base = z0 - (1 if has_lo else 0)  # global id of wp[0]
    zh = wp[hi_g - base] * cz
    zl = wp[lo_g - base] * cz
    szh = swp[hi_g - base] * cz
    szl = swp[lo_g - base] * cz
    mu = (((((xh - xl) + yh) - yl) + zh) - zl).reshape(nzl * plane)
    var = (((((sxh * sxh + sxl * sxl) + syh * syh) + syl * syl) + szh * szh) + szl * szl)
    return mu, np.sqrt(var.reshape(nzl * plane))
