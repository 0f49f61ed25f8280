"""Seeded synthetic inputs for BASELINE.json configs 0-4 (bench / test inputs).

The paper's datasets are not available; BASELINE.json
defines synthetic stand-ins with the same shapes.  Mean fields follow the
reference's synthetic recipe (synthetic.py:30-52): Gaussian sources/sinks
A*(x-c)*exp(-|x-c|^2/w^2) with seeded centres, A = +-1, widths 5-15 cells,
plus a rotational vortex (2D) or a divergence-free shear flow (3D).  Small 2D
configs (0, 2) are generated on the host with numpy; 3D configs and the 2D
ensemble (1) are generated on the device by the K5 kernel, slab by slab, so
any GPU can build its own shard (counter-based noise).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from ._lib import check as _check
from ._lib import lib


@dataclass(frozen=True)
class Config:
    cid: int
    name: str
    nx: int
    ny: int
    nz: int = 1
    members: int = 0
    dtype: str = "f64"
    t: float = 0.0
    seed: int = 0
    n_samples: int = 0
    bytes_per_point: int = 0     # algorithmic (compulsory) HBM bytes per grid point

    @property
    def n_points(self) -> int:
        return self.nx * self.ny * self.nz


CONFIGS = {
    0: Config(0, "2D analytic fp64 128x128 (6 sources/sinks + vortex)", 128, 128, dtype="f64",
              seed=100, bytes_per_point=32 + 24),
    1: Config(1, "2D ensemble fp32 1024x1024 M=20, fused reduce+analytic+P(div>0)", 1024, 1024,
              members=20, dtype="f32", seed=101, bytes_per_point=20 * 2 * 4 + 3 * 4),
    2: Config(2, "2D Monte Carlo fp64 256x256 N=2000", 256, 256, dtype="f64", seed=102,
              n_samples=2000, bytes_per_point=48),
    3: Config(3, "3D analytic fp32 512^3 (64 sources/sinks + shear), P(div>0), P(div<0)", 512, 512,
              512, dtype="f32", t=0.0, seed=103, bytes_per_point=6 * 4 + 4 * 4),
    4: Config(4, "3D ensemble fp32 1024^3 M=16, fused, P(div>0.1), P(div<-0.1)", 1024, 1024, 1024,
              members=16, dtype="f32", t=0.1, seed=104, bytes_per_point=16 * 3 * 4 + 4 * 4),
}


def bumps(seed: int, count: int, extent, dims: int) -> np.ndarray:
    """(count, 5) float32: cx, cy, cz, amp, 1/width^2 (world units, h = 1)."""
    rng = np.random.default_rng(seed)
    c = rng.uniform(0.0, 1.0, (count, 3)) * np.asarray(list(extent) + [1.0] * (3 - len(extent)))
    if dims == 2:
        c[:, 2] = 0.0
    amp = rng.choice([-1.0, 1.0], count)
    width = rng.uniform(5.0, 15.0, count)
    return np.column_stack([c, amp, 1.0 / width**2]).astype(np.float32)


def _gen(bump_arr, dims, nx, ny, nzl, z0, seed, sig_lo, sig_hi, sigma_mode, members, out, mem,
         vortex=(0.0, 0.0, 0.0, 0.0), shear=0.0, device="cuda"):
    b = torch.from_numpy(bump_arr).to(device)
    ptrs = None
    if out is not None:
        import ctypes

        ptrs = (ctypes.c_void_p * len(out))(*[t.data_ptr() for t in out])
    _check(lib.divuq_gen_field_f32(
        b.data_ptr(), bump_arr.shape[0], dims, nx, ny, nzl, z0, 1.0, 1.0, 1.0, *vortex, shear,
        seed, sig_lo, sig_hi, sigma_mode, members, ptrs,
        None if mem is None else mem.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.current_stream().synchronize()


def config3_slab(z0: int, nzl: int, nx=512, ny=512, nz=512, seed=103, device="cuda"):
    """Six fp32 slab tensors (mu_u, mu_v, mu_w, s_u, s_v, s_w) of config 3."""
    n = nx * ny * nzl
    out = [torch.empty(n, dtype=torch.float32, device=device) for _ in range(6)]
    _gen(bumps(seed, 64, (nx - 1, ny - 1, nz - 1), 3), 3, nx, ny, nzl, z0, seed, 0.05, 0.3, 0,
         0, out, None, shear=1.0, device=device)
    return out


def config4_slab(z0: int, nzl: int, nx=1024, ny=1024, nz=1024, members=16, seed=104,
                 device="cuda"):
    """(M, 3, nx*ny*nzl) fp32 member slab of config 4 (206 GB in total at 1024^3)."""
    mem = torch.empty((members, 3, nx * ny * nzl), dtype=torch.float32, device=device)
    _gen(bumps(seed, 64, (nx - 1, ny - 1, nz - 1), 3), 3, nx, ny, nzl, z0, seed, 0.02, 0.5, 1,
         members, None, mem, shear=1.0, device=device)
    return mem


def config1_members(nx=1024, ny=1024, members=20, seed=101, device="cuda"):
    """(M, 2, nx*ny) fp32 ensemble of config 1 (24 sources/sinks + vortex,
    smooth sigma(x) in [0.02, 0.5])."""
    mem = torch.empty((members, 2, nx * ny), dtype=torch.float32, device=device)
    vortex = (1.0, 0.5 * (nx - 1), 0.5 * (ny - 1), 0.25 * min(nx, ny))
    _gen(bumps(seed, 24, (nx - 1, ny - 1), 2), 2, nx, ny, 1, 0, seed, 0.02, 0.5, 1, members, None,
         mem, vortex=vortex, device=device)
    return mem


def host_model2d(nx, ny, n_bumps, seed):
    """fp64 (mu_u, mu_v, s_u, s_v) numpy arrays: config-0-style model."""
    b = bumps(seed, n_bumps, (nx - 1, ny - 1), 2).astype(np.float64)
    j, i = np.divmod(np.arange(nx * ny), nx)
    x, y = i.astype(np.float64), j.astype(np.float64)
    u = np.zeros(nx * ny)
    v = np.zeros(nx * ny)
    for cx, cy, _, a, iw2 in b:
        g = a * np.exp(-((x - cx) ** 2 + (y - cy) ** 2) * iw2)
        u += (x - cx) * g
        v += (y - cy) * g
    cx, cy, r = 0.5 * (nx - 1), 0.5 * (ny - 1), 0.25 * min(nx, ny)
    g = np.exp(-((x - cx) ** 2 + (y - cy) ** 2) / r**2)
    u += -(y - cy) * g
    v += (x - cx) * g
    rng = np.random.default_rng(seed + 1)
    return u, v, rng.uniform(0.05, 0.3, nx * ny), rng.uniform(0.05, 0.3, nx * ny)


def config0_model():
    c = CONFIGS[0]
    return host_model2d(c.nx, c.ny, 6, c.seed)


def config2_model():
    c = CONFIGS[2]
    return host_model2d(c.nx, c.ny, 6, c.seed)
