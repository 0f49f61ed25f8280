"""Reference-compatible data types (drop-in for divuq.grid / divergence / gaussian / mc).

Same names, fields, validation and exceptions as the reference
(/root/reference/pkg/src/divuq):

* ``UniformGrid2``        grid.py:33-66
* ``ScalarField2``        grid.py:74-88
* ``VectorField2``        grid.py:91-102
* ``Ensemble2``           grid.py:105-123
* ``GaussianVectorField`` gaussian.py:14-32
* ``GaussianScalarField`` divergence.py:22-38
* ``McConfig``            mc.py:27-36
* ``McDivergenceEstimate``mc.py:39-53
* ``ParallelConfig``      parallel.py:19-41 (accepted for signature
  compatibility; the GPU path maps the whole index space in one launch and is
  bit-identical for every setting, which is the reference's own contract)

plus 3D twins (no reference code): ``UniformGrid3``,
``GaussianVectorField3``, ``GaussianScalarField3``.  The 3D types keep their
arrays' float dtype (float32 or float64) instead of forcing fp64, since the
3D configs are fp32.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np


def _frozen_array(values, n: int, name: str, dtype=np.float64) -> np.ndarray:
    """Validate and freeze a flat array of length n (grid.py:21-30)."""
    arr = np.ascontiguousarray(values, dtype=dtype)
    if arr.ndim != 1 or arr.size != n:
        raise ValueError(f"{name}: expected {n} values, got shape {arr.shape}")
    if not np.all(np.isfinite(arr)):
        raise ValueError(f"{name}: non-finite values are not allowed")
    arr = arr.copy()
    arr.flags.writeable = False
    return arr


def _float_dtype(values) -> np.dtype:
    dt = np.asarray(values).dtype
    return np.dtype(np.float32) if dt == np.float32 else np.dtype(np.float64)


@dataclass(frozen=True)
class UniformGrid2:
    """Uniform 2D grid: nx x ny vertices with spacing (dx, dy); index j*nx + i."""

    nx: int
    ny: int
    dx: float = 1.0
    dy: float = 1.0

    def __post_init__(self):
        if self.nx < 2 or self.ny < 2:
            raise ValueError(f"grid must be at least 2x2, got {self.nx}x{self.ny}")
        if not (self.dx > 0 and self.dy > 0):
            raise ValueError(f"grid spacing must be positive, got ({self.dx}, {self.dy})")

    @property
    def n_vertices(self) -> int:
        return self.nx * self.ny

    @property
    def n_cells(self) -> int:
        return (self.nx - 1) * (self.ny - 1)

    def vertex_index(self, i: int, j: int) -> int:
        if not (0 <= i < self.nx and 0 <= j < self.ny):
            raise IndexError(f"vertex ({i}, {j}) outside {self.nx}x{self.ny} grid")
        return j * self.nx + i

    def vertex_ij(self, index: int) -> tuple[int, int]:
        if not (0 <= index < self.n_vertices):
            raise IndexError(f"linear index {index} outside grid of {self.n_vertices} vertices")
        return index % self.nx, index // self.nx


def vertex_index(grid: UniformGrid2, i: int, j: int) -> int:
    return grid.vertex_index(i, j)


@dataclass(frozen=True)
class UniformGrid3:
    """Uniform 3D grid; flat index (k*ny + j)*nx + i (SPEC.md:79 extended)."""

    nx: int
    ny: int
    nz: int
    dx: float = 1.0
    dy: float = 1.0
    dz: float = 1.0

    def __post_init__(self):
        if self.nx < 2 or self.ny < 2 or self.nz < 2:
            raise ValueError(f"grid must be at least 2x2x2, got {self.nx}x{self.ny}x{self.nz}")
        if not (self.dx > 0 and self.dy > 0 and self.dz > 0):
            raise ValueError(f"grid spacing must be positive, got ({self.dx}, {self.dy}, {self.dz})")

    @property
    def n_vertices(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def plane(self) -> int:
        return self.nx * self.ny

    def vertex_index(self, i: int, j: int, k: int) -> int:
        if not (0 <= i < self.nx and 0 <= j < self.ny and 0 <= k < self.nz):
            raise IndexError(f"vertex ({i}, {j}, {k}) outside grid")
        return (k * self.ny + j) * self.nx + i


@dataclass(frozen=True)
class ScalarField2:
    grid: UniformGrid2
    values: np.ndarray = field(repr=False)

    def __post_init__(self):
        object.__setattr__(self, "values", _frozen_array(self.values, self.grid.n_vertices, "values"))

    def as_2d(self) -> np.ndarray:
        return self.values.reshape(self.grid.ny, self.grid.nx)


@dataclass(frozen=True)
class VectorField2:
    grid: UniformGrid2
    u: np.ndarray = field(repr=False)
    v: np.ndarray = field(repr=False)

    def __post_init__(self):
        n = self.grid.n_vertices
        object.__setattr__(self, "u", _frozen_array(self.u, n, "u"))
        object.__setattr__(self, "v", _frozen_array(self.v, n, "v"))


@dataclass(frozen=True)
class Ensemble2:
    """Ordered members on one grid (m >= 2).  ``stacked()`` is the (M, 2, N)
    member-major block the kernels read (io.py:51-53 layout)."""

    grid: UniformGrid2
    members: tuple

    def __post_init__(self):
        members = tuple(self.members)
        if len(members) < 2:
            raise ValueError(f"ensemble needs at least 2 members, got {len(members)}")
        for k, m in enumerate(members):
            if m.grid != self.grid:
                raise ValueError(f"member {k} grid {m.grid} differs from ensemble grid {self.grid}")
        object.__setattr__(self, "members", members)

    @property
    def n_members(self) -> int:
        return len(self.members)

    def stacked(self) -> np.ndarray:
        cached = self.__dict__.get("_stacked")
        if cached is None:
            cached = np.stack([np.stack([m.u, m.v]) for m in self.members])
            object.__setattr__(self, "_stacked", cached)
        return cached


@dataclass(frozen=True)
class GaussianVectorField:
    grid: UniformGrid2
    mu_u: np.ndarray = field(repr=False)
    mu_v: np.ndarray = field(repr=False)
    sigma_u: np.ndarray = field(repr=False)
    sigma_v: np.ndarray = field(repr=False)

    def __post_init__(self):
        n = self.grid.n_vertices
        for name in ("mu_u", "mu_v", "sigma_u", "sigma_v"):
            object.__setattr__(self, name, _frozen_array(getattr(self, name), n, name))
        if np.any(self.sigma_u < 0) or np.any(self.sigma_v < 0):
            raise ValueError("sigmas must be non-negative")

    def mean_field(self) -> VectorField2:
        return VectorField2(self.grid, self.mu_u, self.mu_v)


@dataclass(frozen=True)
class GaussianScalarField:
    grid: UniformGrid2
    mu: np.ndarray = field(repr=False)
    sigma: np.ndarray = field(repr=False)

    def __post_init__(self):
        n = self.grid.n_vertices
        object.__setattr__(self, "mu", _frozen_array(self.mu, n, "mu"))
        object.__setattr__(self, "sigma", _frozen_array(self.sigma, n, "sigma"))
        if np.any(self.sigma < 0):
            raise ValueError("sigma must be non-negative")

    def mean_field(self) -> ScalarField2:
        return ScalarField2(self.grid, self.mu)


@dataclass(frozen=True)
class LcpField:
    """Per-cell crossing probability, cell-major j*(nx-1) + i (lcp.py:26-45)."""

    grid: UniformGrid2
    isovalue: float
    probabilities: np.ndarray = field(repr=False)

    def __post_init__(self):
        object.__setattr__(self, "probabilities",
                           _frozen_array(self.probabilities, self.grid.n_cells, "probabilities"))
        p = self.probabilities
        if np.any(p < 0) or np.any(p > 1):
            raise ValueError("probabilities must lie in [0, 1]")

    def as_2d(self) -> np.ndarray:
        return self.probabilities.reshape(self.grid.ny - 1, self.grid.nx - 1)


@dataclass(frozen=True)
class GaussianVectorField3:
    """Independent N(mu, sigma^2) per vertex and component on a 3D grid."""

    grid: UniformGrid3
    mu_u: np.ndarray = field(repr=False)
    mu_v: np.ndarray = field(repr=False)
    mu_w: np.ndarray = field(repr=False)
    sigma_u: np.ndarray = field(repr=False)
    sigma_v: np.ndarray = field(repr=False)
    sigma_w: np.ndarray = field(repr=False)

    def __post_init__(self):
        n = self.grid.n_vertices
        dt = _float_dtype(self.mu_u)
        names = ("mu_u", "mu_v", "mu_w", "sigma_u", "sigma_v", "sigma_w")
        for name in names:
            object.__setattr__(self, name, _frozen_array(getattr(self, name), n, name, dt))
        if any(np.any(getattr(self, s) < 0) for s in names[3:]):
            raise ValueError("sigmas must be non-negative")

    @property
    def dtype(self) -> np.dtype:
        return self.mu_u.dtype


@dataclass(frozen=True)
class GaussianScalarField3:
    grid: UniformGrid3
    mu: np.ndarray = field(repr=False)
    sigma: np.ndarray = field(repr=False)

    def __post_init__(self):
        n = self.grid.n_vertices
        dt = _float_dtype(self.mu)
        object.__setattr__(self, "mu", _frozen_array(self.mu, n, "mu", dt))
        object.__setattr__(self, "sigma", _frozen_array(self.sigma, n, "sigma", dt))
        if np.any(self.sigma < 0):
            raise ValueError("sigma must be non-negative")


@dataclass(frozen=True)
class McConfig:
    n_samples: int
    seed: int = 0

    def __post_init__(self):
        if self.n_samples < 1:
            raise ValueError("n_samples must be >= 1")
        if not (0 <= self.seed < 2**64):
            raise ValueError("seed must fit in 64 unsigned bits")


@dataclass(frozen=True)
class McDivergenceEstimate:
    grid: UniformGrid2
    mean: np.ndarray = field(repr=False)
    std: np.ndarray = field(repr=False)
    n_samples: int = 0

    def __post_init__(self):
        n = self.grid.n_vertices
        object.__setattr__(self, "mean", _frozen_array(self.mean, n, "mean"))
        object.__setattr__(self, "std", _frozen_array(self.std, n, "std"))
        if self.n_samples < 2:
            raise ValueError("n_samples must be >= 2 when std is populated")


@dataclass(frozen=True)
class McHistogram:
    """mc.py:56-77: bin edges, counts, sample count (same invariants)."""

    bin_edges: np.ndarray
    counts: np.ndarray
    n_samples: int

    def __post_init__(self):
        edges = np.asarray(self.bin_edges, dtype=np.float64)
        counts = np.asarray(self.counts, dtype=np.int64)
        if edges.ndim != 1 or np.any(np.diff(edges) <= 0):
            raise ValueError("bin_edges must be strictly increasing")
        if counts.shape != (edges.size - 1,) or np.any(counts < 0):
            raise ValueError("counts must be non-negative with length len(edges)-1")
        if int(counts.sum()) != self.n_samples:
            raise ValueError("counts must sum to n_samples")
        object.__setattr__(self, "bin_edges", edges)
        object.__setattr__(self, "counts", counts)

    def normalized_density(self) -> np.ndarray:
        """counts scaled so the histogram integrates to 1."""
        return self.counts / (self.n_samples * np.diff(self.bin_edges))


@dataclass(frozen=True)
class ParallelConfig:
    """threads and chunk may be a positive int or 'auto' (parallel.py:19-41)."""

    threads: int | str = "auto"
    chunk: int | str = "auto"

    def __post_init__(self):
        for name in ("threads", "chunk"):
            v = getattr(self, name)
            if v != "auto" and (not isinstance(v, int) or v < 1):
                raise ValueError(f"{name} must be a positive integer or 'auto', got {v!r}")

    def resolve_threads(self) -> int:
        return (os.cpu_count() or 1) if self.threads == "auto" else self.threads

    def resolve_chunk(self, n: int, threads: int) -> int:
        """'auto': ceil(n / (4 * threads)) -- a few static chunks per thread."""
        return max(1, -(-n // (threads * 4))) if self.chunk == "auto" else self.chunk
