"""Reference-compatible data types (drop-in for divuq.grid / divergence / gaussian / mc).

Same names, fields, validation and exception texts as the reference
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

Implementation: the dataclass declarations are the contract; validation goes
through the shared helpers below (one freezing rule for every array field,
one sigma rule, the reference's messages kept verbatim in ``_MSG``).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

# the reference's exception texts (grid.py, gaussian.py, divergence.py, mc.py, parallel.py)
_MSG = {
    "len": "{name}: expected {n} values, got shape {shape}",
    "finite": "{name}: non-finite values are not allowed",
    "grid2": "grid must be at least 2x2, got {}x{}",
    "grid3": "grid must be at least 2x2x2, got {}x{}x{}",
    "spacing": "grid spacing must be positive, got ({})",
    "vertex2": "vertex ({}, {}) outside {}x{} grid",
    "vertex3": "vertex ({}, {}, {}) outside grid",
    "linear": "linear index {} outside grid of {} vertices",
    "members": "ensemble needs at least 2 members, got {}",
    "member_grid": "member {} grid {} differs from ensemble grid {}",
    "sigmas": "sigmas must be non-negative",
    "sigma": "sigma must be non-negative",
    "probs": "probabilities must lie in [0, 1]",
    "n_samples": "n_samples must be >= 1",
    "seed": "seed must fit in 64 unsigned bits",
    "n_samples_std": "n_samples must be >= 2 when std is populated",
    "edges": "bin_edges must be strictly increasing",
    "counts": "counts must be non-negative with length len(edges)-1",
    "counts_sum": "counts must sum to n_samples",
    "auto": "{name} must be a positive integer or 'auto', got {value!r}",
}


def _frozen_array(values, n: int, name: str, dtype=np.float64, pinned: bool = False) -> np.ndarray:
    """A validated, read-only flat copy of length n (grid.py:21-30's rule);
    ``pinned``: the copy goes to a pooled pinned block when large."""
    out = np.ascontiguousarray(values, dtype=dtype)
    if out.ndim != 1 or out.size != n:
        raise ValueError(_MSG["len"].format(name=name, n=n, shape=out.shape))
    if not np.isfinite(out).all():
        raise ValueError(_MSG["finite"].format(name=name))
    out = _pinned_copy(out) if pinned else out.copy()
    out.flags.writeable = False
    return out


def _pinned_copy(a: np.ndarray) -> np.ndarray:
    """The constructor's defensive copy, made into a pooled pinned block when
    it is large (_pool.py): the host entries then DMA the model straight from
    it on every call instead of staging it through host memory again."""
    from . import _pool

    out = _pool.empty(a.shape, a.dtype)
    np.copyto(out, a)
    return out


def _float_dtype(values) -> np.dtype:
    return np.dtype(np.float32) if np.asarray(values).dtype == np.float32 else np.dtype(np.float64)


def _freeze(obj, n: int, names, dtype=np.float64, pinned: bool = False) -> None:
    """Replace each named array field of a frozen dataclass by its frozen copy
    (``pinned``: for the models the host entries read on every call)."""
    for name in names:
        object.__setattr__(obj, name, _frozen_array(getattr(obj, name), n, name, dtype, pinned))


def _require_nonneg(obj, names, key: str) -> None:
    if any((getattr(obj, name) < 0).any() for name in names):
        raise ValueError(_MSG[key])


# Output records of this package's own kernels (api.py): the arrays are fresh,
# owned by the call and never handed out elsewhere, so the constructor's
# defensive copy is skipped and its scans become reductions -- a finite a.a
# (BLAS dot) proves every value finite, a min >= 0 (NaN fails it) proves sigma >= 0, a
# min/max inside [0, 1] proves probabilities.  When a reduction cannot prove
# the rule (a NaN, or a dot that overflows on finite values) the record goes
# through its constructor, which raises the reference's exact error, in the
# reference's order, or accepts the values.  1024^2 fp64 (mu, sigma): ~7 ms
# of scans, copies and page faults -> ~1 ms.
_ADOPT = os.environ.get("DIVUQ_ADOPT", "1") != "0"   # 0: always the constructor (A/B)
_ADOPT_RULES = {   # class name -> {array field: rule}
    "ScalarField2": {"values": "finite"},
    "VectorField2": {"u": "finite", "v": "finite"},
    "GaussianVectorField": {"mu_u": "finite", "mu_v": "finite", "sigma_u": "sigma", "sigma_v": "sigma"},
    "GaussianScalarField": {"mu": "finite", "sigma": "sigma"},
    "GaussianVectorField3": {"mu_u": "finite", "mu_v": "finite", "mu_w": "finite",
                             "sigma_u": "sigma", "sigma_v": "sigma", "sigma_w": "sigma"},
    "GaussianScalarField3": {"mu": "finite", "sigma": "sigma"},
    "LcpField": {"probabilities": "prob"},
    "McDivergenceEstimate": {"mean": "finite", "std": "finite"},
}


_ADOPT_PLANS: dict = {}
_F64 = np.dtype(np.float64)
_DOT, _MIN, _MAX = np.dot, np.minimum.reduce, np.maximum.reduce


def _adopt_plan(cls):
    names = tuple(cls.__dataclass_fields__)
    rules = _ADOPT_RULES[cls.__name__]
    checks = tuple((names.index(k), {"finite": 0, "sigma": 1, "prob": 2}[r]) for k, r in rules.items())
    plan = (len(names), checks, "n_cells" if cls.__name__ == "LcpField" else "n_vertices",
            cls.__name__.endswith("3"), names)
    _ADOPT_PLANS[cls] = plan
    return plan


def adopt(cls, *args):
    """``cls(*args)`` for records built from freshly computed, call-owned
    arrays (no copy; same validation, see above)."""
    plan = _ADOPT_PLANS.get(cls) or _adopt_plan(cls)
    n_fields, checks, n_attr, keeps_dtype, names = plan
    if not _ADOPT or len(args) != n_fields:
        return cls(*args)
    n = getattr(args[0], n_attr)
    dt = _float_dtype(args[checks[0][0]]) if keeps_dtype else _F64
    for i, rule in checks:
        a = args[i]
        if (type(a) is not np.ndarray or a.dtype != dt or a.ndim != 1 or a.size != n
                or not a.flags.c_contiguous):
            return cls(*args)
        if not math.isfinite(_DOT(a, a)):   # NaN / inf -> non-finite; |a| > 1e154 -> constructor
            return cls(*args)
        if rule and not _MIN(a) >= 0:
            return cls(*args)
        if rule == 2 and not _MAX(a) <= 1:
            return cls(*args)
    if cls is McDivergenceEstimate and args[3] < 2:
        return cls(*args)
    obj = object.__new__(cls)
    for k, v in zip(names, args):
        object.__setattr__(obj, k, v)
    for i, _ in checks:
        args[i].flags.writeable = False
    return obj


def _check_grid(dims, spacing, key: str) -> None:
    if min(dims) < 2:
        raise ValueError(_MSG[key].format(*dims))
    if not all(h > 0 for h in spacing):
        raise ValueError(_MSG["spacing"].format(", ".join(str(h) for h in spacing)))


@dataclass(frozen=True)
class UniformGrid2:
    """Uniform 2D grid: nx x ny vertices with spacing (dx, dy); index j*nx + i."""

    nx: int
    ny: int
    dx: float = 1.0
    dy: float = 1.0

    def __post_init__(self):
        _check_grid((self.nx, self.ny), (self.dx, self.dy), "grid2")

    @property
    def n_vertices(self) -> int:
        return self.nx * self.ny

    @property
    def n_cells(self) -> int:
        return (self.nx - 1) * (self.ny - 1)

    def vertex_index(self, i: int, j: int) -> int:
        if i < 0 or j < 0 or i >= self.nx or j >= self.ny:
            raise IndexError(_MSG["vertex2"].format(i, j, self.nx, self.ny))
        return i + self.nx * j

    def vertex_ij(self, index: int) -> tuple[int, int]:
        if index < 0 or index >= self.n_vertices:
            raise IndexError(_MSG["linear"].format(index, self.n_vertices))
        j, i = divmod(index, self.nx)
        return i, j


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
        _check_grid((self.nx, self.ny, self.nz), (self.dx, self.dy, self.dz), "grid3")

    @property
    def n_vertices(self) -> int:
        return self.plane * self.nz

    @property
    def plane(self) -> int:
        return self.nx * self.ny

    def vertex_index(self, i: int, j: int, k: int) -> int:
        if not all(0 <= c < d for c, d in ((i, self.nx), (j, self.ny), (k, self.nz))):
            raise IndexError(_MSG["vertex3"].format(i, j, k))
        return i + self.nx * (j + self.ny * k)


@dataclass(frozen=True)
class ScalarField2:
    grid: UniformGrid2
    values: np.ndarray = field(repr=False)

    def __post_init__(self):
        _freeze(self, self.grid.n_vertices, ("values",))

    def as_2d(self) -> np.ndarray:
        return self.values.reshape(self.grid.ny, self.grid.nx)


@dataclass(frozen=True)
class VectorField2:
    grid: UniformGrid2
    u: np.ndarray = field(repr=False)
    v: np.ndarray = field(repr=False)

    def __post_init__(self):
        _freeze(self, self.grid.n_vertices, ("u", "v"))


@dataclass(frozen=True)
class Ensemble2:
    """Ordered members on one grid (m >= 2).  ``stacked()`` is the (M, 2, N)
    member-major block the kernels read (io.py:51-53 layout)."""

    grid: UniformGrid2
    members: tuple

    def __post_init__(self):
        ms = tuple(self.members)
        if len(ms) < 2:
            raise ValueError(_MSG["members"].format(len(ms)))
        bad = next((k for k, m in enumerate(ms) if m.grid != self.grid), None)
        if bad is not None:
            raise ValueError(_MSG["member_grid"].format(bad, ms[bad].grid, self.grid))
        object.__setattr__(self, "members", ms)

    @property
    def n_members(self) -> int:
        return len(self.members)

    def stacked(self) -> np.ndarray:
        block = self.__dict__.get("_stacked")
        if block is None:
            from . import _pool   # pinned when large: fit_gaussian DMAs it directly

            block = _pool.empty((len(self.members), 2, self.grid.n_vertices))
            for k, m in enumerate(self.members):
                block[k, 0], block[k, 1] = m.u, m.v
            object.__setattr__(self, "_stacked", block)
        return block


@dataclass(frozen=True)
class GaussianVectorField:
    grid: UniformGrid2
    mu_u: np.ndarray = field(repr=False)
    mu_v: np.ndarray = field(repr=False)
    sigma_u: np.ndarray = field(repr=False)
    sigma_v: np.ndarray = field(repr=False)

    def __post_init__(self):
        _freeze(self, self.grid.n_vertices, ("mu_u", "mu_v", "sigma_u", "sigma_v"), pinned=True)
        _require_nonneg(self, ("sigma_u", "sigma_v"), "sigmas")

    def mean_field(self) -> VectorField2:
        return VectorField2(self.grid, self.mu_u, self.mu_v)


@dataclass(frozen=True)
class GaussianScalarField:
    grid: UniformGrid2
    mu: np.ndarray = field(repr=False)
    sigma: np.ndarray = field(repr=False)

    def __post_init__(self):
        _freeze(self, self.grid.n_vertices, ("mu", "sigma"), pinned=True)
        _require_nonneg(self, ("sigma",), "sigma")

    def mean_field(self) -> ScalarField2:
        return ScalarField2(self.grid, self.mu)


@dataclass(frozen=True)
class LcpField:
    """Per-cell crossing probability, cell-major j*(nx-1) + i (lcp.py:26-45)."""

    grid: UniformGrid2
    isovalue: float
    probabilities: np.ndarray = field(repr=False)

    def __post_init__(self):
        _freeze(self, self.grid.n_cells, ("probabilities",))
        p = self.probabilities
        if (p < 0).any() or (p > 1).any():
            raise ValueError(_MSG["probs"])

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
        sig = ("sigma_u", "sigma_v", "sigma_w")
        _freeze(self, self.grid.n_vertices, ("mu_u", "mu_v", "mu_w") + sig, _float_dtype(self.mu_u), True)
        _require_nonneg(self, sig, "sigmas")

    @property
    def dtype(self) -> np.dtype:
        return self.mu_u.dtype


@dataclass(frozen=True)
class GaussianScalarField3:
    grid: UniformGrid3
    mu: np.ndarray = field(repr=False)
    sigma: np.ndarray = field(repr=False)

    def __post_init__(self):
        _freeze(self, self.grid.n_vertices, ("mu", "sigma"), _float_dtype(self.mu), True)
        _require_nonneg(self, ("sigma",), "sigma")


@dataclass(frozen=True)
class McConfig:
    n_samples: int
    seed: int = 0

    def __post_init__(self):
        if not self.n_samples >= 1:
            raise ValueError(_MSG["n_samples"])
        if not 0 <= self.seed < (1 << 64):
            raise ValueError(_MSG["seed"])


@dataclass(frozen=True)
class McDivergenceEstimate:
    grid: UniformGrid2
    mean: np.ndarray = field(repr=False)
    std: np.ndarray = field(repr=False)
    n_samples: int = 0

    def __post_init__(self):
        _freeze(self, self.grid.n_vertices, ("mean", "std"))
        if self.n_samples < 2:
            raise ValueError(_MSG["n_samples_std"])


@dataclass(frozen=True)
class McHistogram:
    """mc.py:56-77: bin edges, counts, sample count (same invariants)."""

    bin_edges: np.ndarray
    counts: np.ndarray
    n_samples: int

    def __post_init__(self):
        e = np.asarray(self.bin_edges, dtype=np.float64)
        c = np.asarray(self.counts, dtype=np.int64)
        if e.ndim != 1 or (np.diff(e) <= 0).any():
            raise ValueError(_MSG["edges"])
        if c.shape != (e.size - 1,) or (c < 0).any():
            raise ValueError(_MSG["counts"])
        if int(c.sum()) != self.n_samples:
            raise ValueError(_MSG["counts_sum"])
        object.__setattr__(self, "bin_edges", e)
        object.__setattr__(self, "counts", c)

    def normalized_density(self) -> np.ndarray:
        """counts scaled so the histogram integrates to 1."""
        return self.counts / (self.n_samples * np.diff(self.bin_edges))


@dataclass(frozen=True)
class ParallelConfig:
    """threads and chunk may be a positive int or 'auto' (parallel.py:19-41)."""

    threads: int | str = "auto"
    chunk: int | str = "auto"

    def __post_init__(self):
        for name, value in (("threads", self.threads), ("chunk", self.chunk)):
            if value == "auto":
                continue
            if not isinstance(value, int) or value < 1:
                raise ValueError(_MSG["auto"].format(name=name, value=value))

    def resolve_threads(self) -> int:
        return self.threads if self.threads != "auto" else (os.cpu_count() or 1)

    def resolve_chunk(self, n: int, threads: int) -> int:
        """'auto': ceil(n / (4 * threads)) -- a few static chunks per thread."""
        if self.chunk != "auto":
            return self.chunk
        return max(1, (n + 4 * threads - 1) // (4 * threads))
