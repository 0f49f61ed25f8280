"""z-slab partitioning of 3D grids over the GPUs of one box (north star item 4).

One process per GPU (torch.distributed, backend "nccl" on B200s; "gloo" for
the CPU tests).  Rank r owns global planes [z0_r, z1_r) of every input array.
The only coupling between slabs is the w component along z, so the exchange
is ONE plane per neighbour per array:

* K2 (analytic, config 3): the raw (mu_w, s_w) edge planes;
* K3 (fused ensemble, config 4): the REDUCED w moments of the edge planes
  (2 planes instead of 2*M), computed by the owner with the same moment
  arithmetic, so sharded results are bit-identical to the 1-GPU run.

Schedule per step (``SlabStep.run``):
  1. post the neighbour sends/receives (``batch_isend_irecv``; NCCL runs them on
     its own stream over NVLink),
  2. launch the interior planes [1, nzl-1) on the compute stream -- they need
     no halo, so the exchange overlaps them,
  3. wait for the exchange, launch the two edge planes.
The x/y stencils never cross a slab, and the one-sided boundary rule is applied
only at the global faces z = 0 and z = nz-1.

The compute functions are injected (``compute``) so the orchestration -- slab
bounds, which planes travel where, the interior/edge split -- is testable
on CPU with gloo against the whole-domain oracle (tests/test_shard.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def slab_bounds(nz: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous z-slab of rank r: [r*nz//P, (r+1)*nz//P)."""
    if not (0 <= rank < world) or world < 1:
        raise ValueError("bad rank/world")
    if nz < 2 * world:
        raise ValueError(f"nz={nz} too small for {world} slabs (need >= 2 planes each)")
    return nz * rank // world, nz * (rank + 1) // world


@dataclass
class SlabStep:
    """One rank's share of a sharded 3D step.

    ``edge_planes(kind)`` returns the (first, last) planes to send (tuple of
    tensors each), ``compute(k_range, halo_lo, halo_hi)`` enqueues the kernel(s)
    for local planes [kb, ke).  Halo buffers are allocated once and reused.
    """

    nx: int
    ny: int
    nz_global: int
    rank: int
    world: int
    n_arrays: int = 2          # arrays per exchanged plane (mu_w, s_w)
    dtype: torch.dtype = torch.float32
    device: str | torch.device = "cuda"
    group: object = None

    def __post_init__(self):
        self.z0, self.z1 = slab_bounds(self.nz_global, self.world, self.rank)
        self.nzl = self.z1 - self.z0
        plane = self.nx * self.ny
        mk = lambda: tuple(torch.empty(plane, dtype=self.dtype, device=self.device)
                           for _ in range(self.n_arrays))
        self.halo_lo = mk() if self.rank > 0 else None
        self.halo_hi = mk() if self.rank < self.world - 1 else None
        self.launches = 0

    def _exchange_ops(self, first, last):
        ops = []
        lo, hi = self.rank - 1, self.rank + 1
        if self.rank > 0:
            for a in range(self.n_arrays):
                ops.append(dist.P2POp(dist.isend, first[a], lo, self.group))
                ops.append(dist.P2POp(dist.irecv, self.halo_lo[a], lo, self.group))
        if self.rank < self.world - 1:
            for a in range(self.n_arrays):
                ops.append(dist.P2POp(dist.isend, last[a], hi, self.group))
                ops.append(dist.P2POp(dist.irecv, self.halo_hi[a], hi, self.group))
        return ops

    def run(self, edge_planes, compute):
        """Exchange + overlapped interior + edges.  Returns #kernel launches."""
        launches = 0
        if self.world == 1:
            launches += compute((0, self.nzl), None, None)
            self.launches = launches
            return launches
        first, last = edge_planes()
        reqs = dist.batch_isend_irecv(self._exchange_ops(first, last))
        # interior planes need no halo: overlap them with the exchange
        if self.nzl > 2:
            launches += compute((1, self.nzl - 1), None, None)
        for r in reqs:
            r.wait()
        launches += compute((0, 1), self.halo_lo, self.halo_hi)
        launches += compute((self.nzl - 1, self.nzl), self.halo_lo, self.halo_hi)
        self.launches = launches
        return launches


def propagate3d_step(step: SlabStep, fields, out, dx, dy, dz, t, check=False):
    """K2 sharded step on this rank's slab tensors (fields = 6 slab tensors)."""
    from . import device as dev

    plane = step.nx * step.ny
    mu_w, s_w = fields[2], fields[5]

    def edges():
        return ((mu_w[:plane], s_w[:plane]), (mu_w[-plane:], s_w[-plane:]))

    def compute(k_range, lo, hi):
        dev.propagate3d(*fields, step.nx, step.ny, step.nzl, dx, dy, dz, t, z0=step.z0,
                        nz_global=step.nz_global, halo_lo=step.halo_lo, halo_hi=step.halo_hi,
                        k_range=k_range, out=out, check=check)
        return 1

    return step.run(edges, compute)


def ensemble3d_step(step: SlabStep, members, out, dx, dy, dz, t, check=False):
    """K3 sharded step: the owner reduces its edge planes' w moments, the
    neighbours receive 2 planes each instead of 2*M raw member planes."""
    from . import device as dev

    def edges():
        first = dev.w_moments_plane(members, step.nx, step.ny, step.nzl, 0, check=check)
        last = dev.w_moments_plane(members, step.nx, step.ny, step.nzl, step.nzl - 1, check=check)
        return first, last

    def compute(k_range, lo, hi):
        dev.ensemble_divergence3d(members, step.nx, step.ny, step.nzl, dx, dy, dz, t, z0=step.z0,
                                  nz_global=step.nz_global, halo_lo=step.halo_lo,
                                  halo_hi=step.halo_hi, k_range=k_range, out=out, check=check)
        return 1

    n = step.run(edges, compute)
    return n + (4 if step.world > 1 else 0)  # 2 gathers + 2 fits for the edge moments
