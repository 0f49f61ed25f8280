"""z-slab partitioning of 3D grids over the GPUs of one box (north star item 4).

One process per GPU (torch.distributed, backend "nccl" on B200s; "gloo" for
the CPU tests).  Rank r owns global planes [z0_r, z1_r) of every input array.
The only coupling between slabs is the w component along z, so the exchange
is ONE plane per neighbour per array:

* K2 (analytic, config 3): the raw (mu_w, s_w) edge planes;
* K3 (fused ensemble, config 4): the REDUCED w moments of the edge planes
  (3 planes -- mu, sigma and the means' rounding residual r -- instead of
  2*M), computed by the owner with the same moment arithmetic, so sharded
  results are bit-identical to the 1-GPU run.

Two exchange modes (``SlabStep(exchange=...)``):

* ``"p2p"`` (default on GPUs): no exchange step at all.  Each rank maps its
  z-neighbours' slabs once through CUDA IPC (peer.py) and its kernels read the
  halo planes straight from the neighbour's HBM over NVLink while they
  compute: K2 is ONE launch over the whole slab with the halo pointers aimed
  at the neighbours' edge planes; K3 reduces the neighbours' edge-plane w
  moments with a strided K1 reading their member planes in place (side
  stream), overlapped with the interior planes, then the two edge planes.
  Inputs are read in place, so the p2p step is fenced on both sides by
  default: ``sync_inputs=True`` drains every rank's producers before the
  first peer read, and the closing fence (stream sync + barrier) keeps a
  neighbour from rewriting or freeing its slab while this rank still reads
  it.  Re-mapping after a buffer moved is a collective decision (every rank
  learns whether ANY rank's buffers changed), so no rank skips the handle
  exchange another rank enters.
* ``"nccl"``: the classic schedule (``SlabStep.run``) --
  1. post the neighbour sends/receives (``batch_isend_irecv``; NCCL runs them
     on its own stream over NVLink),
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
    n_arrays: int = 2          # arrays per exchanged plane: K2 (mu_w, s_w); K3 3 (mu_w, s_w, r_w)
    dtype: torch.dtype = torch.float32
    device: str | torch.device = "cuda"
    group: object = None
    exchange: str = "nccl"     # "nccl" | "p2p" (peer memory, see module docstring)

    def __post_init__(self):
        if self.exchange not in ("nccl", "p2p"):
            raise ValueError("exchange must be 'nccl' or 'p2p'")
        self.peers = None
        self._attached = None
        self._side = None
        self.z0, self.z1 = slab_bounds(self.nz_global, self.world, self.rank)
        self.nzl = self.z1 - self.z0
        plane = self.nx * self.ny
        mk = lambda: tuple(torch.empty(plane, dtype=self.dtype, device=self.device)
                           for _ in range(self.n_arrays))
        self.halo_lo = mk() if self.rank > 0 else None
        self.halo_hi = mk() if self.rank < self.world - 1 else None
        self.launches = 0

    def neighbour_nzl(self, r: int) -> int:
        z0, z1 = slab_bounds(self.nz_global, self.world, r)
        return z1 - z0

    def attach(self, arrays: dict) -> None:
        """p2p: export ``arrays`` and map the neighbours' (collective).  Every
        rank calls it every step; the handles are re-exchanged when ANY rank's
        buffers moved (one all-reduced flag), so all ranks agree on entering
        the handle all-gather and nobody keeps a stale mapping."""
        from . import peer

        key = tuple((k, v.data_ptr()) for k, v in sorted(arrays.items()))
        if self.world > 1:
            dev = self.device if dist.get_backend(self.group) == "nccl" else "cpu"
            changed = torch.tensor([int(self._attached != key)], dtype=torch.int32, device=dev)
            dist.all_reduce(changed, op=dist.ReduceOp.MAX, group=self.group)
            if int(changed.item()) == 0:
                return
        elif self._attached == key:
            return
        if self.peers:
            for arrs in self.peers.values():
                for a in arrs.values():
                    a.close()
        self.peers = peer.exchange_handles(arrays, self.rank, self.world, self.group)
        self._attached = key

    def side_stream(self):
        if self._side is None:
            self._side = torch.cuda.Stream(device=self.device)
        return self._side

    def _exchange_ops(self, first, last, halo_lo, halo_hi):
        ops = []
        lo, hi = self.rank - 1, self.rank + 1
        if self.rank > 0:
            for a in range(self.n_arrays):
                ops.append(dist.P2POp(dist.isend, first[a], lo, self.group))
                ops.append(dist.P2POp(dist.irecv, halo_lo[a], lo, self.group))
        if self.rank < self.world - 1:
            for a in range(self.n_arrays):
                ops.append(dist.P2POp(dist.isend, last[a], hi, self.group))
                ops.append(dist.P2POp(dist.irecv, halo_hi[a], hi, self.group))
        return ops

    def run(self, edge_planes, compute):
        """Exchange + overlapped interior + edges.  Returns #kernel launches."""
        launches = 0
        if self.world == 1:
            launches += compute((0, self.nzl), None, None)
            self.launches = launches
            return launches
        first, last = edge_planes()
        # gloo cannot move CUDA tensors (the one-device dry runs of bench.py and
        # the tests): stage the edge and halo planes through host memory there
        staged = (dist.get_backend(self.group) == "gloo" and first is not None
                  and len(first) and first[0].is_cuda)
        hlo, hhi = self.halo_lo, self.halo_hi
        if staged:
            first = tuple(x.cpu() for x in first)
            last = tuple(x.cpu() for x in last)
            hlo = tuple(torch.empty_like(x, device="cpu") for x in hlo) if hlo else None
            hhi = tuple(torch.empty_like(x, device="cpu") for x in hhi) if hhi else None
        reqs = dist.batch_isend_irecv(self._exchange_ops(first, last, hlo, hhi))
        # interior planes need no halo: overlap them with the exchange
        if self.nzl > 2:
            launches += compute((1, self.nzl - 1), None, None)
        for r in reqs:
            r.wait()
        if staged:
            for dst, src in ((self.halo_lo, hlo), (self.halo_hi, hhi)):
                for d, s_ in zip(dst or (), src or ()):
                    d.copy_(s_)
        launches += compute((0, 1), self.halo_lo, self.halo_hi)
        launches += compute((self.nzl - 1, self.nzl), self.halo_lo, self.halo_hi)
        self.launches = launches
        return launches


def _sync_inputs(step: SlabStep):
    torch.cuda.current_stream().synchronize()
    dist.barrier(group=step.group)


def _fence(step: SlabStep):
    """Closing fence of a p2p step: this rank's peer reads are complete before
    any neighbour may rewrite or free the slab they read."""
    torch.cuda.current_stream().synchronize()
    dist.barrier(group=step.group)


def ensure_p2p(step: SlabStep, arrays: dict) -> bool:
    """Collective: map the neighbours' ``arrays`` for the p2p exchange; if any
    rank cannot (no peer access, IPC refused), every rank switches this step
    to the NCCL schedule instead.  Returns whether p2p is in use."""
    if step.exchange != "p2p" or step.world == 1:
        return step.exchange == "p2p"
    ok = 1
    try:
        step.attach(arrays)
    except Exception:   # export failures are raised on every rank alike
        ok = 0
    flag = torch.tensor([ok], dtype=torch.int32, device=step.device if dist.get_backend(step.group) == "nccl"
                        else "cpu")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=step.group)
    if int(flag.item()) == 1:
        return True
    for arrs in (step.peers or {}).values():
        for a in arrs.values():
            a.close()
    step.peers, step._attached, step.exchange = {}, None, "nccl"
    return False


def propagate3d_step(step: SlabStep, fields, out, dx, dy, dz, t, check=False, sync_inputs=True,
                     fence=True, remap=True):
    """K2 sharded step on this rank's slab tensors (fields = 6 slab tensors).

    p2p safety defaults: ``remap`` (collective re-attach check), ``sync_inputs``
    and ``fence`` (see the module docstring).  A caller whose slabs are neither
    moved nor rewritten between steps (bench.py's timed loop, after one
    ``ensure_p2p`` and one barrier) may pass all three False: the step is then
    one kernel launch with no collective."""
    from . import device as dev

    plane = step.nx * step.ny
    mu_w, s_w = fields[2], fields[5]
    if step.exchange == "p2p" and step.world > 1:
        # ONE launch: the halo planes are read from the neighbours' HBM in place
        if remap:
            step.attach({"mu_w": mu_w, "s_w": s_w})
        if sync_inputs:
            _sync_inputs(step)
        es = mu_w.element_size()
        lo = hi = None
        if step.rank > 0:
            nb, off = step.peers[step.rank - 1], (step.neighbour_nzl(step.rank - 1) - 1) * plane * es
            lo = (nb["mu_w"].at(off), nb["s_w"].at(off))
        if step.rank < step.world - 1:
            nb = step.peers[step.rank + 1]
            hi = (nb["mu_w"].at(0), nb["s_w"].at(0))
        dev.propagate3d(*fields, step.nx, step.ny, step.nzl, dx, dy, dz, t, z0=step.z0,
                        nz_global=step.nz_global, halo_lo=lo, halo_hi=hi, out=out, check=check)
        if fence:
            _fence(step)
        step.launches = 1
        return 1

    def edges():
        return ((mu_w[:plane], s_w[:plane]), (mu_w[-plane:], s_w[-plane:]))

    def compute(k_range, lo, hi):
        dev.propagate3d(*fields, step.nx, step.ny, step.nzl, dx, dy, dz, t, z0=step.z0,
                        nz_global=step.nz_global, halo_lo=step.halo_lo, halo_hi=step.halo_hi,
                        k_range=k_range, out=out, check=check)
        return 1

    return step.run(edges, compute)


def ensemble3d_step(step: SlabStep, members, out, dx, dy, dz, t, check=False, sync_inputs=True,
                    fence=True, remap=True):
    """K3 sharded step.  nccl: the owner reduces its edge planes' w moments and
    the neighbours receive 2 planes each instead of 2*M raw member planes.
    p2p: each rank reduces its neighbours' edge planes itself, reading their
    member planes in place over NVLink on a side stream, overlapped with its
    interior planes."""
    from . import device as dev

    if step.world > 1 and step.n_arrays != 3:
        raise ValueError("ensemble3d_step exchanges (mu_w, s_w, r_w): build the SlabStep with n_arrays=3")
    if step.exchange == "p2p" and step.world > 1:
        if remap:
            step.attach({"members": members})
        if sync_inputs:
            _sync_inputs(step)
        m = members.shape[0]
        main = torch.cuda.current_stream()
        side = step.side_stream()
        side.wait_stream(main)
        with torch.cuda.stream(side):   # neighbours' edge-plane moments, read over NVLink
            if step.rank > 0:
                r = step.rank - 1
                dev.w_moments_plane_ptr(step.peers[r]["members"].ptr, m, step.nx, step.ny,
                                        step.neighbour_nzl(r), step.neighbour_nzl(r) - 1,
                                        device=members.device, out=step.halo_lo, check=check)
            if step.rank < step.world - 1:
                r = step.rank + 1
                dev.w_moments_plane_ptr(step.peers[r]["members"].ptr, m, step.nx, step.ny,
                                        step.neighbour_nzl(r), 0, device=members.device,
                                        out=step.halo_hi, check=check)
        n = 2
        # the interior planes never read the halo buffers (still being filled)
        common = dict(z0=step.z0, nz_global=step.nz_global, halo_lo=step.halo_lo,
                      halo_hi=step.halo_hi, out=out, check=check)
        if step.nzl > 2:   # interior: overlaps the peer reads
            dev.ensemble_divergence3d(members, step.nx, step.ny, step.nzl, dx, dy, dz, t,
                                      k_range=(1, step.nzl - 1), **common)
            n += 1
        main.wait_stream(side)
        for kr in ((0, 1), (step.nzl - 1, step.nzl)):
            dev.ensemble_divergence3d(members, step.nx, step.ny, step.nzl, dx, dy, dz, t,
                                      k_range=kr, **common)
        n += 2
        if fence:
            _fence(step)
        step.launches = n
        return n

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
    return n + (2 if step.world > 1 else 0)  # 2 strided fits for the edge moments
