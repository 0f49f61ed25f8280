"""z-slab multi-GPU orchestration on CPU: gloo, world_size 2 and 3.

Each rank owns a contiguous z-slab, exchanges one plane of (mu_w, s_w) -- or
of the REDUCED w moments for the fused ensemble path -- with its neighbours
through ``shard.SlabStep`` (batch_isend_irecv), computes interior planes
before the exchange completes and the two edge planes after, exactly like the
GPU path.  The per-slab compute here is the CPU oracle (tests may use it);
the assembled result must equal the whole-domain oracle BIT FOR BIT.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ref2d, ref3d

NX, NY, NZ = 9, 7, 13
SPACING = (0.3, 0.7, 1.1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _fields(seed=5):
    rng = np.random.default_rng(seed)
    n = NX * NY * NZ
    return [rng.normal(size=n) for _ in range(3)] + [rng.uniform(0.1, 1.0, n) for _ in range(3)]


def _members(seed=6, m=5):
    rng = np.random.default_rng(seed)
    return rng.normal(0, 1, (m, 3, NX * NY * NZ))


def _worker(rank, world, port, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_01190_b200.shard import SlabStep

        plane = NX * NY
        step = SlabStep(NX, NY, NZ, rank, world, dtype=torch.float64, device="cpu")
        z0, z1 = step.z0, step.z1
        out_mu = np.full(step.nzl * plane, np.nan)
        out_sg = np.full(step.nzl * plane, np.nan)
        if mode == "analytic":
            f = _fields()
            sl = [x[z0 * plane:z1 * plane] for x in f]
            mu_w, s_w = torch.from_numpy(sl[2].copy()), torch.from_numpy(sl[5].copy())

            def edges():
                return ((mu_w[:plane], s_w[:plane]), (mu_w[-plane:], s_w[-plane:]))

            slab_fields = sl
        else:
            mem = _members()
            slab = mem[:, :, z0 * plane:z1 * plane]
            mu_r, sg_r = ref2d.fit_moments(slab)  # the owner's reduced moments

            def edges():
                first = (torch.from_numpy(mu_r[2][:plane].copy()), torch.from_numpy(sg_r[2][:plane].copy()))
                last = (torch.from_numpy(mu_r[2][-plane:].copy()), torch.from_numpy(sg_r[2][-plane:].copy()))
                return first, last

            slab_fields = list(mu_r) + list(sg_r)

        calls = []

        def compute(k_range, lo, hi):
            kb, ke = k_range
            calls.append((kb, ke))
            ghost_lo = None if step.halo_lo is None else tuple(t.numpy() for t in step.halo_lo)
            ghost_hi = None if step.halo_hi is None else tuple(t.numpy() for t in step.halo_hi)
            mu, sg = ref3d.propagate3d_slab(slab_fields, ghost_lo, ghost_hi, NX, NY, z0, NZ, *SPACING)
            out_mu[kb * plane:ke * plane] = mu[kb * plane:ke * plane]
            out_sg[kb * plane:ke * plane] = sg[kb * plane:ke * plane]
            return 1

        launches = step.run(edges, compute)
        q.put((rank, z0, z1, out_mu, out_sg, launches, calls))
    finally:
        dist.destroy_process_group()


def _run(world, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda r: r[0])


@pytest.mark.parametrize("world", [2, 3])
def test_analytic_slabs_over_gloo_equal_whole_domain_bitwise(world):
    f = _fields()
    mu, sg = ref3d.propagate3d(*f, NX, NY, NZ, *SPACING)
    plane = NX * NY
    res = _run(world, "analytic")
    covered = 0
    for rank, z0, z1, omu, osg, launches, calls in res:
        assert np.array_equal(omu, mu[z0 * plane:z1 * plane]), rank
        assert np.array_equal(osg, sg[z0 * plane:z1 * plane]), rank
        # interior first (overlapping the exchange), then the two edge planes
        nzl = z1 - z0
        assert calls == [(1, nzl - 1), (0, 1), (nzl - 1, nzl)] and launches == 3
        covered += nzl
    assert covered == NZ


def test_ensemble_slabs_exchange_reduced_moments_bitwise():
    mem = _members()
    mu_r, sg_r = ref2d.fit_moments(mem)
    mu, sg = ref3d.propagate3d(*mu_r, *sg_r, NX, NY, NZ, *SPACING)
    plane = NX * NY
    for _, z0, z1, omu, osg, _, _ in _run(2, "ensemble"):
        assert np.array_equal(omu, mu[z0 * plane:z1 * plane])
        assert np.array_equal(osg, sg[z0 * plane:z1 * plane])


def test_slab_bounds():
    from paper_2510_01190_b200.shard import slab_bounds

    assert [slab_bounds(512, 8, r) for r in (0, 7)] == [(0, 64), (448, 512)]
    b = [slab_bounds(13, 3, r) for r in range(3)]
    assert b == [(0, 4), (4, 8), (8, 13)]
    with pytest.raises(ValueError):
        slab_bounds(3, 2, 0)


def test_exchange_modes_and_neighbour_extents():
    from paper_2510_01190_b200.shard import SlabStep

    with pytest.raises(ValueError):
        SlabStep(4, 4, 8, 0, 2, device="cpu", exchange="mpi")
    s = SlabStep(4, 4, 13, 1, 3, device="cpu", exchange="p2p")
    assert (s.z0, s.z1) == (4, 8)
    assert [s.neighbour_nzl(r) for r in range(3)] == [4, 4, 5]
    # the halo planes a p2p rank reads in place: the last plane of rank-1 and
    # the first plane of rank+1 (byte offsets into their slabs)
    plane, es = 16, 4
    assert (s.neighbour_nzl(0) - 1) * plane * es == 192


def _fallback_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_01190_b200 import shard

        step = shard.SlabStep(NX, NY, NZ, rank, world, dtype=torch.float64, device="cpu", exchange="p2p")
        plane = NX * NY
        w = torch.zeros(step.nzl * plane, dtype=torch.float64)
        used = shard.ensure_p2p(step, {"mu_w": w, "s_w": w.clone()})   # host memory: no IPC handle
        q.put((rank, used, step.exchange, step.peers))
    finally:
        dist.destroy_process_group()


def test_p2p_mapping_failure_falls_back_to_nccl_on_every_rank():
    """bench.py calls shard.ensure_p2p before timing: if any rank cannot map
    its neighbours' buffers, all ranks agree (one all-reduce) and run the NCCL
    schedule instead -- nobody is left blocked in the handle all-gather."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fallback_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(2)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [(r[1], r[2], r[3]) for r in res] == [(False, "nccl", {})] * 2
