"""z-slab exchange through peer memory (CUDA IPC), on the GPU.

``SlabStep(exchange="p2p")``: every rank maps its neighbours' slabs once and
its kernels read the halo planes in place -- K2 in ONE launch, K3 with the
neighbours' edge-plane w moments reduced from their member planes over the
peer mapping.  Two (or three) processes share cuda:0 here (IPC mappings of the
same device are valid), each owning a z-slab; nothing waits on another
rank's kernels (inputs are static, published with a barrier), so this is safe
on one GPU.  The assembled slabs must equal the single-process whole-domain
GPU result BIT FOR BIT (the slab kernels are the same code either way).
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

NX, NY, NZ = 128, 40, 23   # nx multiple of 128: the TMA kernels run
M = 5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs():
    rng = np.random.default_rng(17)
    n = NX * NY * NZ
    f = [rng.normal(size=n).astype(np.float32) for _ in range(3)]
    f += [rng.uniform(0.05, 0.4, n).astype(np.float32) for _ in range(3)]
    mem = rng.normal(0, 1, (M, 3, n)).astype(np.float32)
    return f, mem


def _worker(rank, world, port, outdir):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import __graft_entry__

        __graft_entry__.build()
        from paper_2510_01190_b200 import shard

        f, mem = _inputs()
        plane = NX * NY
        step = shard.SlabStep(NX, NY, NZ, rank, world, exchange="p2p", device="cuda")
        z0, z1 = step.z0, step.z1
        fields = [torch.from_numpy(x[z0 * plane:z1 * plane].copy()).cuda() for x in f]
        out = {k: torch.empty(step.nzl * plane, device="cuda") for k in ("mu", "sigma", "p_src", "p_snk")}
        n2 = shard.propagate3d_step(step, fields, out, 1.0, 0.5, 2.0, 0.0, check=True,
                                    sync_inputs=True)
        torch.cuda.synchronize()
        res = {f"k2_{k}": v.cpu().numpy() for k, v in out.items()}

        step3 = shard.SlabStep(NX, NY, NZ, rank, world, n_arrays=3, exchange="p2p", device="cuda")
        members = torch.from_numpy(np.ascontiguousarray(mem[:, :, z0 * plane:z1 * plane])).cuda()
        out3 = {k: torch.empty(step.nzl * plane, device="cuda") for k in ("mu", "sigma", "p_src", "p_snk")}
        n3 = shard.ensemble3d_step(step3, members, out3, 1.0, 0.5, 2.0, 0.1, check=True,
                                   sync_inputs=True)
        torch.cuda.synchronize()
        res.update({f"k3_{k}": v.cpu().numpy() for k, v in out3.items()})
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), z0=z0, z1=z1, n2=n2, n3=n3, **res)
        dist.barrier()   # keep every mapping alive until all ranks are done reading
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_slabs_equal_whole_domain_bitwise(world, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    import __graft_entry__

    __graft_entry__.build()
    from paper_2510_01190_b200 import device as dev

    f, mem = _inputs()
    whole = dev.propagate3d(*[torch.from_numpy(x).cuda() for x in f], NX, NY, NZ, 1.0, 0.5, 2.0,
                            0.0, check=True)
    whole3 = dev.ensemble_divergence3d(torch.from_numpy(mem).cuda(), NX, NY, NZ, 1.0, 0.5, 2.0, 0.1,
                                       check=True)
    torch.cuda.synchronize()
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       start_method="spawn", join=True)
    plane = NX * NY
    covered = 0
    for r in range(world):
        d = np.load(tmp_path / f"rank{r}.npz")
        z0, z1 = int(d["z0"]), int(d["z1"])
        assert int(d["n2"]) == 1   # K2: one launch, halos read in place
        for k in ("mu", "sigma", "p_src", "p_snk"):
            assert np.array_equal(d[f"k2_{k}"], whole[k].cpu().numpy()[z0 * plane:z1 * plane]), (r, k)
            assert np.array_equal(d[f"k3_{k}"], whole3[k].cpu().numpy()[z0 * plane:z1 * plane]), (r, k)
        covered += z1 - z0
    assert covered == NZ
