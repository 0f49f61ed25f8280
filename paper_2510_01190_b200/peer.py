"""Peer memory between the ranks of one box (CUDA IPC over NVLink / NVSwitch).

The z-slab exchange (``shard.SlabStep(exchange="p2p")``) does not copy halo
planes at all: every rank exports the allocations holding the arrays its
neighbours need, the neighbours map them once, and their kernels read the
halo planes straight out of the owner's HBM while they compute -- the transfer
happens inside the compute kernels, tile by tile, instead of in a separate
NCCL step.  Handles travel once, at setup, over the process group
(``all_gather_object``: gloo or NCCL).

Same-device mappings are valid too (two processes on one GPU), which is how
the parity tests exercise this path on a single B200.
"""

from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from ._lib import check as _check
from ._lib import lib

_HANDLE_BYTES = int(lib.divuq_ipc_handle_bytes())


def export_tensor(t: torch.Tensor) -> tuple[bytes, int, int]:
    """(IPC handle of t's allocation, t's byte offset in it, t's size in bytes)."""
    if not t.is_cuda:
        raise TypeError("export_tensor: expected a CUDA tensor")
    h = ctypes.create_string_buffer(_HANDLE_BYTES)
    off = ctypes.c_int64(0)
    _check(lib.divuq_ipc_export(ctypes.c_void_p(t.data_ptr()), h, ctypes.byref(off)))
    return h.raw, int(off.value), t.numel() * t.element_size()


class PeerArray:
    """A neighbour's exported array mapped into this process: ``ptr`` is a
    device address this rank's kernels can read (peer access over NVLink)."""

    def __init__(self, handle: bytes, offset: int, nbytes: int):
        base = ctypes.c_void_p(0)
        ptr = ctypes.c_void_p(0)
        _check(lib.divuq_ipc_import(handle, int(offset), ctypes.byref(base), ctypes.byref(ptr)))
        self._base = base
        self.ptr = int(ptr.value)
        self.nbytes = int(nbytes)

    def at(self, byte_offset: int) -> int:
        if not (0 <= byte_offset < self.nbytes):
            raise ValueError("offset outside the peer array")
        return self.ptr + byte_offset

    def close(self) -> None:
        if self._base is not None and self._base.value:
            lib.divuq_ipc_close(self._base)
        self._base = None


def exchange_handles(arrays: dict[str, torch.Tensor], rank: int, world: int, group=None,
                     want=None) -> dict[int, dict[str, PeerArray]]:
    """Export ``arrays``, all-gather every rank's handles, map the ranks in
    ``want`` (default: the z-neighbours rank-1 and rank+1).  Collective."""
    try:
        mine = {k: export_tensor(v) for k, v in arrays.items()}
    except Exception as exc:   # still join the collective, so no rank blocks in it
        mine = {"__error__": repr(exc)}
    allh = [None] * world
    dist.all_gather_object(allh, mine, group=group)
    bad = [r for r in range(world) if "__error__" in allh[r]]
    if bad:
        raise RuntimeError(f"peer export failed on rank(s) {bad}: {allh[bad[0]]['__error__']}")
    want = [r for r in (rank - 1, rank + 1) if 0 <= r < world] if want is None else want
    return {r: {k: PeerArray(*allh[r][k]) for k in allh[r]} for r in want}
