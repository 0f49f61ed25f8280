"""Pinned host blocks for the drop-in layer's large arrays (api.py results,
types.py's frozen copies, the stacked ensemble): see OutputPool.

Pinning needs the CUDA library and a device; where registration fails (no
GPU) the pool switches itself off and every request is a plain np.empty.
"""

from __future__ import annotations

import sys

import numpy as np

from ._lib import lib


def _p(a):
    return a.__array_interface__["data"][0]


class OutputPool:
    """Page-locked host blocks for the drop-in layer's large arrays.

    A fresh ``np.empty`` result of megabytes is unpopulated memory: the copy
    that fills it page-faults every 4 KB (fit_gaussian 1024^2 x 20: 8.7 ms in
    the C entry with warm outputs, 17 ms with fresh ones).  Results of at
    least ``MIN_BYTES`` are instead views of pooled blocks that were pinned
    once (``divuq_host_register``): the host entries DMA -- or, for small
    calls, copy-kernel -- straight into them (from 256 KB: 500^2 results
    0.6 -> 0.5 ms, 724^2 2.0 -> 0.93 ms, tools/bounce_probe.py).  A block is reused only when no
    array refers to it any more (every result is a view whose ``.base`` is
    the block, so the block's reference count says whether one is alive).
    Pinned bytes are capped (``DIVUQ_OUT_POOL_MB``, default 512; 0 disables
    the pool): past the cap free blocks are released, then plain ``np.empty``
    is used.  Same values, shapes and dtypes either way.
    """

    MIN_BYTES = 256 << 10

    def __init__(self):
        import os
        import threading

        self._cap = int(os.environ.get("DIVUQ_OUT_POOL_MB", "512")) << 20
        self._min = int(os.environ.get("DIVUQ_OUT_POOL_MIN_KB", str(self.MIN_BYTES >> 10))) << 10
        self._blocks: list = []
        self._sentinel = [np.empty(1, np.uint8)]
        self._bytes = 0
        self._lock = threading.Lock()

    def empty(self, shape, dtype=np.float64):
        dt = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * dt.itemsize
        if self._cap <= 0 or nbytes < self._min or nbytes == 0:
            return np.empty(shape, dt)
        with self._lock:
            # a block nothing else refers to has the reference count of the
            # never-handed-out sentinel, measured the same way (no guess at
            # the interpreter's own references)
            idle = _refs(self._sentinel, 0)
            for i in range(len(self._blocks)):
                if self._blocks[i].nbytes == nbytes and _refs(self._blocks, i) == idle:
                    block = self._blocks.pop(i)    # most recently used last
                    self._blocks.append(block)
                    return block.view(dt).reshape(shape)
            i = 0
            while self._bytes + nbytes > self._cap and i < len(self._blocks):
                if _refs(self._blocks, i) == idle:
                    block = self._blocks.pop(i)
                    lib.divuq_host_unregister(_p(block))
                    self._bytes -= block.nbytes
                    del block
                else:
                    i += 1
            if self._bytes + nbytes > self._cap:
                return np.empty(shape, dt)
            block = np.empty(nbytes, np.uint8)
            if lib.divuq_host_register(_p(block), nbytes) != 0:
                self._cap = 0          # no pinning here (no device): plain arrays from now on
                return np.empty(shape, dt)
            self._blocks.append(block)
            self._bytes += nbytes
            return block.view(dt).reshape(shape)


def _refs(lst, i):
    """Reference count of lst[i] as seen from here (same for every list)."""
    for b in lst[i:i + 1]:
        return sys.getrefcount(b)


POOL = OutputPool()
empty = POOL.empty
