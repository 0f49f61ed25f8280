"""``parallel_map`` / ``bench`` / ``BenchReport`` -- the reference's seam, kept
for drop-in callers (parallel.py:19-129 of the reference).

The hot-path functions of this package never go through ``parallel_map``: each
is one sm_100a kernel launch over the whole index space.  The
map is kept for callers that map their OWN per-index Python kernels, with the
reference's contract: static contiguous chunks (``ParallelConfig``: 'auto' =
ceil(n / (4 * threads))), each chunk writes its own output slice, results
bit-identical to a serial loop for any (threads, chunk), and on failure the
error of the lowest failing index is raised.

``bench`` follows the reference's protocol (one untimed warm-up, then ``runs``
timed runs, mean/min/max) and additionally drains the CUDA device around every
run, so a thunk that only enqueues kernels (the ``device`` API) is timed to
completion rather than to launch.
"""

from __future__ import annotations

import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from .types import ParallelConfig


@dataclass(frozen=True)
class BenchReport:
    label: str
    runs: int
    mean_seconds: float
    min_seconds: float
    max_seconds: float

    def __post_init__(self):
        if self.runs < 1:
            raise ValueError("runs must be >= 1")
        if not (0 < self.min_seconds <= self.mean_seconds <= self.max_seconds):
            raise ValueError("timings must satisfy 0 < min <= mean <= max")

    def csv_row(self) -> str:
        fields = (self.label, self.runs, repr(self.mean_seconds), repr(self.min_seconds),
                  repr(self.max_seconds))
        return ",".join(str(f) for f in fields)


def _chunks(n: int, config: ParallelConfig):
    threads = config.resolve_threads()
    size = config.resolve_chunk(n, threads)
    return threads, [(lo, min(lo + size, n)) for lo in range(0, n, size)]


def parallel_map(n: int, kernel, config: ParallelConfig | None = None, *,
                 vectorized: bool = False, width: int = 1, dtype=np.float64) -> np.ndarray:
    """Evaluate kernel over indices 0..n-1 (kernel(i) -> value, or with
    vectorized=True kernel(index_array) -> (len,) / (len, width))."""
    if n < 0:
        raise ValueError("n must be non-negative")
    out = np.empty(n if width == 1 else (n, width), dtype=dtype)
    if n == 0:
        return out
    threads, spans = _chunks(n, config or ParallelConfig())

    def fill(span):
        lo, hi = span
        if vectorized:
            out[lo:hi] = kernel(np.arange(lo, hi, dtype=np.intp))
        else:
            for i in range(lo, hi):
                out[i] = kernel(i)

    if threads == 1 or len(spans) == 1:
        for span in spans:
            fill(span)
        return out

    def guarded(span):
        try:
            fill(span)
            return None
        except Exception as exc:   # surfaced below in index order
            return span[0], exc

    with ThreadPoolExecutor(max_workers=threads) as pool:
        errors = sorted((e for e in pool.map(guarded, spans) if e is not None),
                        key=lambda e: e[0])
    if errors:
        raise errors[0][1]
    return out


def _drain():
    try:
        import torch

        if torch.cuda.is_available() and torch.cuda.is_initialized():
            torch.cuda.synchronize()
    except ImportError:
        pass


def bench(label: str, runs: int, thunk) -> BenchReport:
    """One untimed warm-up, then ``runs`` timed runs of thunk()."""
    if runs < 1:
        raise ValueError("runs must be >= 1")
    thunk()
    _drain()
    samples = []
    for _ in range(runs):
        t0 = time.perf_counter()
        thunk()
        _drain()
        samples.append(time.perf_counter() - t0)
    return BenchReport(label, runs, sum(samples) / runs, min(samples), max(samples))
