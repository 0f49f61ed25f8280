"""The reference's parallel seam kept for drop-in callers (parallel.py:19-129):
the reference suite's own properties (pkg/tests/test_parallel.py) on this
package -- determinism for any (threads, chunk), vectorised == scalar, first
failure by index, BenchReport invariants -- plus the hot path's side of the
contract: propagation is bit-identical for every ParallelConfig (one kernel
launch, the config is accepted and has no effect).  CPU-only except the last."""

import numpy as np
import pytest


@pytest.fixture(scope="module")
def d():
    import __graft_entry__

    __graft_entry__.build()
    import paper_2510_01190_b200

    return paper_2510_01190_b200


def test_map_contract(d):
    assert d.parallel_map(0, lambda i: i).shape == (0,)
    ref = d.parallel_map(1000, lambda i: float(i), d.ParallelConfig(threads=1))
    for threads in (4, 16):
        got = d.parallel_map(1000, lambda i: float(i), d.ParallelConfig(threads=threads, chunk=7))
        assert np.array_equal(ref, got)
    a = d.parallel_map(500, lambda idx: np.sin(idx.astype(float)), d.ParallelConfig(threads=3, chunk=11),
                       vectorized=True)
    assert np.array_equal(a, np.sin(np.arange(500, dtype=float)))
    w = d.parallel_map(10, lambda i: (i, 2 * i), width=2)
    assert w.shape == (10, 2) and w[3, 1] == 6


def test_first_error_by_index_order(d):
    def kernel(i):
        if i in (42, 7):
            raise RuntimeError(f"boom at {i}")
        return float(i)

    with pytest.raises(RuntimeError, match="boom at 7"):
        d.parallel_map(100, kernel, d.ParallelConfig(threads=4, chunk=5))
    with pytest.raises(ValueError):
        d.parallel_map(-1, lambda i: i)


def test_bench_and_report(d):
    r = d.bench("noop", 3, lambda: sum(range(1000)))
    assert r.runs == 3 and 0 < r.min_seconds <= r.mean_seconds <= r.max_seconds
    assert r.csv_row().startswith("noop,3,")
    with pytest.raises(ValueError):
        d.BenchReport("x", 0, 1.0, 1.0, 1.0)
    with pytest.raises(ValueError):
        d.BenchReport("x", 1, 1.0, 2.0, 3.0)
    with pytest.raises(ValueError):
        d.bench("x", 0, lambda: None)
    assert d.ParallelConfig(threads=2).resolve_chunk(100, 2) == 13


@pytest.mark.gpu
def test_propagation_bit_identical_for_every_config(d):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(3)
    g = d.UniformGrid2(120, 90, 0.2, 0.9)
    n = g.n_vertices
    model = d.GaussianVectorField(g, rng.normal(0, 2, n), rng.normal(0, 2, n),
                                  rng.uniform(0.05, 0.6, n), rng.uniform(0.05, 0.6, n))
    serial = d.propagate_divergence(model)
    for threads in (1, 2, 8):
        for chunk in ("auto", 101):
            par = d.propagate_divergence(model, d.ParallelConfig(threads=threads, chunk=chunk))
            assert np.array_equal(serial.mu, par.mu) and np.array_equal(serial.sigma, par.sigma)
