"""DIVUQ1 container (reference io.py:1-134).

The ``.duq`` fixtures in tests/golden were written by the reference's own
``write_members`` (make_golden.py); ours must parse them and re-emit identical
bytes.  The reference suite's io cases (pkg/tests/test_io.py) are mirrored,
plus header edge cases of Python's int()/float() parsing.  Header parsing,
payload reads and writes are host-side native code (no kernel launches), so
these run in the CPU suite; the pinned-staging HBM ingest runs under -m gpu.
"""

import math
import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN

GOLD = ["ens_a", "ens_b", "ens_c", "ens_d"]


@pytest.fixture(scope="module")
def d():
    import __graft_entry__

    __graft_entry__.build()
    import paper_2510_01190_b200

    return paper_2510_01190_b200


@pytest.fixture(scope="module")
def io(d):
    from paper_2510_01190_b200 import io

    return io


def _gold(name):
    return os.path.join(GOLDEN, f"divuq1_{name}.duq")


def _split(path):
    raw = open(path, "rb").read()
    nl = raw.index(b"\n") + 1
    return raw[:nl].decode(), np.frombuffer(raw[nl:], dtype="<f4")


def _ref_fmt(x):
    # the reference's _fmt (io.py:38-40), for comparison only
    return repr(int(x)) if float(x).is_integer() and abs(x) < 2**53 else repr(float(x))


def _ens(d, rng, nx=6, ny=5, members=4, dx=0.5, dy=2.0):
    g = d.UniformGrid2(nx, ny, dx, dy)
    mk = []
    for _ in range(members):
        u = rng.normal(size=g.n_vertices).astype(np.float32).astype(np.float64)
        v = rng.normal(size=g.n_vertices).astype(np.float32).astype(np.float64)
        mk.append(d.VectorField2(g, u, v))
    return d.Ensemble2(g, tuple(mk))


@pytest.mark.parametrize("name", GOLD)
def test_reads_reference_written_files(io, name):
    header, payload = _split(_gold(name))
    parts = header.split()
    grid, members = io.read_members(_gold(name))
    assert (grid.nx, grid.ny) == (int(parts[1]), int(parts[2]))
    assert (grid.dx, grid.dy) == (float(parts[3]), float(parts[4]))
    assert len(members) == int(parts[5])
    planes = payload.reshape(len(members), 2, grid.n_vertices)
    for k, m in enumerate(members):
        assert np.array_equal(m.u, planes[k, 0].astype(np.float64))
        assert np.array_equal(m.v, planes[k, 1].astype(np.float64))


@pytest.mark.parametrize("name", GOLD)
def test_writes_reference_identical_bytes(io, tmp_path, name):
    grid, members = io.read_members(_gold(name))
    p = tmp_path / "again.duq"
    io.write_members(grid, members, p)
    assert p.read_bytes() == open(_gold(name), "rb").read()


def test_header_reals_match_python_repr(io):
    rng = np.random.default_rng(7)
    xs = [0.1, 1e-3, 0.5, 2.0, 1.0, 123456.789, 3e-7, 1e16, 1e15, 2.0**53, 2.0**53 - 1,
          2.0**53 + 2, 1e-4, 1e-5, 0.0001234, 9.999999999999999e15, 1e22, 5e-324,
          1.7976931348623157e308, 2.2250738585072014e-308, 0.3333333333333333, -0.25,
          -7.0, 0.0, -0.0, math.inf, -math.inf, math.nan, 100.5, 1234567890123456.7]
    xs += list(rng.normal(size=200) * 10.0 ** rng.integers(-30, 30, 200))
    xs += list(rng.integers(-(2**60), 2**60, 50).astype(np.float64))
    xs += list(np.frombuffer(rng.bytes(8 * 300), dtype=np.float64))
    for x in xs:
        assert io._fmt(float(x)) == _ref_fmt(float(x)), x


# ---- pkg/tests/test_io.py cases --------------------------------------------

def test_single_member_zero_file(d, io, tmp_path):
    p = tmp_path / "zero.duq"
    p.write_bytes(b"DIVUQ1 2 2 1 1 1\n" + b"\x00" * 32)
    grid, members = io.read_members(p)
    assert grid == d.UniformGrid2(2, 2, 1.0, 1.0)
    assert len(members) == 1 and np.all(members[0].u == 0.0) and np.all(members[0].v == 0.0)


def test_hand_assembled_indexing_convention(io, tmp_path):
    u = np.zeros(6, dtype="<f4")
    u[1] = 1.0
    p = tmp_path / "hand.duq"
    p.write_bytes(b"DIVUQ1 3 2 1 1 1\n" + u.tobytes() + np.zeros(6, dtype="<f4").tobytes())
    _, members = io.read_members(p)
    assert members[0].u[1] == 1.0 and members[0].u.sum() == 1.0


def test_ensemble_roundtrip_bit_exact(d, io, tmp_path, rng):
    ens = _ens(d, rng)
    p = tmp_path / "ens.duq"
    io.write_ensemble(ens, p)
    back = io.read_ensemble(p)
    assert back.grid == ens.grid
    for a, b in zip(ens.members, back.members):
        assert np.array_equal(a.u, b.u) and np.array_equal(a.v, b.v)
    p2 = tmp_path / "ens2.duq"
    io.write_ensemble(back, p2)
    assert p.read_bytes() == p2.read_bytes()


def test_file_size_arithmetic(d, io, tmp_path, rng):
    ens = _ens(d, rng, nx=10, ny=8, members=20)
    p = tmp_path / "sized.duq"
    io.write_ensemble(ens, p)
    header = b"DIVUQ1 10 8 0.5 2 20\n"
    assert p.read_bytes().startswith(header)
    assert p.stat().st_size == len(header) + 20 * 2 * 80 * 4


def test_fp64_members_round_to_fp32_like_numpy(d, io, tmp_path):
    g = d.UniformGrid2(4, 4)
    rng = np.random.default_rng(3)
    members = [d.VectorField2(g, rng.normal(size=16), rng.normal(size=16)) for _ in range(2)]
    p = tmp_path / "r.duq"
    io.write_members(g, members, p)
    _, payload = _split(p)
    want = np.concatenate([np.concatenate([m.u, m.v]) for m in members]).astype("<f4")
    assert payload.tobytes() == want.tobytes()


@pytest.mark.parametrize("header,exc", [
    (b"NOTDUQ 2 2 1 1 1\n", "FormatError"),
    (b"DIVUQ1 2 2 1 1\n", "FormatError"),
    (b"DIVUQ1 2 2 1 1 1 1\n", "FormatError"),
    (b"DIVUQ1 2.0 2 1 1 1\n", "FormatError"),
    (b"DIVUQ1 2 2 0x1p0 1 1\n", "FormatError"),
    (b"DIVUQ1 2 2 nan 1 1\n", "FormatError"),
    (b"DIVUQ1 2 2 0 1 1\n", "FormatError"),
    (b"DIVUQ1 2 2 -1 1 1\n", "FormatError"),
    (b"DIVUQ1 1 2 1 1 1\n", "FormatError"),
    (b"DIVUQ1 2 2 1 1 0\n", "FormatError"),
    (b"DIVUQ1 2 2 1e 1 1\n", "FormatError"),
    (b"DIVUQ1 2 2 1._5 1 1\n", "FormatError"),
    (b"", "FormatError"),
    (b"DIVUQ1 4611686018427387904 4 1 1 1\n", "LengthError"),
])
def test_malformed_headers(io, tmp_path, header, exc):
    p = tmp_path / "bad.duq"
    p.write_bytes(header + b"\x00" * 32)
    with pytest.raises(getattr(io, exc)):
        io.read_members(p)


@pytest.mark.parametrize("header", [
    b"DIVUQ1 2 2 1 1 1\r\n", b"DIVUQ1\t2 2 1.0 1e0 1\n", b"  DIVUQ1 2 2 +1 1 1\n",
    b"DIVUQ1 2 2 1_0.5 1 1\n", b"DIVUQ1 0_2 2 1 1 1\n", b"DIVUQ1 2 2 Infinity 1 1\n",
])
def test_python_number_syntax_accepted(io, tmp_path, header):
    p = tmp_path / "ok.duq"
    p.write_bytes(header + b"\x00" * 32)
    grid, members = io.read_members(p)
    parts = header.split()
    assert grid.dx == float(parts[3].decode()) and grid.nx == int(parts[1].decode())


def test_truncated_and_overlong_payload(io, tmp_path):
    for n in (31, 33, 0):
        p = tmp_path / f"len{n}.duq"
        p.write_bytes(b"DIVUQ1 2 2 1 1 1\n" + b"\x00" * n)
        with pytest.raises(io.LengthError):
            io.read_members(p)
    p = tmp_path / "nonl.duq"
    p.write_bytes(b"DIVUQ1 2 2 1 1 1")  # no newline: all header, empty payload
    with pytest.raises(io.LengthError):
        io.read_members(p)


def test_non_finite_payload(io, tmp_path):
    for bad in (float("nan"), float("inf"), float("-inf")):
        p = tmp_path / "nan.duq"
        p.write_bytes(b"DIVUQ1 2 2 1 1 1\n" + struct.pack("<f", 0.0) * 7 + struct.pack("<f", bad))
        with pytest.raises(io.DataError):
            io.read_members(p)


def test_exception_hierarchy_and_missing_file(io, tmp_path):
    assert issubclass(io.FormatError, ValueError) and issubclass(io.LengthError, ValueError)
    assert issubclass(io.DataError, ValueError)
    with pytest.raises(OSError):
        io.read_members(tmp_path / "nope.duq")


def test_read_ensemble_requires_two_members(io, tmp_path):
    p = tmp_path / "one.duq"
    p.write_bytes(b"DIVUQ1 2 2 1 1 1\n" + b"\x00" * 32)
    with pytest.raises(io.DataError):
        io.read_ensemble(p)


def test_write_to_unwritable_path(d, io, tmp_path, rng):
    with pytest.raises(OSError):
        io.write_ensemble(_ens(d, rng), tmp_path / "missing_dir" / "x.duq")


def test_scalar_roundtrip(d, io, tmp_path):
    g = d.UniformGrid2(4, 3, 0.25, 0.5)
    values = np.arange(12, dtype=np.float64)
    p = tmp_path / "scalar.duq"
    io.write_scalar(d.ScalarField2(g, values), p)
    back = io.read_scalar(p)
    assert back.grid == g and np.array_equal(back.values, values)
    with pytest.raises(io.DataError):
        io.read_scalar(_gold("ens_a"))


def test_model_roundtrip_and_checks(d, io, tmp_path, rng):
    ens = _ens(d, rng)
    st = ens.stacked()
    mu, sg = st.mean(axis=0), st.std(axis=0, ddof=1)
    model = d.GaussianVectorField(ens.grid, mu[0], mu[1], sg[0], sg[1])
    io.write_model(model, tmp_path / "mu.duq", tmp_path / "sg.duq")
    back = io.read_model(tmp_path / "mu.duq", tmp_path / "sg.duq")
    assert np.allclose(back.mu_u, model.mu_u, rtol=1e-7)
    assert np.allclose(back.sigma_v, model.sigma_v, rtol=1e-6, atol=1e-7)
    # sigmas must be non-negative; grids must agree
    io.write_members(ens.grid, (d.VectorField2(ens.grid, -sg[0], sg[1]),), tmp_path / "neg.duq")
    with pytest.raises(io.DataError):
        io.read_model(tmp_path / "mu.duq", tmp_path / "neg.duq")
    g2 = d.UniformGrid2(6, 5, 0.5, 2.5)
    io.write_members(g2, (d.VectorField2(g2, sg[0], sg[1]),), tmp_path / "g2.duq")
    with pytest.raises(io.DataError):
        io.read_model(tmp_path / "mu.duq", tmp_path / "g2.duq")


def test_grid_spacing_survives_header(d, io, tmp_path):
    g = d.UniformGrid2(3, 3, 0.1, 1e-3)
    members = tuple(d.VectorField2(g, np.zeros(9), np.zeros(9)) for _ in range(2))
    p = tmp_path / "spacing.duq"
    io.write_members(g, members, p)
    grid, _ = io.read_members(p)
    assert grid.dx == 0.1 and grid.dy == 1e-3


# ---- HBM ingest ------------------------------------------------------------

@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.gpu
@pytest.mark.parametrize("name", GOLD)
def test_ingest_golden_to_hbm(io, torch_cuda, name):
    grid, x = io.load_ensemble_device(_gold(name))
    _, payload = _split(_gold(name))
    assert x.is_cuda and x.dtype == torch_cuda.float32
    assert np.array_equal(x.cpu().numpy().ravel(), payload)


@pytest.mark.gpu
def test_ingest_multi_chunk_file_and_fused_pipeline(d, io, torch_cuda, tmp_path):
    # 3 members x 2 x 3.2M floats = 19.2M floats: crosses the 16M-float staging
    # chunk, so both pinned buffers are reused at least once
    from paper_2510_01190_b200 import device

    g = d.UniformGrid2(2000, 1600, 0.01, 0.02)
    rng = np.random.default_rng(11)
    block = rng.normal(size=(3, 2, g.n_vertices)).astype(np.float32)
    p = tmp_path / "big.duq"
    with open(p, "wb") as fh:
        fh.write(f"DIVUQ1 {g.nx} {g.ny} 0.01 0.02 3\n".encode())
        fh.write(block.tobytes())
    grid, x = io.load_ensemble_device(p)
    assert grid == g
    assert torch_cuda.equal(x.cpu(), torch_cuda.from_numpy(block))
    got = device.ensemble_divergence2d(x, g.nx, g.ny, g.dx, g.dy, 0.1)
    want = device.ensemble_divergence2d(torch_cuda.from_numpy(block).cuda(), g.nx, g.ny, g.dx,
                                        g.dy, 0.1)
    for k in want:
        assert torch_cuda.equal(got[k], want[k])


@pytest.mark.gpu
def test_ingest_non_finite_rejected_by_consumer(d, io, torch_cuda, tmp_path):
    from paper_2510_01190_b200 import device

    p = tmp_path / "nan.duq"
    vals = np.zeros((2, 2, 9), dtype="<f4")
    vals[1, 0, 4] = np.nan
    p.write_bytes(b"DIVUQ1 3 3 1 1 2\n" + vals.tobytes())
    grid, x = io.load_ensemble_device(p)
    with pytest.raises(ValueError):
        device.ensemble_divergence2d(x, 3, 3)
    with pytest.raises(io.DataError):
        io.read_ensemble(p)


def _read_in_child(path, q):
    from paper_2510_01190_b200 import io as dio

    ens = dio.read_ensemble(path)
    q.put(float(sum(float(m.u.sum()) + float(m.v.sum()) for m in ens.members)))


def test_parallel_reader_survives_fork(d, io, tmp_path, rng):
    """The native reader splits large payloads over a persistent host worker
    pool; a fork()ed child (multiprocessing's default on Linux) has none of
    the parent's workers and must build its own instead of waiting forever."""
    import multiprocessing as mp

    ens = _ens(d, rng, nx=512, ny=512, members=2)    # 4 MB payload: 4 workers
    p = tmp_path / "big.duq"
    io.write_ensemble(ens, p)
    back = io.read_ensemble(p)                        # the parent's pool exists now
    want = float(sum(float(m.u.sum()) + float(m.v.sum()) for m in back.members))
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    proc = ctx.Process(target=_read_in_child, args=(str(p), q))
    proc.start()
    got = q.get(timeout=60)
    proc.join(timeout=30)
    assert proc.exitcode == 0 and got == want
