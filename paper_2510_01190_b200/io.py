"""DIVUQ1 container: drop-in for the reference's ``divuq.io``.

Same names, layout, exceptions and bytes as /root/reference/pkg/src/divuq/io.py
(header ``DIVUQ1 nx ny dx dy M\\n`` then M blocks of u-plane, v-plane as
little-endian fp32, io.py:1-14).  Header parsing, the payload read and the
byte-deterministic writer are native (``divuq_divuq1_*`` in the C ABI); the
payload is already the (M, 2, N) member-major fp32 block the ensemble kernels
read, so ``load_ensemble_device`` streams it disk -> pinned -> HBM with no
host-side reshaping, ready for ``device.ensemble_divergence2d``.  The CSV
helpers (io.py:137-148) serve the CLI routing (``cli.py``).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from ._lib import lib
from .types import Ensemble2, GaussianVectorField, ScalarField2, UniformGrid2, VectorField2

MAGIC = "DIVUQ1"


class FormatError(ValueError):
    """Bad magic or malformed header (io.py:26-27)."""


class LengthError(ValueError):
    """Payload shorter or longer than the header promises (io.py:30-31)."""


class DataError(ValueError):
    """Payload parses but contains invalid values (io.py:34-35)."""


def _raise(status: int, path, what: str) -> None:
    if status == _lib.OK:
        return
    msg = f"{path}: {lib.divuq_status_string(status).decode()}"
    if status == _lib.EFORMAT:
        raise FormatError(msg)
    if status == _lib.ELENGTH:
        raise LengthError(msg)
    if status == _lib.EDATA:
        raise DataError(msg)
    if status == _lib.EOS:
        raise OSError(f"cannot {what} {path}")
    _lib.check(status)


def _fmt(x: float) -> str:
    """Shortest decimal that parses back to exactly x (io.py:38-40), native."""
    buf = ctypes.create_string_buffer(64)
    _lib.check(lib.divuq_divuq1_format_real(float(x), buf, 64))
    return buf.value.decode("ascii")


def read_header(path) -> tuple[UniformGrid2, int]:
    """Parse and validate the header and payload length (io.py:58-86)."""
    nx, ny, m = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    dx, dy = ctypes.c_double(), ctypes.c_double()
    _raise(lib.divuq_divuq1_read_header(os.fsencode(path), ctypes.addressof(nx),
                                        ctypes.addressof(ny), ctypes.addressof(dx),
                                        ctypes.addressof(dy), ctypes.addressof(m)), path, "read")
    return UniformGrid2(nx.value, ny.value, dx.value, dy.value), m.value


def read_payload_f32(path) -> tuple[UniformGrid2, np.ndarray]:
    """Header + the (M, 2, N) fp32 payload, non-finite values rejected."""
    grid, m = read_header(path)
    out = np.empty((m, 2, grid.n_vertices), dtype=np.float32)
    _raise(lib.divuq_divuq1_read_f32(os.fsencode(path), out.ctypes.data, out.size, 1), path, "read")
    return grid, out


def _write_planes(grid: UniformGrid2, planes, path) -> None:
    """(u, v) plane pairs -> one DIVUQ1 file (fp64 values rounded to fp32)."""
    planes = list(planes)
    block = np.empty((len(planes), 2, grid.n_vertices), dtype=np.float32)
    for k, (u, v) in enumerate(planes):
        block[k] = (u, v)
    _raise(lib.divuq_divuq1_write_f32(os.fsencode(path), grid.nx, grid.ny, float(grid.dx),
                                      float(grid.dy), len(planes), block.ctypes.data),
           path, "write")


def write_members(grid: UniformGrid2, members, path) -> None:
    """Byte-identical to io.py:43-55."""
    _write_planes(grid, ((mb.u, mb.v) for mb in members), path)


def read_members(path) -> tuple[UniformGrid2, tuple[VectorField2, ...]]:
    """io.py:58-93: members as fp64 fields (exact widening of the fp32 payload)."""
    grid, block = read_payload_f32(path)
    wide = block.astype(np.float64)
    return grid, tuple(VectorField2(grid, wide[k, 0], wide[k, 1]) for k in range(wide.shape[0]))


def _single_block(path, what: str):
    """The one (u, v) block of a scalar / model file, with io.py's errors."""
    grid, blocks = read_members(path)
    if len(blocks) != 1:
        if what == "scalar":
            raise DataError(f"{path}: expected a single-block scalar file, got {len(blocks)} blocks")
        raise DataError("model files must contain exactly one block each")
    return grid, blocks[0]


def write_ensemble(ensemble: Ensemble2, path) -> None:
    write_members(ensemble.grid, ensemble.members, path)


def read_ensemble(path) -> Ensemble2:
    """io.py:100-104: at least two members."""
    grid, found = read_members(path)
    if len(found) < 2:
        raise DataError(f"{path}: an ensemble needs >= 2 members, file has {len(found)}")
    return Ensemble2(grid, found)


def write_scalar(fld: ScalarField2, path) -> None:
    """A scalar is a one-block file with v = 0 (io.py:107-111)."""
    _write_planes(fld.grid, [(fld.values, np.zeros_like(fld.values))], path)


def read_scalar(path) -> ScalarField2:
    grid, block = _single_block(path, "scalar")
    return ScalarField2(grid, block.u)


def write_model(model: GaussianVectorField, mu_path, sigma_path) -> None:
    """Two one-block files: (mu_u, mu_v) and (sigma_u, sigma_v) (io.py:114-119)."""
    for path, pair in ((mu_path, (model.mu_u, model.mu_v)), (sigma_path, (model.sigma_u, model.sigma_v))):
        _write_planes(model.grid, [pair], path)


def read_model(mu_path, sigma_path) -> GaussianVectorField:
    """io.py:122-134 (same checks, same order)."""
    g_mu, blocks_mu = read_members(mu_path)
    g_sg, blocks_sg = read_members(sigma_path)
    if g_mu != g_sg:
        raise DataError(f"{mu_path} and {sigma_path} are on different grids")
    if len(blocks_mu) != 1 or len(blocks_sg) != 1:
        raise DataError("model files must contain exactly one block each")
    mean, spread = blocks_mu[0], blocks_sg[0]
    if (spread.u < 0).any() or (spread.v < 0).any():
        raise DataError(f"{sigma_path}: sigmas must be non-negative")
    return GaussianVectorField(g_mu, mean.u, mean.v, spread.u, spread.v)


def load_ensemble_device(path, device=None):
    """DIVUQ1 ensemble -> (grid, (M, 2, N) fp32 CUDA tensor), streamed through
    a ring of pinned staging buffers (parallel pread, async H2D).  Non-finite payload values are not scanned
    here: the consuming kernels reject them (device.* ``check=True`` raises
    ValueError, the DataError condition) inside the same pass that reads them."""
    import torch

    grid, m = read_header(path)
    if m < 2:
        raise DataError(f"{path}: an ensemble needs >= 2 members, file has {m}")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    out = torch.empty((m, 2, grid.n_vertices), dtype=torch.float32, device=dev)
    torch.cuda.current_stream(dev).synchronize()  # the allocation may reuse memory in flight
    _raise(lib.divuq_divuq1_ingest_f32(os.fsencode(path), out.data_ptr(), out.numel(),
                                       dev.index if dev.index is not None else 0), path, "read")
    return grid, out


def csv_float(x: float) -> str:
    """Full round-trip precision for CSV cells (io.py:137-139)."""
    return repr(float(x))


def write_csv(path, header: str, rows) -> None:
    """Header row + comma-joined rows, \\n line endings (io.py:142-148)."""
    with open(path, "w", encoding="ascii", newline="\n") as out:   # streamed: LCP CSVs are large
        out.write(header + "\n")
        out.writelines(",".join(map(str, row)) + "\n" for row in rows)
