"""DIVUQ1 container restated -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates the reference reader (/root/reference/pkg/src/divuq/io.py:58-93):
readline() header, split(), int/float fields, UniformGrid2 validation
(grid.py:41-45), payload length check, fp32 -> fp64 widening, finiteness.
Raises ValueError subclasses named like the reference's (FormatError,
LengthError, DataError) as plain strings in ``kind`` so the checker does not
depend on the product's exception classes.  Pinned by tests/test_divuq1.py
against files written by the reference itself (tests/golden/divuq1_*.duq).
"""

from __future__ import annotations

import numpy as np


class OracleIOError(ValueError):
    def __init__(self, kind, msg):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


def read_members(path):
    """-> ((nx, ny, dx, dy), (M, 2, N) float64 array)  (io.py:58-93)."""
    with open(path, "rb") as fh:
        header = fh.readline()
        payload = fh.read()
    parts = header.decode("ascii", errors="replace").split()
    if len(parts) != 6 or parts[0] != "DIVUQ1":
        raise OracleIOError("FormatError", "bad magic")
    try:
        nx, ny = int(parts[1]), int(parts[2])
        dx, dy = float(parts[3]), float(parts[4])
        m = int(parts[5])
    except ValueError as exc:
        raise OracleIOError("FormatError", str(exc)) from exc
    if m < 1 or nx < 2 or ny < 2 or not (dx > 0 and dy > 0):
        raise OracleIOError("FormatError", "bad header values")
    if len(payload) != m * 2 * nx * ny * 4:
        raise OracleIOError("LengthError", f"{len(payload)} bytes")
    planes = np.frombuffer(payload, dtype="<f4").astype(np.float64).reshape(m, 2, nx * ny)
    if not np.all(np.isfinite(planes)):
        raise OracleIOError("DataError", "non-finite")
    return (nx, ny, dx, dy), planes


def fmt_real(x: float) -> str:
    """io.py:38-40."""
    return repr(int(x)) if float(x).is_integer() and abs(x) < 2**53 else repr(float(x))


def header(nx, ny, dx, dy, m) -> bytes:
    """io.py:45-47."""
    return f"DIVUQ1 {nx} {ny} {fmt_real(dx)} {fmt_real(dy)} {m}\n".encode("ascii")
