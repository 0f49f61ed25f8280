"""ctypes binding of libdivuq_b200.so (declared in include/divuq_b200.h).

There is deliberately no fallback: if the CUDA library is missing or does not
load, importing the package raises.  Build it with
``python -c "import __graft_entry__ as g; g.build()"`` (or ``make -C
paper_2510_01190_b200/csrc``).
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# DIVUQ_LIB_PATH: load an experimental build instead (tools/ sweeps only)
LIB_PATH = os.environ.get("DIVUQ_LIB_PATH") or os.path.join(_HERE, "libdivuq_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: the B200 CUDA library has not been built "
        "(run __graft_entry__.build()); there is no CPU fallback"
    )

lib = ctypes.CDLL(LIB_PATH)

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_f64 = ctypes.c_double
_int = ctypes.c_int

# name -> (restype, argtypes)
SIGNATURES = {
    "divuq_abi_version": (_int, []),
    "divuq_status_string": (ctypes.c_char_p, [_int]),
    "divuq_propagate2d_f64": (_int, [_p] * 4 + [_i64, _i64, _f64, _f64, _f64] + [_p] * 4 + [_p, _p]),
    "divuq_propagate2d_f32": (_int, [_p] * 4 + [_i64, _i64, _f64, _f64, _f64] + [_p] * 4 + [_p, _p]),
    "divuq_propagate3d_f32": (
        _int, [_p] * 10 + [_i64] * 7 + [_f64] * 4 + [_p] * 4 + [_p, _p]),
    "divuq_propagate3d_f64": (
        _int, [_p] * 10 + [_i64] * 7 + [_f64] * 4 + [_p] * 4 + [_p, _p]),
    "divuq_fit_gaussian_f64": (_int, [_p, _i64, _i64, _i64, _p, _p, _p, _p]),
    "divuq_fit_gaussian_f32": (_int, [_p, _i64, _i64, _i64, _p, _p, _p, _p]),
    "divuq_ensemble_divergence2d_f32": (
        _int, [_p, _i64, _i64, _i64, _f64, _f64, _f64] + [_p] * 6 + [_p, _p]),
    "divuq_ensemble_divergence3d_f32": (
        _int, [_p, _i64] + [_p] * 6 + [_i64] * 7 + [_f64] * 4 + [_p] * 6 + [_p, _p]),
    "divuq_tail_probs_f64": (_int, [_p, _p, _i64, _f64, _p, _p, _p, _p]),
    "divuq_tail_probs_f32": (_int, [_p, _p, _i64, _f64, _p, _p, _p, _p]),
    "divuq_host_tail_probs_f64": (_int, [_p, _p, _i64, _f64, _p, _p, _int]),
    "divuq_lcp2d_f64": (_int, [_p, _p, _i64, _i64, _f64, _p, _p, _p]),
    "divuq_lcp2d_f32": (_int, [_p, _p, _i64, _i64, _f64, _p, _p, _p]),
    "divuq_cell_crossing_f64": (_int, [_p, _p, _i64, _f64, _p, _p, _p]),
    "divuq_host_lcp2d_f64": (_int, [_p, _p, _i64, _i64, _f64, _p, _int]),
    "divuq_error_metrics_f64": (_int, [_p] * 4 + [_i64, _p, _p, _p]),
    "divuq_error_metrics_scratch_bytes": (_i64, []),
    "divuq_host_error_metrics_f64": (_int, [_p] * 4 + [_i64, _p, _int]),
    "divuq_propagate_lcp2d_f64": (_int, [_p] * 4 + [_i64, _i64, _f64, _f64, _f64] + [_p] * 4 + [_p]),
    "divuq_host_propagate_lcp2d_f64": (_int, [_p] * 4 + [_i64, _i64, _f64, _f64, _f64] + [_p] * 3 + [_int]),
    "divuq_host_cell_crossing_f64": (_int, [_p, _p, _i64, _f64, _p, _int]),
    "divuq_velocity_magnitude_f64": (_int, [_p, _p, _i64, _p, _p, _p]),
    "divuq_gradient2d_f64": (_int, [_p, _i64, _i64, _f64, _f64, _p, _p, _p]),
    "divuq_gradient_ensemble2d_f64": (_int, [_p, _i64, _i64, _i64, _f64, _f64, _p, _p, _p]),
    "divuq_gradient_ensemble2d_f32": (_int, [_p, _i64, _i64, _i64, _f64, _f64, _p, _p, _p]),
    "divuq_host_velocity_magnitude_f64": (_int, [_p, _p, _i64, _p, _int]),
    "divuq_host_gradient2d_f64": (_int, [_p, _i64, _i64, _f64, _f64, _p, _int]),
    "divuq_host_gradient_ensemble2d_f64": (_int, [_p, _i64, _i64, _i64, _f64, _f64, _p, _int]),
    "divuq_divuq1_read_header": (_int, [ctypes.c_char_p, _p, _p, _p, _p, _p]),
    "divuq_divuq1_read_f32": (_int, [ctypes.c_char_p, _p, _i64, _int]),
    "divuq_divuq1_ingest_f32": (_int, [ctypes.c_char_p, _p, _i64, _int]),
    "divuq_divuq1_write_f32": (_int, [ctypes.c_char_p, _i64, _i64, _f64, _f64, _i64, _p]),
    "divuq_divuq1_format_real": (_int, [_f64, ctypes.c_char_p, _i64]),
    "divuq_mc_scratch_bytes": (_i64, [_i64, _i64, _i64, _i64]),
    "divuq_mc_divergence2d_f64": (
        _int, [_p] * 4 + [_i64, _i64, _f64, _f64, _i64, _u64, _i64, _i64] + [_p] * 3 + [_p, _p]),
    "divuq_gen_field_f32": (
        _int, [_p, _int, _int, _i64, _i64, _i64, _i64, _f64, _f64, _f64, _f64, _f64, _f64, _f64,
               _f64, _u64, _f64, _f64, _int, _i64, _p, _p, _p]),
    "divuq_host_propagate2d_f64": (
        _int, [_p] * 4 + [_i64, _i64, _f64, _f64, _f64] + [_p] * 4 + [_int]),
    "divuq_host_propagate3d_f32": (
        _int, [_p] * 6 + [_i64] * 3 + [_f64] * 4 + [_p] * 4 + [_i64, _int]),
    "divuq_host_ensemble_divergence3d_f32": (
        _int, [_p] + [_i64] * 6 + [_p, _p, _i64] + [_f64] * 4 + [_p] * 4 + [_i64, _int]),
    "divuq_gradient_ensemble_divergence2d_f32": (
        _int, [_p, _i64, _i64, _i64, _f64, _f64, _f64] + [_p] * 6 + [_p, _p]),
    "divuq_host_gradient_ensemble_divergence2d_f32": (
        _int, [_p, _i64, _i64, _i64, _f64, _f64, _f64] + [_p] * 6 + [_int]),
    "divuq_host_fit_gaussian_f64": (_int, [_p, _i64, _i64, _i64, _p, _p, _int]),
    "divuq_host_ensemble_divergence2d_f32": (
        _int, [_p, _i64, _i64, _i64, _f64, _f64, _f64] + [_p] * 6 + [_int]),
    "divuq_host_mc_divergence2d_f64": (
        _int, [_p] * 4 + [_i64, _i64, _f64, _f64, _i64, _u64, _p, _p, _int]),
    "divuq_mc_divergence2d_ref_f64": (
        _int, [_p] * 4 + [_i64, _i64, _f64, _f64, _i64, _u64, _i64, _i64] + [_p] * 2 + [_p, _p]),
    "divuq_sample_divergence1d_f64": (_int, [_p, _f64, _f64, _i64, _u64, _p, _p]),
    "divuq_minmax_f64": (_int, [_p, _i64, _p, _p, _p]),
    "divuq_histogram_uniform_f64": (_int, [_p, _i64, _f64, _f64, _i64, _p, _p, _p]),
    "divuq_host_mc_divergence2d_ref_f64": (
        _int, [_p] * 4 + [_i64, _i64, _f64, _f64, _i64, _u64, _p, _p, _int]),
    "divuq_fit_gaussian_strided_f32": (_int, [_p, _i64, _i64, _i64, _p, _p, _p, _p, _p]),
    "divuq_host_register": (_int, [_p, _i64]),
    "divuq_host_unregister": (_int, [_p]),
    "divuq_ipc_handle_bytes": (_i64, []),
    "divuq_ipc_export": (_int, [_p, _p, _p]),
    "divuq_ipc_import": (_int, [_p, _i64, _p, _p]),
    "divuq_ipc_close": (_int, [_p]),
    "divuq_host_mc_histogram1d_f64": (
        _int, [_p, _f64, _f64, _i64, _u64, _i64, _p, _p, _p, _p, _int]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _fn = getattr(lib, _name)  # AttributeError here = header/library mismatch
    _fn.restype = _res
    _fn.argtypes = _args

ABI_VERSION = lib.divuq_abi_version()
if ABI_VERSION != 2:
    raise ImportError(f"libdivuq_b200 ABI {ABI_VERSION} != 2 (rebuild: __graft_entry__.build())")

# status codes (include/divuq_b200.h)
OK, EINVAL, EGRID, EMEMBERS, ESAMPLES, ENONFINITE, ENEGSIGMA = 0, -1, -2, -3, -4, -10, -11
EFORMAT, ELENGTH, EOS, EDATA = -20, -21, -22, -23


class DivuqError(RuntimeError):
    """CUDA-side failure (status > 0 is a cudaError_t)."""


def check(status: int) -> None:
    """Map a C status to the reference's exception types."""
    if status == OK:
        return
    msg = lib.divuq_status_string(status).decode()
    if status < 0:
        raise ValueError(msg)
    raise DivuqError(f"CUDA error {status}: {msg}")
