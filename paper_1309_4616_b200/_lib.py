"""ctypes binding of libexpstencil_b200.so (include/expstencil_b200.h).

This is the product's only compute path: there is no CPU or PyTorch fallback.
If the library is missing or no CUDA device is usable, every operator call
raises immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ConvergenceError, DomainError, ExpStencilError

_HERE = os.path.dirname(os.path.abspath(__file__))
# ES_LIB: an alternative build of the same library (A/B kernel experiments)
LIB_PATH = os.environ.get("ES_LIB") or os.path.join(_HERE, "_lib", "libexpstencil_b200.so")

ES_OK, ES_ERR_ARG, ES_ERR_NOT_CONVERGED, ES_ERR_DOMAIN, ES_ERR_CUDA, ES_ERR_RANGE, ES_ERR_TYPE = 0, 1, 2, 3, 4, 5, 6
ES_KIND_F32, ES_KIND_F64, ES_KIND_C128 = 0, 1, 2
ES_NONLIN_NONE, ES_NONLIN_COMBUSTION = 0, 1
ES_MODE_ZERO, ES_MODE_PERIODIC, ES_MODE_FACES, ES_MODE_NEUMANN = 0, 1, 2, 3
ES_COEFF_NONE, ES_COEFF_RADIAL, ES_COEFF_ARRAY = 0, 1, 2

# every symbol include/expstencil_b200.h declares
EXPORTS = (
    "es_abi_version", "es_last_error", "es_device_available", "es_stencil_fused_slab",
    "es_csr_fused_rows", "es_combustion_pointwise", "es_leja_stencil_workspace_bytes",
    "es_leja_stencil", "es_leja_csr_workspace_bytes", "es_leja_csr", "es_axpy", "es_scale",
    "es_half_sum", "es_combustion_jacobian", "es_max_abs", "es_leja_stencil_async", "es_leja_fetch",
    "es_leja_csr_async", "es_rosenbrock_prologue", "es_leja_dist_begin", "es_leja_dist_source",
    "es_leja_dist_nslices", "es_leja_dist_node", "es_leja_dist_decide", "es_leja_dist_end",
    "es_leja_state_offset", "es_leja_csr_dist_begin", "es_leja_csr_dist_source", "es_leja_csr_dist_nslices",
    "es_leja_csr_dist_node", "es_leja_csr_dist_end", "es_csr_fused_rows_z", "es_leja_csr_z_workspace_bytes",
    "es_leja_csr_z", "es_leja_csr_z_async", "es_leja_stencil_nslices", "es_leja_p2p", "es_ipc_handle",
    "es_ipc_open", "es_ipc_close", "es_leja_csr_nslices", "es_leja_csr_p2p", "es_stencil_fused_slab_f32",
    "es_combustion_pointwise_f32", "es_expeuler_step", "es_exprb_step", "es_exprb_finish", "es_csr_fused_rows_ex",
)


class StencilDesc(ctypes.Structure):
    _fields_ = [
        ("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("lz", ctypes.c_int64),
        ("z0", ctypes.c_int64), ("nz_total", ctypes.c_int64),
        ("wx", ctypes.c_double), ("wy", ctypes.c_double), ("wz", ctypes.c_double),
        ("mode", ctypes.c_int32), ("coeff_kind", ctypes.c_int32),
        ("coeff", ctypes.c_void_p), ("faces", ctypes.c_void_p * 6),
    ]


class P2PDesc(ctypes.Structure):
    _fields_ = [
        ("nranks", ctypes.c_int32), ("rank", ctypes.c_int32),
        ("slice_offset", ctypes.c_int64), ("total_slices", ctypes.c_int64),
        ("halo_lo", ctypes.c_void_p * 2), ("halo_hi", ctypes.c_void_p * 2),
        ("peer_lo", ctypes.c_void_p * 2), ("peer_hi", ctypes.c_void_p * 2),
        ("rank_slices", ctypes.c_void_p), ("rank_arrive", ctypes.c_void_p), ("arrive_local", ctypes.c_void_p),
        ("base", ctypes.c_uint64), ("timeout_ns", ctypes.c_int64),
        ("halo_planes", ctypes.c_int32), ("gdiag_lo", ctypes.c_void_p), ("gdiag_hi", ctypes.c_void_p),
    ]


class P2PRowsDesc(ctypes.Structure):
    _fields_ = [
        ("nranks", ctypes.c_int32), ("rank", ctypes.c_int32),
        ("slice_offset", ctypes.c_int64), ("total_slices", ctypes.c_int64),
        ("row_offset", ctypes.c_int64), ("npad", ctypes.c_int64),
        ("xg_local", ctypes.c_void_p * 2), ("rank_xg", ctypes.c_void_p),
        ("rank_slices", ctypes.c_void_p), ("rank_arrive", ctypes.c_void_p), ("arrive_local", ctypes.c_void_p),
        ("base", ctypes.c_uint64), ("timeout_ns", ctypes.c_int64),
    ]


class SeriesResult(ctypes.Structure):
    _fields_ = [
        ("matvecs", ctypes.c_int32), ("converged", ctypes.c_int32),
        ("last_term", ctypes.c_double), ("last_pnorm", ctypes.c_double),
        ("passes", ctypes.c_int32), ("reserved", ctypes.c_int32),
    ]


class StepResult(ctypes.Structure):
    _fields_ = [
        ("exp_series", SeriesResult), ("phi1_series", SeriesResult),
        ("status_exp", ctypes.c_int32), ("status_phi1", ctypes.c_int32), ("first_bad", ctypes.c_int64),
        ("gprime_min", ctypes.c_double), ("gprime_max", ctypes.c_double),
        ("lo", ctypes.c_double), ("hi", ctypes.c_double), ("series_ms", ctypes.c_float),
    ]


_lock = threading.Lock()
_lib = None


def _declare(lib):
    vp, i64, i32, d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    sz = ctypes.c_size_t
    P = ctypes.POINTER
    sig = {
        "es_abi_version": ([], ctypes.c_int),
        "es_last_error": ([], ctypes.c_char_p),
        "es_device_available": ([], ctypes.c_int),
        "es_stencil_fused_slab": ([P(StencilDesc), vp, vp, d, d, vp, vp, vp], ctypes.c_int),
        "es_csr_fused_rows": ([i64, i64, vp, vp, vp, vp, vp, d, d, i32, vp], ctypes.c_int),
        "es_combustion_pointwise": ([vp, vp, i64, P(i64), vp], ctypes.c_int),
        "es_leja_stencil_workspace_bytes": ([P(StencilDesc)], sz),
        "es_leja_stencil": ([P(StencilDesc), vp, vp, vp, vp, i32, d, d, d, vp, vp, sz,
                             P(SeriesResult), vp], ctypes.c_int),
        "es_leja_csr_workspace_bytes": ([i64], sz),
        "es_leja_csr": ([i64, vp, vp, vp, vp, vp, vp, vp, i32, d, d, d, vp, sz, P(SeriesResult), vp],
                        ctypes.c_int),
        "es_leja_stencil_async": ([P(StencilDesc), vp, vp, vp, vp, i32, d, d, d, vp, vp, sz, vp], ctypes.c_int),
        "es_leja_fetch": ([vp, P(SeriesResult), vp], ctypes.c_int),
        "es_leja_csr_async": ([i64, vp, vp, vp, vp, vp, vp, vp, i32, d, d, d, vp, sz, vp], ctypes.c_int),
        "es_rosenbrock_prologue": ([P(StencilDesc), vp, vp, vp, P(d), P(i64), vp, vp, vp, vp], ctypes.c_int),
        "es_leja_dist_begin": ([P(StencilDesc), vp, vp, vp, vp, i32, d, d, d, vp, vp, vp, vp, sz, vp], ctypes.c_int),
        "es_leja_dist_source": ([vp, i32, P(vp)], ctypes.c_int),
        "es_leja_dist_nslices": ([vp, P(i32)], ctypes.c_int),
        "es_leja_dist_node": ([vp, vp, vp], ctypes.c_int),
        "es_leja_dist_decide": ([vp, vp, i32, vp], ctypes.c_int),
        "es_leja_dist_end": ([vp, vp], ctypes.c_int),
        "es_leja_state_offset": ([], sz),
        "es_leja_csr_dist_begin": ([i64, vp, vp, vp, vp, i64, vp, vp, vp, vp, i32, d, d, d, vp, sz, vp],
                                   ctypes.c_int),
        "es_leja_csr_dist_source": ([vp, i32, P(vp)], ctypes.c_int),
        "es_csr_fused_rows_z": ([i64, i64, vp, vp, vp, i32, vp, vp, d, d, d, d, i32, vp], ctypes.c_int),
        "es_csr_fused_rows_ex": ([i64, i64, vp, vp, i32, vp, i32, vp, vp, i32, d, d, d, d, i32, vp], ctypes.c_int),
        "es_leja_csr_z_workspace_bytes": ([i64], sz),
        "es_leja_stencil_nslices": ([P(StencilDesc), P(i32)], ctypes.c_int),
        "es_leja_p2p": ([P(StencilDesc), P(P2PDesc), vp, vp, vp, vp, i32, d, d, d, vp, vp, sz, vp], ctypes.c_int),
        "es_ipc_handle": ([vp, vp, P(i64)], ctypes.c_int),
        "es_ipc_open": ([vp, i64, P(vp)], ctypes.c_int),
        "es_ipc_close": ([vp], ctypes.c_int),
        "es_leja_csr_nslices": ([i64, P(i32)], ctypes.c_int),
        "es_stencil_fused_slab_f32": ([P(StencilDesc), vp, vp, d, d, vp, vp, vp, vp, vp], ctypes.c_int),
        "es_combustion_pointwise_f32": ([vp, vp, i64, vp], ctypes.c_int),
        "es_leja_csr_p2p": ([i64, vp, vp, vp, P(P2PRowsDesc), vp, vp, vp, vp, i32, d, d, d, vp, sz, vp], ctypes.c_int),
        "es_leja_csr_z": ([i64, vp, vp, vp, i32, vp, vp, vp, vp, vp, i32, d, d, d, d, vp, sz, P(SeriesResult), vp],
                          ctypes.c_int),
        "es_leja_csr_z_async": ([i64, vp, vp, vp, i32, vp, vp, vp, vp, vp, i32, d, d, d, d, vp, sz, vp],
                                ctypes.c_int),
        "es_leja_csr_dist_nslices": ([vp, P(i32)], ctypes.c_int),
        "es_leja_csr_dist_node": ([vp, vp, vp], ctypes.c_int),
        "es_leja_csr_dist_end": ([vp, vp], ctypes.c_int),
        "es_axpy": ([vp, vp, d, vp, i64, vp], ctypes.c_int),
        "es_scale": ([vp, d, vp, i64, vp], ctypes.c_int),
        "es_half_sum": ([vp, vp, vp, i64, vp], ctypes.c_int),
        "es_combustion_jacobian": ([vp, vp, vp, i64, vp], ctypes.c_int),
        "es_max_abs": ([vp, i64, vp, vp], ctypes.c_int),
        "es_expeuler_step": ([P(StencilDesc), vp, vp, vp, i32, vp, i32, vp, d, d, d, d, i32, vp, vp, vp, vp, sz,
                              P(StepResult), vp], ctypes.c_int),
        "es_exprb_step": ([P(StencilDesc), vp, vp, vp, vp, i32, d, d, d, d, d, d, d, d, vp, vp, vp, sz,
                           P(StepResult), vp], ctypes.c_int),
        "es_exprb_finish": ([P(StencilDesc), vp, vp, vp, vp, i32, d, d, d, d, vp, vp, sz, P(StepResult), vp],
                            ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res


def load(require_device: bool = True):
    """The loaded library; raises when it is missing (no fallback path)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_1309_4616_b200.build` "
                    "(expstencil_b200 has no CPU fallback)"
                )
            lib = ctypes.CDLL(LIB_PATH)
            _declare(lib)
            _lib = lib
    if require_device and not _lib.es_device_available():
        raise RuntimeError("expstencil_b200 needs a CUDA device (B200, sm_100a); none is available")
    return _lib


def last_error() -> str:
    return load(require_device=False).es_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc == ES_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == ES_ERR_ARG:
        raise ValueError(msg)
    if rc == ES_ERR_TYPE:
        raise TypeError(msg)
    if rc == ES_ERR_DOMAIN:
        raise DomainError(msg)
    if rc == ES_ERR_NOT_CONVERGED:
        raise ConvergenceError(msg)
    raise ExpStencilError(msg)
