"""Kernel backend "b200" for the reference package ``expstencil``.

The reference resolves its kernel module in ``_kernels.get_kernels(backend)``
(reference ``pkg/src/expstencil/_kernels.py:43-53``) and lists the choices in
``available_backends()`` (``:39-40``).  A module with ``backend_name``,
``MODE_*``, ``stencil_fused_slab``, ``csr_fused``, ``csr_fused_rows`` and
``combustion_pointwise`` (the protocol ``_core.pyx:176-348`` implements) is a
backend.  This file is that module for the B200 library: every call goes
through the C ABI of ``include/expstencil_b200.h``
(``libexpstencil_b200.so``) -- there is no CPU path here.

Use (what a maintainer adds to ``_kernels.py``, or what a test does)::

    import expstencil
    import expstencil_b200_backend as b200
    b200.install(expstencil._kernels)       # adds "b200" to the seam
    op = expstencil.StencilOperator(grid, bc, backend="b200")

Semantics match the compiled core: f64 and f32 slabs (float arithmetic for
float data, weights / alpha / beta rounded to float), halos, z0 / nz_total,
sampled coefficients, Dirichlet faces; CSR rows for every dtype combination
of ``_core.csr_fused_rows`` plus int64 columns, summed in storage order;
combustion without a domain check (the caller checks, integrator.py:45-50).
``traversal`` / ``tile`` select a loop order on the CPU; the device has one
order and the results are traversal-invariant bit for bit (the reference's
own contract, tests/test_stencil.py:134-145), so they are accepted and
validated but do not change the result.  Arguments may be numpy arrays
(copied to and from the device per call) or CUDA tensors (used in place).
"""

from __future__ import annotations

import ctypes
import os
import sys
import types

import numpy as np
import torch

_REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if _REPO not in sys.path:
    sys.path.insert(0, _REPO)

from paper_1309_4616_b200 import _lib  # noqa: E402

backend_name = "b200"

MODE_ZERO = 0
MODE_PERIODIC = 1
MODE_FACES = 2

_TORCH = {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32,
          np.dtype(np.complex128): torch.complex128, np.dtype(np.int32): torch.int32,
          np.dtype(np.int64): torch.int64}
_KIND = {torch.float32: _lib.ES_KIND_F32, torch.float64: _lib.ES_KIND_F64, torch.complex128: _lib.ES_KIND_C128}


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _dev(a, dtype=None):
    """CUDA tensor for a numpy array or tensor (no copy for a contiguous CUDA
    tensor of the right dtype)."""
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        t = a if a.is_cuda else a.cuda()
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        return t.contiguous()
    arr = np.ascontiguousarray(a)
    if dtype is not None:
        arr = np.ascontiguousarray(arr, dtype={v: k for k, v in _TORCH.items()}[dtype])
    if arr.dtype not in _TORCH:
        raise TypeError(f"b200 kernels do not support dtype {arr.dtype}")
    return torch.from_numpy(arr).cuda()


def _dtype_of(a):
    return a.dtype if isinstance(a, torch.Tensor) else _TORCH.get(np.asarray(a).dtype)


def _write_back(dst, src: torch.Tensor, rows=None) -> None:
    if isinstance(dst, torch.Tensor):
        if rows is None:
            dst.copy_(src.view(dst.shape))
        else:
            dst.view(-1)[rows[0]:rows[1]].copy_(src[rows[0]:rows[1]])
        return
    host = src.cpu().numpy()
    if rows is None:
        dst[...] = host.reshape(dst.shape)
    else:
        dst[rows[0]:rows[1]] = host[rows[0]:rows[1]]


def _check_traversal(traversal, tile) -> None:
    if traversal not in ("naive", "tiled"):
        raise ValueError(f"unknown traversal {traversal!r}")
    if len(tuple(tile)) != 2:
        raise ValueError("tile must be a (tx, ty) pair")


def stencil_fused_slab(u3, out3, alpha, beta, weights, mode, faces=None, halo_lo=None, halo_hi=None, z0=0,
                       nz_total=None, coeff3=None, traversal="naive", tile=(64, 8)):
    """out3 = alpha * (D A u3) + beta * u3 on one z-slab (_core.pyx:176-226)."""
    _check_traversal(traversal, tile)
    dt = _dtype_of(u3)
    if dt not in (torch.float64, torch.float32):
        raise TypeError(f"b200 stencil kernel supports f32/f64, got {getattr(u3, 'dtype', type(u3))}")
    lz, ny, nx = (int(s) for s in u3.shape)
    d = _lib.StencilDesc()
    d.nx, d.ny, d.lz, d.z0 = nx, ny, lz, int(z0)
    d.nz_total = lz if nz_total is None else int(nz_total)
    d.wx, d.wy, d.wz = (float(w) for w in weights)
    d.mode = int(mode)
    u = _dev(u3, dt)
    out = torch.empty(u.numel(), dtype=dt, device=u.device)
    hl, hh = _dev(halo_lo, dt), _dev(halo_hi, dt)
    keep = [u, out, hl, hh]
    c = _dev(coeff3, dt)
    fdev = None if faces is None else [_dev(f, dt) for f in faces]
    p = lambda t: None if t is None else t.data_ptr()  # noqa: E731
    if dt == torch.float64:
        if c is not None:
            d.coeff_kind, d.coeff = _lib.ES_COEFF_ARRAY, c.data_ptr()
        if fdev is not None:
            for i, f in enumerate(fdev):
                d.faces[i] = f.data_ptr()
        rc = _lib.load().es_stencil_fused_slab(ctypes.byref(d), p(u), p(out), float(alpha), float(beta), p(hl),
                                               p(hh), _stream())
    else:
        table = None
        if fdev is not None:
            table = (ctypes.c_void_p * 6)(*[f.data_ptr() for f in fdev])  # host array of device pointers
        d.coeff_kind = _lib.ES_COEFF_NONE
        rc = _lib.load().es_stencil_fused_slab_f32(ctypes.byref(d), p(u), p(out), float(alpha), float(beta), p(c),
                                                   None if table is None else ctypes.cast(table, ctypes.c_void_p),
                                                   p(hl), p(hh), _stream())
    _lib.check(rc, "b200 stencil_fused_slab")
    _write_back(out3, out)
    del keep, c, fdev


def csr_fused_rows(row_lo, row_hi, row_ptr, col_idx, vals, x, y, alpha, beta, use_beta):
    """y[row_lo:row_hi] = alpha (A x)[rows] (+ beta x[rows]) (_core.pyx:281-315)."""
    row_lo, row_hi = int(row_lo), int(row_hi)
    if row_hi <= row_lo:
        return
    vt, xt = _dtype_of(vals), _dtype_of(x)
    if xt not in _KIND or vt not in _KIND:
        raise TypeError(f"b200 CSR kernel does not support vals={vt}, x={xt}")
    if vt == torch.float32 and xt != torch.float32:
        vt = torch.float64  # exact widening; the product then rounds like the f64 / complex kernels
    ct = _dtype_of(col_idx)
    if ct not in (torch.int32, torch.int64):
        raise TypeError(f"b200 CSR kernel needs int32/int64 column indices, got {ct}")
    rp = _dev(row_ptr, torch.int64)
    ci = _dev(col_idx, ct)
    va = _dev(vals, vt)
    xd = _dev(x, xt)
    yd = torch.empty_like(xd) if (xd.numel() == _len(y)) else torch.empty(_len(y), dtype=xt, device=xd.device)
    a, b = complex(alpha), complex(beta)
    rc = _lib.load().es_csr_fused_rows_ex(row_lo, row_hi, rp.data_ptr(), ci.data_ptr(), 4 if ct == torch.int32 else 8,
                                          va.data_ptr(), _KIND[vt], xd.data_ptr(), yd.data_ptr(), _KIND[xt],
                                          a.real, a.imag, b.real, b.imag, int(bool(use_beta)), _stream())
    _lib.check(rc, "b200 csr_fused_rows")
    _write_back(y, yd, rows=(row_lo, row_hi))


def _len(a) -> int:
    return int(a.numel()) if isinstance(a, torch.Tensor) else int(np.asarray(a).shape[0])


def csr_fused(nrows, row_ptr, col_idx, vals, x, y, alpha, beta, use_beta):
    csr_fused_rows(0, nrows, row_ptr, col_idx, vals, x, y, alpha, beta, use_beta)


def combustion_pointwise(u, out):
    """out = (2 - u)/4 exp(20 (1 - 1/u)) (_core.pyx:323-348); like the core,
    no domain check here -- the caller (combustion_g) checks u > 0."""
    dt = _dtype_of(u)
    if dt not in (torch.float64, torch.float32):
        raise TypeError(f"b200 combustion kernel supports f32/f64, got {getattr(u, 'dtype', type(u))}")
    ud = _dev(u, dt)
    od = torch.empty_like(ud)
    lib = _lib.load()
    if dt == torch.float64:
        bad = ctypes.c_int64(-1)
        rc = lib.es_combustion_pointwise(ud.data_ptr(), od.data_ptr(), ud.numel(), ctypes.byref(bad), _stream())
        if rc == _lib.ES_ERR_DOMAIN:  # values are written for every point; the caller owns the check
            rc = _lib.ES_OK
    else:
        rc = lib.es_combustion_pointwise_f32(ud.data_ptr(), od.data_ptr(), ud.numel(), _stream())
    _lib.check(rc, "b200 combustion_pointwise")
    _write_back(out, od)


def install(kernels_module: types.ModuleType, default: bool = False) -> None:
    """Register this module as backend "b200" in the reference's
    ``expstencil._kernels`` (idempotent).  ``get_kernels("b200")`` returns it
    and ``available_backends()`` lists it after the reference's own; with
    ``default=True`` it also becomes what ``"auto"`` resolves to, so every
    operator, CSR product, partitioned wrapper and nonlinearity of the
    reference runs on the B200 kernels (``uninstall`` restores the seam)."""
    if default:
        kernels_module._b200_saved_default = getattr(kernels_module, "_b200_saved_default",
                                                     kernels_module._DEFAULT)
        kernels_module._DEFAULT = "b200"
    if getattr(kernels_module, "_b200_installed", False):
        return
    me = sys.modules[__name__]
    orig_get, orig_avail = kernels_module.get_kernels, kernels_module.available_backends

    def get_kernels(backend: str = "auto"):
        if backend in (None, "auto"):
            backend = kernels_module._DEFAULT
        if backend == "b200":
            return me
        return orig_get(backend)

    def available_backends() -> tuple:
        return tuple(orig_avail()) + ("b200",)

    get_kernels.__doc__ = orig_get.__doc__
    kernels_module._b200_orig = (orig_get, orig_avail)
    kernels_module.get_kernels = get_kernels
    kernels_module.available_backends = available_backends
    kernels_module._b200_installed = True


def uninstall(kernels_module: types.ModuleType) -> None:
    if not getattr(kernels_module, "_b200_installed", False):
        return
    kernels_module.get_kernels, kernels_module.available_backends = kernels_module._b200_orig
    if hasattr(kernels_module, "_b200_saved_default"):
        kernels_module._DEFAULT = kernels_module._b200_saved_default
        del kernels_module._b200_saved_default
    kernels_module._b200_installed = False
