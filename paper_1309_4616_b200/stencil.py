"""Matrix-free stencil operator A = -laplacian_h on B200 (drop-in for the
reference's stencil.py).

The operator object keeps the reference's surface -- ``StencilOperator``,
``fused_apply_flat(alpha, beta, x)``, ``weights()``, ``coeff_values()``,
``gershgorin_bounds`` (stencil.py:86-155, :315-348) -- but every product runs
in the sm_100a kernels behind ``es_stencil_fused_slab`` / ``es_leja_stencil``.
Host numpy arrays in give host arrays out; CUDA tensors stay on the device.

Boundary kinds: 'none' (periodic), 'homogeneous' (Dirichlet 0), 'function'
(Dirichlet data, plain applies only, as in the reference) and the
build-defined 'neumann' (homogeneous Neumann: the ghost equals the adjacent
interior value, i.e. zero flux across the half cell).
"""

from __future__ import annotations

import ctypes
from typing import Callable, Optional

import numpy as np
import torch

from . import _lib, timing
from .device import Workspace, empty, is_host, like_input, ptr, stream_handle, to_device
from .errors import BoundaryKindError, EvaluationError, GridMismatchError
from .grid import SCALAR_KINDS, Field, Grid3D, eval_on_grid, zeros_field

MODE_ZERO, MODE_PERIODIC, MODE_FACES, MODE_NEUMANN = (
    _lib.ES_MODE_ZERO, _lib.ES_MODE_PERIODIC, _lib.ES_MODE_FACES, _lib.ES_MODE_NEUMANN)

DEFAULT_TILE = (64, 8)  # accepted for signature compatibility; the device tiling is fixed

_MODE_OF_KIND = {"none": MODE_PERIODIC, "homogeneous": MODE_ZERO, "function": MODE_FACES,
                 "neumann": MODE_NEUMANN}


class BoundaryCondition:
    """Boundary tag: 'none' | 'homogeneous' | 'function' | 'neumann'."""

    __slots__ = ("kind", "fn", "text")

    def __init__(self, kind: str, fn: Optional[Callable] = None, text: Optional[str] = None):
        if kind not in _MODE_OF_KIND:
            raise ValueError(f"unknown boundary kind {kind!r}")
        if kind == "function" and fn is None:
            raise ValueError("boundary kind 'function' requires a callable")
        self.kind, self.fn, self.text = kind, fn, text

    @classmethod
    def none(cls):
        return cls("none")

    @classmethod
    def homogeneous(cls):
        return cls("homogeneous")

    @classmethod
    def neumann(cls):
        return cls("neumann")

    @classmethod
    def function(cls, fn: Callable, text: Optional[str] = None):
        return cls("function", fn, text)

    @classmethod
    def from_spec(cls, spec: str):
        s = spec.strip().lower()
        if s == "none":
            return cls.none()
        if s in ("homogeneous", "dirichlet0"):
            return cls.homogeneous()
        if s in ("neumann", "neumann0"):
            return cls.neumann()
        raise ValueError(f"boundary spec {spec!r}: pass expression boundaries as "
                         "BoundaryCondition.function(callable)")

    def label(self) -> str:
        return (self.text or "function") if self.kind == "function" else self.kind

    def __repr__(self):
        return f"BoundaryCondition({self.label()!r})"


class RadialCoefficient:
    """D(x, y, z) = 1/sqrt(1 + x^2 + y^2) (reference bench.py:40-41, the
    paper's position-dependent diffusion).  Operators built with it evaluate
    D inside the kernel instead of streaming a sampled array."""

    es_kind = "radial"

    def __call__(self, x, y, z):
        return 1.0 / np.sqrt(1.0 + x * x + y * y)

    def __repr__(self):
        return "RadialCoefficient()"


radial_coeff = RadialCoefficient()


def _radial_grid(g: Grid3D) -> np.ndarray:
    x = g.axis_coords("x")[None, :]
    y = g.axis_coords("y")[:, None]
    return 1.0 / np.sqrt(1.0 + x * x + y * y)


class StencilOperator:
    """Seven-point operator bound to a grid, a boundary rule and an optional
    positive coefficient D at the output point."""

    def __init__(self, grid: Grid3D, bc: BoundaryCondition, coeff: Optional[Callable] = None,
                 traversal: str = "naive", tile=DEFAULT_TILE, backend: str = "auto"):
        if traversal not in ("naive", "tiled"):
            raise ValueError(f"unknown traversal {traversal!r}")
        self.grid, self.bc, self.coeff = grid, bc, coeff
        self.traversal, self.tile, self.backend = traversal, tile, backend
        self._coeff_cache: dict[str, np.ndarray] = {}
        self._coeff_kind: Optional[int] = None
        self._coeff_dev: dict[int, torch.Tensor] = {}
        self._ws = Workspace()

    @property
    def n(self) -> int:
        return self.grid.n

    def weights(self):
        """Per-axis 1/dx^2, zero for single-point axes (stencil.py:116-122)."""
        g = self.grid
        return tuple(0.0 if m == 1 else 1.0 / (d * d)
                     for m, d in ((g.nx, g.dx), (g.ny, g.dy), (g.nz, g.dz)))

    def coeff_values(self, kind: str = "f64") -> Optional[np.ndarray]:
        if self.coeff is None:
            return None
        if kind not in self._coeff_cache:
            if getattr(self.coeff, "es_kind", None) == "radial":
                vals = np.broadcast_to(_radial_grid(self.grid), self.grid.shape).copy()
            else:
                vals = eval_on_grid(self.grid, self.coeff, kind="f64").values.reshape(self.grid.shape)
            if np.any(vals <= 0.0):
                bad = int(np.argmax(vals.reshape(-1) <= 0.0))
                raise EvaluationError(f"coefficient must be positive; value {vals.reshape(-1)[bad]} at index {bad}")
            self._coeff_cache[kind] = vals.astype(SCALAR_KINDS[kind])
        return self._coeff_cache[kind]

    # -- device descriptors -------------------------------------------------

    def coeff_kind(self) -> int:
        """ES_COEFF_RADIAL when D is (bit-for-bit) the radial coefficient --
        evaluated in-kernel, no extra HBM traffic -- else a staged array.
        Single-plane grids take the radial D as a sampled array too: their
        one-node series kernel is fp64-issue bound on the in-kernel sqrt and
        reciprocal, and streaming D through its TMA ring is faster (4096^2
        Neumann node: 122.5 vs 133.3 us); the values are identical."""
        if self._coeff_kind is None:
            if self.coeff is None:
                self._coeff_kind = _lib.ES_COEFF_NONE
            elif getattr(self.coeff, "es_kind", None) == "radial":
                self._coeff_kind = _lib.ES_COEFF_ARRAY if self.grid.nz == 1 else _lib.ES_COEFF_RADIAL
            else:
                vals = self.coeff_values("f64")
                same = np.array_equal(vals, np.broadcast_to(_radial_grid(self.grid), vals.shape))
                self._coeff_kind = _lib.ES_COEFF_RADIAL if same and self.grid.nz > 1 else _lib.ES_COEFF_ARRAY
        return self._coeff_kind

    def _coeff_device(self, kind: str = "f64") -> torch.Tensor:
        key = (torch.cuda.current_device(), kind)
        if key not in self._coeff_dev:
            vals = self.coeff_values(kind).reshape(-1)
            self._coeff_dev[key] = (to_device(vals) if kind == "f64"
                                    else torch.from_numpy(np.ascontiguousarray(vals)).cuda())
        return self._coeff_dev[key]

    def desc(self, z0: int = 0, lz: Optional[int] = None, faces=None):
        """es_stencil_desc of the slab [z0, z0+lz) plus the tensors it points at."""
        g = self.grid
        lz = g.nz if lz is None else lz
        d = _lib.StencilDesc()
        d.nx, d.ny, d.lz, d.z0, d.nz_total = g.nx, g.ny, lz, z0, g.nz
        d.wx, d.wy, d.wz = self.weights()
        d.mode = _MODE_OF_KIND[self.bc.kind]
        d.coeff_kind = self.coeff_kind()
        keep = []
        if d.coeff_kind == _lib.ES_COEFF_ARRAY:
            c = self._coeff_device()[z0 * g.nx * g.ny:(z0 + lz) * g.nx * g.ny]
            keep.append(c)
            d.coeff = c.data_ptr()
        if faces is not None:
            for i, f in enumerate(faces):
                keep.append(f)
                d.faces[i] = f.data_ptr()
        return d, keep

    # -- flat-vector protocol (stencil.py:142-148) -----------------------------

    def fused_apply_flat(self, alpha, beta, x):
        if self.bc.kind == "function":
            raise BoundaryKindError(
                "fused apply needs a linear operator; use apply_affine_split for "
                "Dirichlet-function boundaries")
        return _fused_flat(self, alpha, beta, x, faces=None)

    def with_traversal(self, traversal: str) -> "StencilOperator":
        return StencilOperator(self.grid, self.bc, self.coeff, traversal, self.tile, self.backend)

    # -- fused Newton-Leja series (matfunc.newton_apply's device path) --------

    def leja_workspace_bytes(self) -> int:
        d, _ = self.desc()
        return int(_lib.load().es_leja_stencil_workspace_bytes(ctypes.byref(d)))

    def _leja(self, v: torch.Tensor, p_out: torch.Tensor, dd: torch.Tensor, xi: torch.Tensor,
              alpha: float, shift: float, tol: float, gdiag: Optional[torch.Tensor] = None):
        lib = _lib.load()
        d, keep = self.desc()
        nbytes = lib.es_leja_stencil_workspace_bytes(ctypes.byref(d))
        ws = self._ws.get(nbytes)
        tm = timing.active()
        ev0 = timing.event() if tm else None
        rc = lib.es_leja_stencil_async(ctypes.byref(d), ptr(v), ptr(p_out), ptr(dd), ptr(xi), dd.numel(),
                                       float(alpha), float(shift), float(tol), ptr(gdiag), ptr(ws),
                                       ws.numel(), stream_handle())
        _lib.check(rc, "es_leja_stencil_async")
        ev1 = timing.event() if tm else None
        res = _lib.SeriesResult()
        rc = lib.es_leja_fetch(ptr(ws), ctypes.byref(res), stream_handle())
        if rc != _lib.ES_ERR_NOT_CONVERGED:
            _lib.check(rc, "es_leja_fetch")
        if tm:
            tm.add(ev0, ev1, res.matvecs, res.passes)
        del keep
        return res

    def two_node_passes(self) -> bool:
        """Whether series on this operator run two Leja nodes per HBM pass
        (csrc/stencil_tb.cuh; the C side decides, this mirrors its rule for
        the bench's launch counts and roofline)."""
        import os

        g = self.grid
        base = (os.environ.get("ES_TB", "1") != "0" and g.nx % 2 == 0
                and self.bc.kind in ("homogeneous", "neumann") and os.environ.get("ES_KERNEL", "") != "v1")
        if g.nz > 1:
            return base
        # single-plane grids (stencil_tb2d.cuh): not where the persistent
        # small-grid series takes over (series_small.cu)
        small = os.environ.get("ES_SMALL", "1") != "0" and g.nx <= 512 and g.nx * g.ny <= (1 << 20)
        return base and os.environ.get("ES_TB2D", "1") != "0" and not small

    def __repr__(self):
        g = self.grid
        return (f"StencilOperator({g.nx}x{g.ny}x{g.nz}, bc={self.bc.label()!r}, "
                f"coeff={'yes' if self.coeff else 'no'}, device='b200')")


def kind_dtype(kind: str):
    return SCALAR_KINDS[kind]


def _face_sample(fn, x, y, z) -> np.ndarray:
    shape = np.broadcast(x, y, z).shape
    try:
        vals = np.asarray(fn(x, y, z), dtype=np.float64)
        return vals if vals.shape == shape else np.broadcast_to(vals, shape).copy()
    except (TypeError, ValueError):
        bx, by, bz = np.broadcast_arrays(x, y, z)
        return np.vectorize(lambda a, b, c: float(fn(a, b, c)))(bx, by, bz)


def boundary_faces(op: StencilOperator, dtype=np.float64):
    """Dirichlet data on the six faces (stencil.py:179-204 layout): fx_* are
    (nz, ny), fy_* (nz, nx), fz_* (ny, nx)."""
    g, fn = op.grid, op.bc.fn
    xc, yc, zc = g.axis_coords("x"), g.axis_coords("y"), g.axis_coords("z")
    z_ny, y_ny = np.meshgrid(zc, yc, indexing="ij")
    z_nx, x_nx = np.meshgrid(zc, xc, indexing="ij")
    y_xy, x_xy = np.meshgrid(yc, xc, indexing="ij")
    faces = (_face_sample(fn, 0.0, y_ny, z_ny), _face_sample(fn, 1.0, y_ny, z_ny),
             _face_sample(fn, x_nx, 0.0, z_nx), _face_sample(fn, x_nx, 1.0, z_nx),
             _face_sample(fn, x_xy, y_xy, 0.0), _face_sample(fn, x_xy, y_xy, 1.0))
    for name, f in zip(("x=0", "x=1", "y=0", "y=1", "z=0", "z=1"), faces):
        if not np.all(np.isfinite(f)):
            raise EvaluationError(f"non-finite boundary evaluation on face {name}")
    return tuple(np.ascontiguousarray(f, dtype=dtype) for f in faces)


def fused_slab(op: StencilOperator, alpha, beta, x3, out3, halo_lo=None, halo_hi=None, z0: int = 0,
               faces=None) -> None:
    """One slab through es_stencil_fused_slab (device tensors; the
    decomposition layer's entry point, stencil.py:207-243)."""
    kind = op.bc.kind
    lz = int(x3.numel()) // (op.grid.nx * op.grid.ny)
    if kind == "none" and (z0 != 0 or lz != op.grid.nz):
        raise BoundaryKindError("periodic wraparound is not defined on a partitioned slab")
    if kind == "function" and faces is None:
        raise BoundaryKindError("Dirichlet-function apply needs precomputed face values")
    if x3.dtype == torch.float32:
        return _fused_slab_f32(op, alpha, beta, x3, out3, halo_lo, halo_hi, z0, lz, faces)
    dfaces = None if faces is None else [to_device(np.asarray(f).reshape(-1)) for f in faces]
    d, keep = op.desc(z0=z0, lz=lz, faces=dfaces)
    rc = _lib.load().es_stencil_fused_slab(ctypes.byref(d), ptr(x3), ptr(out3), float(alpha), float(beta),
                                           ptr(halo_lo), ptr(halo_hi), stream_handle())
    _lib.check(rc, "es_stencil_fused_slab")
    del keep


def _fused_slab_f32(op: StencilOperator, alpha, beta, x3, out3, halo_lo, halo_hi, z0, lz, faces) -> None:
    """Single precision, like the reference's `_stencil_impl[float]`
    (weights / alpha / beta cast to float, float arithmetic throughout)."""
    g = op.grid
    d, _ = op.desc(z0=z0, lz=lz)
    coeff = None
    if op.coeff is not None:
        coeff = op._coeff_device("f32")[z0 * g.nx * g.ny:(z0 + lz) * g.nx * g.ny]
    keep = []
    face_ptrs = None
    if faces is not None:
        keep = [torch.from_numpy(np.ascontiguousarray(f, dtype=np.float32).reshape(-1)).cuda() for f in faces]
        table = (ctypes.c_void_p * 6)(*[f.data_ptr() for f in keep])  # host array of 6 device pointers
        keep.append(table)
        face_ptrs = ctypes.cast(table, ctypes.c_void_p)
    rc = _lib.load().es_stencil_fused_slab_f32(ctypes.byref(d), ptr(x3), ptr(out3), float(alpha), float(beta),
                                               ptr(coeff), face_ptrs, ptr(halo_lo), ptr(halo_hi), stream_handle())
    _lib.check(rc, "es_stencil_fused_slab_f32")
    del keep


def _fused_flat(op: StencilOperator, alpha, beta, x, faces):
    g = op.grid
    host = is_host(x)
    shape = tuple(x.shape)
    if shape != (g.n,):
        raise GridMismatchError(f"vector length {shape} does not match grid n={g.n}")
    if (np.iscomplexobj(x) if host else x.is_complex()):
        re = _fused_flat(op, 1.0, 0.0, x.real.copy() if host else x.real.contiguous(), faces)
        im = _fused_flat(op, 1.0, 0.0, x.imag.copy() if host else x.imag.contiguous(), faces)
        return alpha * (re + 1j * im) + beta * x
    f32 = (np.asarray(x).dtype == np.float32) if host else x.dtype == torch.float32
    if f32:  # the reference's float kernel: float in, float out
        xd = torch.from_numpy(np.ascontiguousarray(x)).cuda() if host else x.contiguous()
        out = torch.empty(g.n, dtype=torch.float32, device=xd.device)
    elif not host and x.dtype != torch.float64 or host and np.asarray(x).dtype != np.float64:
        raise TypeError(f"stencil kernels support f32/f64, got {x.dtype}")
    else:
        xd = to_device(x)
        out = empty(g.n)
    fused_slab(op, alpha, beta, xd, out, faces=faces)
    return like_input(out, host)


def apply(op: StencilOperator, u: Field) -> Field:
    """A u with the operator's boundary handling (faces evaluated per call)."""
    if u.grid != op.grid:
        raise GridMismatchError("field is bound to a different grid")
    faces = None
    if op.bc.kind == "function":
        if (np.iscomplexobj(u.values) if is_host(u.values) else u.values.is_complex()):
            raise BoundaryKindError("Dirichlet-function boundaries are real-valued")
        faces = boundary_faces(op, np.float32 if u.kind == "f32" else np.float64)
    return Field(u.grid, _fused_flat(op, 1.0, 0.0, u.values, faces))


def fused_apply(op: StencilOperator, alpha, beta, x: Field) -> Field:
    if x.grid != op.grid:
        raise GridMismatchError("field is bound to a different grid")
    return Field(x.grid, op.fused_apply_flat(alpha, beta, x.values))


def homogeneous_part(op: StencilOperator) -> StencilOperator:
    return StencilOperator(op.grid, BoundaryCondition.homogeneous(), op.coeff, op.traversal, op.tile,
                           op.backend)


def boundary_source_field(op: StencilOperator, kind: str = "f64") -> Field:
    """b = A(0) of a Dirichlet-function operator."""
    if op.bc.kind != "function":
        raise BoundaryKindError("boundary source requires a Dirichlet-function boundary")
    zero = zeros_field(op.grid, kind=kind)
    faces = boundary_faces(op, np.float32 if kind == "f32" else np.float64)
    return Field(op.grid, _fused_flat(op, 1.0, 0.0, zero.values, faces))


def apply_affine_split(op: StencilOperator, u: Field):
    """A u = A_hom u + b for Dirichlet-function boundaries (stencil.py:281-296)."""
    if op.bc.kind != "function":
        raise BoundaryKindError("apply_affine_split requires a Dirichlet-function boundary")
    if u.grid != op.grid:
        raise GridMismatchError("field is bound to a different grid")
    hom = Field(u.grid, _fused_flat(homogeneous_part(op), 1.0, 0.0, u.values, None))
    return hom, boundary_source_field(op, u.kind)


def gershgorin_bounds(op: StencilOperator, gdiag_range=None):
    """Gershgorin interval of the (linear) stencil matrix, per-row centres and
    radii from the neighbour counts, scaled by D (stencil.py:315-348).  Under
    Neumann every row's diagonal equals its off-diagonal mass (lower end 0).
    ``gdiag_range=(lo, hi)`` shifts it for A - diag(g')."""
    if op.bc.kind == "function":
        raise BoundaryKindError("spectral bounds are defined for the linear operator")
    g = op.grid
    w = op.weights()
    periodic = op.bc.kind == "none"

    def counts(m):
        c = np.full(m, 2.0)
        if not periodic and m >= 2:
            c[0] = c[-1] = 1.0
        return c

    cx, cy, cz = counts(g.nx), counts(g.ny), counts(g.nz)
    neumann = op.bc.kind == "neumann"
    d = op.coeff_values("f64") if op.coeff_kind() == _lib.ES_COEFF_ARRAY else None
    if d is None:
        # rounding is monotone, so the z-extreme of fl(fl(r_xy) + wz*cz) is
        # reached at the largest wz*cz: exact without the (nz, ny, nx) array
        r_xy = w[0] * cx[None, :] + w[1] * cy[:, None]
        radius = r_xy + np.max(w[2] * cz)
    else:
        radius = w[0] * cx[None, None, :] + w[1] * cy[None, :, None] + w[2] * cz[:, None, None]
    centre = radius if neumann else 2.0 * (w[0] + w[1] + w[2])
    lo_rows, hi_rows = centre - radius, centre + radius
    if d is None and op.coeff is not None:  # z-invariant radial D(x, y)
        d = _radial_grid(g)
    if d is not None:
        lo, hi = float(np.min(d * lo_rows)), float(np.max(d * hi_rows))
    else:
        lo, hi = float(np.min(lo_rows)), float(np.max(hi_rows))
    if gdiag_range is not None:
        lo, hi = lo - float(gdiag_range[1]), hi - float(gdiag_range[0])
    return lo, hi
