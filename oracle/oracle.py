"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A CPU restatement of the reference's hot path (arXiv 1309.4616 reference,
package ``expstencil``): the per-point stencil arithmetic, the Newton-Leja
series, CSR rows, and the combustion nonlinearity live in plain C
(``oracle.c``, built by ``oracle/Makefile``); the host-side interpolant set-up
(Leja nodes, divided differences) and the integrator step composition are
restated here in numpy with the reference's operation order.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module, and only as the checker / CPU baseline.  The product
(``paper_1309_4616_b200``) never imports it.

Pinned by ``tests/test_oracle_golden.py`` against fixtures the reference
itself produced (``tests/golden/make_golden.py``).  Neumann ghosts and the
exponential Rosenbrock step are build-defined (no reference counterpart) and
pinned against dense-matrix oracles only.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")

MODE_ZERO, MODE_PERIODIC, MODE_FACES, MODE_NEUMANN = 0, 1, 2, 3
COEFF_NONE, COEFF_RADIAL, COEFF_ARRAY = 0, 1, 2

_dp = ctypes.POINTER(ctypes.c_double)


class _Slab(ctypes.Structure):
    _fields_ = [
        ("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("lz", ctypes.c_int64),
        ("z0", ctypes.c_int64), ("nz_total", ctypes.c_int64),
        ("wx", ctypes.c_double), ("wy", ctypes.c_double), ("wz", ctypes.c_double),
        ("mode", ctypes.c_int32), ("coeff_kind", ctypes.c_int32),
        ("coeff", _dp), ("faces", _dp * 6),
        ("halo_lo", _dp), ("halo_hi", _dp), ("gdiag", _dp),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
        i64, i32, d = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        vp = ctypes.c_void_p
        _lib.orc_stencil_fused_slab.argtypes = [vp, vp, vp, d, d]
        _lib.orc_newton_stencil.argtypes = [vp, vp, vp, vp, vp, i32, d, d, d, vp, vp, vp, vp]
        _lib.orc_newton_stencil.restype = ctypes.c_int
        _lib.orc_csr_fused_rows.argtypes = [i64, i64, vp, vp, vp, vp, vp, d, d, ctypes.c_int]
        _lib.orc_newton_csr.argtypes = [i64, vp, vp, vp, vp, vp, vp, vp, i32, d, d, d, vp, vp, vp, vp]
        _lib.orc_newton_csr.restype = ctypes.c_int
        _lib.orc_csr_fused_rows_z.argtypes = [i64, i64, vp, vp, vp, ctypes.c_int, vp, vp, d, d, d, d, ctypes.c_int]
        _lib.orc_newton_csr_z.argtypes = [i64, vp, vp, vp, ctypes.c_int, vp, vp, vp, vp, vp, i32, d, d, d, d, vp,
                                          vp, vp, vp]
        _lib.orc_newton_csr_z.restype = ctypes.c_int
        _lib.orc_combustion.argtypes = [vp, vp, i64]
        _lib.orc_combustion.restype = i64
        _lib.orc_combustion_jac.argtypes = [vp, vp, i64]
        _lib.orc_axpy_step.argtypes = [vp, vp, d, vp, i64]
        _lib.orc_num_threads.restype = ctypes.c_int
    return _lib


def build() -> None:
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def num_threads() -> int:
    return int(lib().orc_num_threads())


# ---------------------------------------------------------------------------
# Stencil geometry (grid.py:36-93, stencil.py:116-122, :315-348)


@dataclass
class StencilSpec:
    nx: int
    ny: int
    nz: int
    mode: int = MODE_ZERO
    coeff_kind: int = COEFF_NONE
    coeff: Optional[np.ndarray] = None  # (nz, ny, nx) for COEFF_ARRAY
    faces: Optional[tuple] = None

    @property
    def n(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def shape(self):
        return (self.nz, self.ny, self.nx)

    def weights(self):
        def w(m):
            d = 1.0 / (m + 1)
            return 0.0 if m == 1 else 1.0 / (d * d)

        return (w(self.nx), w(self.ny), w(self.nz))

    def coeff_grid(self) -> Optional[np.ndarray]:
        """D sampled on the grid the way eval_on_grid would (grid.py:145-172)."""
        if self.coeff_kind == COEFF_ARRAY:
            return self.coeff
        if self.coeff_kind != COEFF_RADIAL:
            return None
        x = np.arange(1, self.nx + 1, dtype=np.float64) / (self.nx + 1)
        y = np.arange(1, self.ny + 1, dtype=np.float64) / (self.ny + 1)
        d2 = 1.0 / np.sqrt(1.0 + x[None, :] * x[None, :] + y[:, None] * y[:, None])
        return np.broadcast_to(d2, self.shape).copy()

    def gershgorin(self, gdiag: Optional[np.ndarray] = None):
        """Analytic Gershgorin interval; Neumann rows lose one neighbour per
        boundary face they touch (build-defined)."""
        wx, wy, wz = self.weights()
        periodic = self.mode == MODE_PERIODIC
        neumann = self.mode == MODE_NEUMANN

        def counts(n):
            c = np.full(n, 2.0)
            if not periodic and n >= 2:
                c[0] = c[-1] = 1.0
            return c

        ex, ey, ez = counts(self.nx), counts(self.ny), counts(self.nz)
        radius = wx * ex[None, None, :] + wy * ey[None, :, None] + wz * ez[:, None, None]
        if neumann:
            center = radius  # diagonal == off-diagonal mass on every row
        else:
            center = np.full(radius.shape, 2.0 * (wx + wy + wz))
        d = self.coeff_grid()
        lo_rows = center - radius
        hi_rows = center + radius
        if d is not None:
            lo_rows = d * lo_rows
            hi_rows = d * hi_rows
        if gdiag is not None:
            g3 = gdiag.reshape(self.shape)
            lo_rows = lo_rows - g3
            hi_rows = hi_rows - g3
        return float(np.min(lo_rows)), float(np.max(hi_rows))


def _slab(spec: StencilSpec, z0=0, lz=None, halo_lo=None, halo_hi=None, gdiag=None, coeff=None):
    wx, wy, wz = spec.weights()
    s = _Slab()
    s.nx, s.ny = spec.nx, spec.ny
    s.lz = spec.nz if lz is None else lz
    s.z0, s.nz_total = z0, spec.nz
    s.wx, s.wy, s.wz = wx, wy, wz
    s.mode, s.coeff_kind = spec.mode, spec.coeff_kind
    keep = []
    if spec.coeff_kind == COEFF_ARRAY:
        c = np.ascontiguousarray(coeff if coeff is not None else spec.coeff, dtype=np.float64)
        keep.append(c)
        s.coeff = _ptr(c)
    if spec.faces is not None:
        for i, f in enumerate(spec.faces):
            f = np.ascontiguousarray(f, dtype=np.float64)
            keep.append(f)
            s.faces[i] = _ptr(f)
    for name, arr in (("halo_lo", halo_lo), ("halo_hi", halo_hi), ("gdiag", gdiag)):
        if arr is not None:
            arr = np.ascontiguousarray(arr, dtype=np.float64)
            keep.append(arr)
            setattr(s, name, _ptr(arr))
    return s, keep


def stencil_fused(spec: StencilSpec, alpha, beta, x: np.ndarray, gdiag=None, **slab_kw) -> np.ndarray:
    """out = alpha * (D A x [- g' x]) + beta * x (restates _core.pyx:176-226)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    s, keep = _slab(spec, gdiag=gdiag, lz=x.size // (spec.nx * spec.ny), **slab_kw)
    lib().orc_stencil_fused_slab(ctypes.byref(s), _ptr(x), _ptr(out), float(alpha), float(beta))
    return out


# ---------------------------------------------------------------------------
# Interpolant set-up (matfunc.py:31-268), numpy in the reference's op order


_PHI1_COEFF = [1.0 / math.factorial(k + 1) for k in range(8)]


def phi1_scalar(z):
    """matfunc.py:46-71 (real or complex scalar)."""
    z = complex(z) if isinstance(z, complex) or np.iscomplexobj(z) else float(z)
    if abs(z) <= 1e-2:
        zz = np.asarray([z])
        acc = np.full_like(zz, _PHI1_COEFF[7])
        for c in reversed(_PHI1_COEFF[:7]):
            acc = acc * zz + c
        return acc[0]
    if isinstance(z, complex):
        x, y = z.real, z.imag
        em1 = complex(np.expm1(x) * np.cos(y) - 2.0 * np.sin(0.5 * y) ** 2, np.exp(x) * np.sin(y))
        return em1 / z
    return np.float64(np.expm1(np.float64(z)) / np.float64(z))


class _Leja:
    """Canonical Leja sequence on [-2, 2] (matfunc.py:125-153)."""

    def __init__(self, size=100001):
        self.grid = np.linspace(-2.0, 2.0, size)
        self.pts = [2.0]
        self.sep = np.abs(self.grid - 2.0)

    def get(self, count):
        while len(self.pts) < count:
            j = int(np.argmax(self.sep))
            x = float(self.grid[j])
            self.pts.append(x)
            self.sep *= np.abs(self.grid - x)
        return np.array(self.pts[:count])


_LEJA = _Leja()


def canonical_leja(count: int) -> np.ndarray:
    return _LEJA.get(count)


def _bidiag_first_column(diag, sub, target):
    """matfunc.py:169-208: Taylor(30) + scaling and squaring."""
    m = len(diag)
    cplx = np.iscomplexobj(diag) or np.iscomplexobj(np.asarray(sub))
    z = np.zeros((m, m), dtype=np.complex128 if cplx else np.float64)
    z[np.arange(m), np.arange(m)] = diag
    if m > 1:
        z[np.arange(1, m), np.arange(m - 1)] = sub
    nrm = np.linalg.norm(z, 1)
    s = 0 if nrm <= 1.0 else int(math.ceil(math.log2(nrm)))
    zs = z / (2.0 ** s)
    eye = np.eye(m, dtype=zs.dtype)
    e, p, te, tp = eye.copy(), eye.copy(), eye.copy(), eye.copy()
    for k in range(1, 31):
        te = (te @ zs) / k
        e += te
        tp = (tp @ zs) / (k + 1)
        p += tp
    for _ in range(s):
        p = 0.5 * (p + e @ p)
        e = e @ e
    f = e if target == "exp" else p
    if not np.all(np.isfinite(f)):
        raise OverflowError("divided differences overflowed")
    return f[:, 0].copy()


@dataclass
class Interp:
    a: float
    b: float
    target: str
    scale: float
    xi: np.ndarray
    dd: np.ndarray

    @property
    def gamma(self):
        return 0.25 * (self.b - self.a)

    @property
    def center(self):
        return 0.5 * (self.a + self.b)


def interpolant(a: float, b: float, target: str, scale: float, max_degree: int = 150) -> Interp:
    """matfunc.make_interpolant (real axis) restated."""
    if a == b:
        f0 = np.exp(scale * a) if target == "exp" else phi1_scalar(scale * a)
        return Interp(a, b, target, scale, np.zeros(1), np.array([f0]))
    xi = canonical_leja(max_degree + 1)
    center, half = 0.5 * (a + b), 0.25 * (b - a)
    nodes = center + half * xi
    dd = _bidiag_first_column(scale * nodes, scale * half, target)
    dd[0] = np.exp(scale * nodes[0]) if target == "exp" else phi1_scalar(scale * nodes[0])
    return Interp(a, b, target, scale, xi, dd)


# ---------------------------------------------------------------------------
# Series and steps


class OracleConvergenceError(Exception):
    def __init__(self, residual, degree):
        super().__init__(f"not converged (degree {degree})")
        self.residual = residual
        self.degree = degree


def newton_stencil(spec: StencilSpec, it: Interp, v: np.ndarray, tol: float, gdiag=None):
    """matfunc.newton_apply on the stencil; returns (p, matvecs)."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    n = v.size
    p = np.empty_like(v)
    if len(it.dd) == 1:
        return it.dd[0] * v, 0
    ws = np.empty(2 * n + spec.nz, dtype=np.float64)
    mv = ctypes.c_int32()
    term = ctypes.c_double()
    pn = ctypes.c_double()
    s, keep = _slab(spec, gdiag=gdiag)
    gamma = it.gamma
    shift = it.center / gamma
    rc = lib().orc_newton_stencil(
        ctypes.byref(s), _ptr(v), _ptr(p), _ptr(np.ascontiguousarray(it.dd)), _ptr(it.xi),
        len(it.dd), 1.0 / gamma, shift, float(tol), _ptr(ws),
        ctypes.byref(mv), ctypes.byref(term), ctypes.byref(pn))
    if rc == 2:
        ref = pn.value
        raise OracleConvergenceError(term.value / ref if ref > 0 else float("inf"), mv.value)
    return p, mv.value


@dataclass
class Csr:
    n: int
    row_ptr: np.ndarray
    col: np.ndarray
    vals: np.ndarray

    def gershgorin(self):
        rows = np.repeat(np.arange(self.n), np.diff(self.row_ptr))
        diag = np.zeros(self.n)
        hit = rows == self.col
        diag[rows[hit]] = self.vals[hit]
        a = np.abs(self.vals)
        sums = np.add.reduceat(np.concatenate([a, [0.0]]), self.row_ptr[:-1])
        sums[self.row_ptr[1:] == self.row_ptr[:-1]] = 0.0
        radius = np.maximum(sums - np.abs(diag), 0.0)
        return float(np.min(diag - radius)), float(np.max(diag + radius))


def csr_fused(a: Csr, alpha, beta, x, use_beta=True):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(a.n)
    lib().orc_csr_fused_rows(0, a.n, a.row_ptr.ctypes.data, a.col.ctypes.data, a.vals.ctypes.data,
                             x.ctypes.data, y.ctypes.data, float(alpha), float(beta), int(use_beta))
    return y


def newton_csr(a: Csr, it: Interp, v: np.ndarray, tol: float):
    v = np.ascontiguousarray(v, dtype=np.float64)
    if len(it.dd) == 1:
        return it.dd[0] * v, 0
    p = np.empty_like(v)
    ws = np.empty(2 * a.n)
    mv, term, pn = ctypes.c_int32(), ctypes.c_double(), ctypes.c_double()
    gamma = it.gamma
    rc = lib().orc_newton_csr(
        a.n, a.row_ptr.ctypes.data, a.col.ctypes.data, a.vals.ctypes.data, v.ctypes.data,
        p.ctypes.data, np.ascontiguousarray(it.dd).ctypes.data, it.xi.ctypes.data, len(it.dd),
        1.0 / gamma, it.center / gamma, float(tol), ws.ctypes.data,
        ctypes.byref(mv), ctypes.byref(term), ctypes.byref(pn))
    if rc == 2:
        ref = pn.value
        raise OracleConvergenceError(term.value / ref if ref > 0 else float("inf"), mv.value)
    return p, mv.value


def _z(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def csr_fused_z(a: Csr, alpha, beta, x, use_beta=True):
    """The reference's complex CSR rows (_core.pyx:263-278 / _csr_same[cplx]):
    real or complex vals, complex x, complex alpha / beta."""
    x = _z(x)
    vals = a.vals if np.iscomplexobj(a.vals) else np.ascontiguousarray(a.vals, dtype=np.float64)
    y = np.empty(a.n, dtype=np.complex128)
    al, be = complex(alpha), complex(beta)
    lib().orc_csr_fused_rows_z(0, a.n, a.row_ptr.ctypes.data, a.col.ctypes.data, vals.ctypes.data,
                               int(np.iscomplexobj(vals)), x.ctypes.data, y.ctypes.data, al.real, al.imag,
                               be.real, be.imag, int(use_beta))
    return y


def newton_csr_z(a: Csr, dd, xi, center: float, gamma: float, alpha, v, tol: float):
    """matfunc.newton_apply with complex divided differences / vectors on a
    CSR operator (the propagate path); alpha is the reference's op_alpha
    (1/gamma, or -1j/gamma on an imaginary-axis interval)."""
    v = _z(v)
    dd = _z(dd)
    if len(dd) == 1:
        return dd[0] * v, 0
    vals = a.vals if np.iscomplexobj(a.vals) else np.ascontiguousarray(a.vals, dtype=np.float64)
    p = np.empty_like(v)
    ws = np.empty(4 * a.n)
    ddabs = np.ascontiguousarray(np.abs(dd))
    xi = np.ascontiguousarray(xi, dtype=np.float64)
    mv, term, pn = ctypes.c_int32(), ctypes.c_double(), ctypes.c_double()
    al = complex(alpha)
    rc = lib().orc_newton_csr_z(
        a.n, a.row_ptr.ctypes.data, a.col.ctypes.data, vals.ctypes.data, int(np.iscomplexobj(vals)),
        v.ctypes.data, p.ctypes.data, dd.ctypes.data, ddabs.ctypes.data, xi.ctypes.data, len(dd), al.real, al.imag,
        center / gamma, float(tol), ws.ctypes.data, ctypes.byref(mv), ctypes.byref(term), ctypes.byref(pn))
    if rc == 2:
        ref = pn.value
        raise OracleConvergenceError(term.value / ref if ref > 0 else float("inf"), mv.value)
    return p, mv.value


def combustion(u: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty_like(u)
    bad = lib().orc_combustion(_ptr(u), _ptr(out), u.size)
    if bad >= 0:
        raise ValueError(f"domain error at index {bad}")
    return out


def combustion_jac(u: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.empty_like(u)
    lib().orc_combustion_jac(_ptr(u), _ptr(out), u.size)
    return out


def expeuler_step(spec: StencilSpec, u: np.ndarray, h: float, tol: float, max_degree=150,
                  interval=None, nonlinear=True, source=None):
    """integrator._StepWorkspace.step (integrator.py:177-189) without rescue.
    ``source`` is the affine-split boundary vector b: the forcing is g(u) - b,
    or -b for a linear problem (SemilinearProblem.forcing, integrator.py:104-123)."""
    a, b = interval if interval is not None else spec.gershgorin()
    ie = interpolant(a, b, "exp", -h, max_degree)
    ip = interpolant(a, b, "phi1", -h, max_degree)
    y, m1 = newton_stencil(spec, ie, u, tol)
    g = combustion(u) if nonlinear else None
    if source is not None:
        g = -source if g is None else g - source
    if g is None:
        return y, (m1, 0)
    z, m2 = newton_stencil(spec, ip, g, tol)
    out = np.empty_like(u)
    lib().orc_axpy_step(_ptr(y), _ptr(np.ascontiguousarray(z)), float(h), _ptr(out), u.size)
    return out, (m1, m2)


def snap_interval(lo: float, hi: float, base_lo: float, base_hi: float):
    """Build-defined Rosenbrock interval quantisation: widen
    [lo, hi] outward to multiples of q = (base_hi - base_lo)/1024 so
    consecutive steps reuse one interpolant."""
    q = (base_hi - base_lo) / 1024.0
    if q <= 0:
        return lo, hi
    return math.floor(lo / q) * q, math.ceil(hi / q) * q


def rosenbrock_step(spec: StencilSpec, u: np.ndarray, h: float, tol: float, max_degree=150):
    """Build-defined exponential Rosenbrock-Euler step:
    u+ = u + h phi1(-h M) F,  M = A - diag(g'(u)),  F = g(u) - A u."""
    g = combustion(u)
    gp = combustion_jac(u)
    au = stencil_fused(spec, 1.0, 0.0, u)
    f = g - au
    a0, b0 = spec.gershgorin()
    lo, hi = a0 - float(np.max(gp)), b0 - float(np.min(gp))
    lo, hi = snap_interval(lo, hi, a0, b0)
    ip = interpolant(lo, hi, "phi1", -h, max_degree)
    z, m = newton_stencil(spec, ip, f, tol, gdiag=gp)
    out = np.empty_like(u)
    lib().orc_axpy_step(_ptr(u), _ptr(np.ascontiguousarray(z)), float(h), _ptr(out), u.size)
    return out, m


def integrate(spec: StencilSpec, u0: np.ndarray, h: float, t_end: float, tol: float, max_degree=150,
              nonlinear=True, source=None):
    """integrator.integrate (integrator.py:209-239) without rescue: exponential
    Euler to t_end, the last step shortened to land on t_end exactly.
    Returns (u, observer records [(step, t, matvecs, max|u|)])."""
    u = np.array(u0, dtype=np.float64, copy=True)
    n_steps = max(1, math.ceil(t_end / h - 1e-12))
    iv = spec.gershgorin()
    t, obs = 0.0, []
    for k in range(n_steps):
        last = k == n_steps - 1
        h_k = t_end - (n_steps - 1) * h if last else h
        if not (last and abs(h_k - h) > 1e-15 * h):
            h_k = h
        u, (m1, m2) = expeuler_step(spec, u, h_k, tol, max_degree, interval=iv, nonlinear=nonlinear,
                                    source=source)
        t = t_end if last else t + h
        obs.append((k + 1, t, m1 + m2, float(np.max(np.abs(u)))))
    return u, obs
