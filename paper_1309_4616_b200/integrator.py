"""Exponential integrators for du/dt + A u = g(u) on B200 (drop-in for the
reference's integrator.py, plus the build-defined exponential Rosenbrock).

Exponential Euler (integrator.py:177-189):
    u+ = exp(-h A) u + h phi1(-h A) (g(u) - b)
Exponential Rosenbrock-Euler (build-defined):
    u+ = u + h phi1(-h M) F,  M = A - diag(g'(u)),  F = g(u) - b - A u.

Within a run the state never leaves HBM: both series, the nonlinearity (with
its on-device domain check), the Jacobian diagonal and the step combination
are device kernels; the host only sees matvec counts and, on request, the
observer's max |u|.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from math import ceil
from typing import Callable, Optional, Union

import numpy as np
import torch

from . import _lib, timing
from .device import empty, is_host, like_input, ptr, stream_handle, to_device
from .errors import ConvergenceError, DomainError
from .grid import Field
from .matfunc import (
    MatfuncStats,
    SpectralInterval,
    apply_matfunc,
    gershgorin_interval,
    make_interpolant,
    newton_apply,
)


def _values(u):
    return u.values if isinstance(u, Field) else u


def combustion_g(u, t=None, backend: str = "auto"):
    """(2 - u)/4 exp(20 (1 - 1/u)) on the device; u <= 0 raises DomainError
    with the first offending index (integrator.py:35-54).  Accepts an optional
    time argument, so SemilinearProblem's g(u, t) probe works (the reference
    binds t to `backend` and crashes)."""
    vals = _values(u)
    host = is_host(vals)
    dt = np.asarray(vals).dtype if host else vals.dtype
    if dt not in (np.float32, np.float64, torch.float32, torch.float64):
        raise DomainError("combustion nonlinearity is real-valued")
    if dt in (np.float32, torch.float32):  # the reference's float kernel (expf)
        return _combustion_f32(u, vals, host)
    ud = to_device(vals)
    out = empty(ud.numel())
    bad = ctypes.c_int64(-1)
    rc = _lib.load().es_combustion_pointwise(ptr(ud), ptr(out), ud.numel(), ctypes.byref(bad), stream_handle())
    if rc == _lib.ES_ERR_DOMAIN:
        i = int(bad.value)
        raise DomainError(f"combustion nonlinearity undefined at index {i} (u={float(ud[i])!r} <= 0)", index=i)
    _lib.check(rc, "es_combustion_pointwise")
    res = like_input(out, host)
    return Field(u.grid, res) if isinstance(u, Field) else res


def _combustion_f32(u, vals, host):
    ud = torch.from_numpy(np.ascontiguousarray(vals)).cuda() if host else vals.contiguous()
    bad = torch.nonzero(ud <= 0)
    if bad.numel():  # first u <= 0, like integrator.py:43-49
        i = int(bad[0, 0])
        raise DomainError(f"combustion nonlinearity undefined at index {i} (u={float(ud[i])!r} <= 0)", index=i)
    out = torch.empty_like(ud)
    _lib.check(_lib.load().es_combustion_pointwise_f32(ptr(ud), ptr(out), ud.numel(), stream_handle()),
               "es_combustion_pointwise_f32")
    res = like_input(out, host)
    return Field(u.grid, res) if isinstance(u, Field) else res


def combustion_jacobian(u):
    """(g'(u), (min g', max g')) on the device (build-defined Rosenbrock
    Jacobian diagonal of the combustion term)."""
    ud = to_device(_values(u))
    out = empty(ud.numel())
    mm = empty(2)
    _lib.check(_lib.load().es_combustion_jacobian(ptr(ud), ptr(out), ptr(mm), ud.numel(), stream_handle()),
               "es_combustion_jacobian")
    return out, mm


NONLINEARITIES: dict[str, Optional[Callable]] = {"zero": None, "combustion": combustion_g}
JACOBIANS: dict[Callable, Callable] = {combustion_g: combustion_jacobian}


def get_nonlinearity(name: str):
    try:
        return NONLINEARITIES[name]
    except KeyError:
        raise KeyError(f"unknown nonlinearity {name!r}; registered: {sorted(NONLINEARITIES)}") from None


def _axpy(y, z, h):
    """y + h z (one fused device pass, numpy rounding y + fl(h z))."""
    out = empty(y.numel())
    _lib.check(_lib.load().es_axpy(ptr(y), ptr(z), float(h), ptr(out), y.numel(), stream_handle()), "es_axpy")
    return out


@dataclass
class SemilinearProblem:
    """Operator, nonlinearity and initial state of du/dt + A u = g(u)."""

    operator: object
    nonlinearity: Optional[Callable] = None
    u0: Union[Field, np.ndarray, torch.Tensor, None] = None
    boundary_source: Optional[object] = None
    interval: Optional[SpectralInterval] = None
    jacobian: Optional[Callable] = None

    def __post_init__(self):
        if self.u0 is None:
            raise ValueError("initial state u0 is required")
        n = int(np.prod(tuple(self.initial_values().shape)))
        if self.boundary_source is not None:
            if int(np.prod(tuple(np.shape(self.boundary_source)))) != n:
                raise ValueError("boundary_source length does not match u0")
            self._b_dev = to_device(self.boundary_source)
        if self.interval is None:
            self.interval = gershgorin_interval(self.operator)
        if self.jacobian is None:
            self.jacobian = JACOBIANS.get(self.nonlinearity)
        self._g_takes_time: Optional[bool] = None

    def initial_values(self):
        return _values(self.u0)

    def _call_g(self, g, u, t):
        if self._g_takes_time is None:
            try:
                gu = g(u, t)
                self._g_takes_time = True
            except TypeError:
                gu = g(u)
                self._g_takes_time = False
            return gu
        return g(u, t) if self._g_takes_time else g(u)

    def forcing(self, u: torch.Tensor, t: float) -> Optional[torch.Tensor]:
        """g(u[, t]) - b on the device, or None for a purely linear problem."""
        g = self.nonlinearity
        if g is None:
            if self.boundary_source is None:
                return None
            neg = empty(self._b_dev.numel())
            _lib.check(_lib.load().es_scale(ptr(self._b_dev), -1.0, ptr(neg), neg.numel(), stream_handle()))
            return neg
        if hasattr(self.operator, "comm"):  # one slab / row block per rank: agree on DomainError
            from .distributed import rank_consistent_pointwise

            gu = rank_consistent_pointwise(self.operator, lambda: self._call_g(g, u, t))
        else:
            gu = self._call_g(g, u, t)
        gu = to_device(gu)
        if self.boundary_source is not None:
            gu = _axpy(gu, self._b_dev, -1.0)
        return gu


@dataclass
class StepperConfig:
    h: float
    t_end: float
    tol: float = 1e-8
    max_degree: int = 150

    def __post_init__(self):
        if not (self.h > 0):
            raise ValueError("time step h must be positive")
        if self.h > self.t_end:
            raise ValueError("h must not exceed t_end")
        if not (self.tol > 0):
            raise ValueError("tolerance must be positive")
        if self.max_degree < 1:
            raise ValueError("max_degree must be >= 1")


@dataclass
class StepStats:
    matvecs: int = 0
    matvecs_exp: int = 0
    matvecs_phi1: int = 0
    degree_exp: int = 0
    degree_phi1: int = 0
    halvings: int = 0


def _plain_stencil(op) -> bool:
    """A single-device stencil operator the fused step entries accept."""
    from .stencil import StencilOperator

    return type(op) is StencilOperator and op.bc.kind != "function"


class _StepWorkspace:
    """Interpolants for one (A, h), reused across steps."""

    def __init__(self, problem: SemilinearProblem, h: float, tol: float, max_degree: int):
        self.problem, self.h, self.tol, self.max_degree = problem, h, tol, max_degree
        iv = problem.interval
        self.exp_interp = make_interpolant(iv, "exp", -h, max_degree, tol)
        self.phi_interp = make_interpolant(iv, "phi1", -h, max_degree, tol)
        ei, pi = self.exp_interp, self.phi_interp
        # one C call per step (es_expeuler_step) where the operator, the
        # nonlinearity and the interpolants allow it
        self._fused = (_plain_stencil(problem.operator) and problem.nonlinearity in (None, combustion_g)
                       and iv.axis == "real" and len(ei.dd) > 1 and len(ei.dd) == len(pi.dd)
                       and not np.iscomplexobj(ei.dd) and not np.iscomplexobj(pi.dd)
                       and np.array_equal(ei.xi, pi.xi))
        self._ws_phi = None
        self._scratch = None
        self._call = None  # cached C-call arguments (_fused_step)

    def _fused_step(self, u: torch.Tensor):
        """Both series concurrently, g_n and y + h z on the device, one host
        sync.  None when a series ran out of nodes or u left the domain: the
        step is then re-run through the reference's orchestration below, which
        raises or rescues exactly as integrator.py:169-189 does."""
        from .device import Workspace

        pr, op, lib = self.problem, self.problem.operator, _lib.load()
        n = u.numel()
        if n != op.n:
            return None
        c = self._call
        if c is None or c["dev"] != u.device:
            # everything but the state pointers is fixed for this (A, h): built once
            d, keep = op.desc()
            nbytes = lib.es_leja_stencil_workspace_bytes(ctypes.byref(d))
            if self._ws_phi is None:
                self._ws_phi = Workspace()
            if self._scratch is None or self._scratch.numel() < 2 * n:
                self._scratch = empty(2 * n)
            ws_exp, ws_phi = op._ws.get(nbytes), self._ws_phi.get(nbytes)
            dde, xi = self.exp_interp.device_coeffs()
            ddp, _ = self.phi_interp.device_coeffs()
            iv = self.exp_interp.interval
            gamma = iv.halfspan
            nonlin = _lib.ES_NONLIN_COMBUSTION if pr.nonlinearity is combustion_g else _lib.ES_NONLIN_NONE
            src = pr._b_dev if pr.boundary_source is not None else None
            res = _lib.StepResult()
            c = self._call = dict(dev=u.device, keep=(d, keep, ws_exp, ws_phi, dde, xi, ddp, src), res=res,
                                  head=(ctypes.byref(d),),
                                  mid=(ptr(dde), dde.numel(), ptr(ddp), ddp.numel(), ptr(xi), 1.0 / gamma,
                                       iv.center / gamma, float(self.tol), float(self.h), nonlin, ptr(src),
                                       ptr(self._scratch), ptr(ws_exp), ptr(ws_phi), nbytes, ctypes.byref(res)))
        out = empty(n)
        res = c["res"]
        rc = lib.es_expeuler_step(*c["head"], ptr(u), ptr(out), *c["mid"], stream_handle())
        if rc in (_lib.ES_ERR_DOMAIN, _lib.ES_ERR_NOT_CONVERGED):
            return None
        _lib.check(rc, "es_expeuler_step")
        mv_e, mv_p = int(res.exp_series.matvecs), int(res.phi1_series.matvecs)
        tm = timing.active()
        if tm:
            tm.add_ms(res.series_ms, mv_e + mv_p, int(res.exp_series.passes) + int(res.phi1_series.passes))
        st = StepStats(matvecs=mv_e + mv_p, matvecs_exp=mv_e, matvecs_phi1=mv_p, degree_exp=mv_e, degree_phi1=mv_p)
        return out, st

    def _series(self, target, interp, v):
        a = self.problem.operator
        try:
            y, mv = newton_apply(a, interp, v, self.tol)
            return y, MatfuncStats(matvecs=mv, degree=mv)
        except ConvergenceError:
            # the reference re-runs level 0 inside the rescue (integrator.py:171-175)
            return apply_matfunc(a, v, target, -self.h, self.problem.interval, self.tol, self.max_degree)

    def step(self, u: torch.Tensor, t: float):
        if self._fused:
            r = self._fused_step(u)
            if r is not None:
                return r
        st = StepStats()
        y, s1 = self._series("exp", self.exp_interp, u)
        st.matvecs_exp, st.degree_exp, st.halvings = s1.matvecs, s1.degree, s1.halvings
        gn = self.problem.forcing(u, t)
        if gn is not None:
            z, s2 = self._series("phi1", self.phi_interp, gn)
            st.matvecs_phi1, st.degree_phi1 = s2.matvecs, s2.degree
            st.halvings = max(st.halvings, s2.halvings)
            y = _axpy(y, z, self.h)
        st.matvecs = st.matvecs_exp + st.matvecs_phi1
        return y, st


def _wrap(u_like, out: torch.Tensor):
    vals = _values(u_like)
    res = like_input(out, is_host(vals))
    return Field(u_like.grid, res) if isinstance(u_like, Field) else res


def exponential_euler_step(problem: SemilinearProblem, u_n, h: float, tol: float, max_degree: int = 150,
                           t: float = 0.0):
    ws = _StepWorkspace(problem, h, tol, max_degree)
    out, stats = ws.step(to_device(_values(u_n)), t)
    return _wrap(u_n, out), stats


def max_abs(u: torch.Tensor) -> float:
    out = empty(1)
    _lib.check(_lib.load().es_max_abs(ptr(u), u.numel(), ptr(out), stream_handle()), "es_max_abs")
    return float(out.item())


def integrate(problem: SemilinearProblem, cfg: StepperConfig, observer: Optional[Callable] = None,
              method: str = "euler"):
    """Fixed-step integration to t_end; the last step is shortened to land on
    t_end (integrator.py:209-239).  method: 'euler' | 'rosenbrock'."""
    u = to_device(problem.initial_values()).clone()
    n_steps = max(1, ceil(cfg.t_end / cfg.h - 1e-12))
    if method == "euler":
        ws = _StepWorkspace(problem, cfg.h, cfg.tol, cfg.max_degree)
        ws_last = None
    elif method == "rosenbrock":
        ros = RosenbrockStepper(problem, cfg.tol, cfg.max_degree)
    else:
        raise ValueError(f"unknown method {method!r}")
    t = 0.0
    for k in range(n_steps):
        last = k == n_steps - 1
        h_k = cfg.t_end - (n_steps - 1) * cfg.h if last else cfg.h
        try:
            if method == "rosenbrock":
                u, stats = ros.step(u, t, h_k)
            elif last and abs(h_k - cfg.h) > 1e-15 * cfg.h:
                if ws_last is None:
                    ws_last = _StepWorkspace(problem, h_k, cfg.tol, cfg.max_degree)
                u, stats = ws_last.step(u, t)
            else:
                u, stats = ws.step(u, t)
        except (ConvergenceError, DomainError) as err:
            raise type(err)(f"step {k + 1} (t={t:.6g}): {err}") from err
        t = cfg.t_end if last else t + cfg.h
        if observer is not None:
            mx = max_abs(u)
            if hasattr(problem.operator, "comm"):  # the global max-norm, like a single-device run
                from .distributed import allreduce_scalar

                mx = allreduce_scalar(problem.operator.comm, mx, torch.distributed.ReduceOp.MAX)
            observer(k + 1, t, stats.matvecs, mx)
    return _wrap(problem.u0, u)


# ---------------------------------------------------------------------------
# exponential Rosenbrock-Euler (build-defined; no reference counterpart)


def snap_interval(lo: float, hi: float, base: SpectralInterval):
    """Widen [lo, hi] outward to multiples of (b - a)/1024 of the operator's
    own interval, so consecutive steps share one interpolant (its divided
    differences cost ~20 ms of host BLAS to build)."""
    q = (base.b - base.a) / 1024.0
    if q <= 0:
        return lo, hi
    return math.floor(lo / q) * q, math.ceil(hi / q) * q


class RosenbrockOperator:
    """M = A - diag(gdiag) for a stencil A: the series kernel reads the
    diagonal in the same pass (40 B/point per node)."""

    def __init__(self, base, gdiag: torch.Tensor):
        self.base_operator, self.gdiag = base, gdiag

    @property
    def n(self):
        return self.base_operator.n

    def _leja(self, v, p_out, dd, xi, alpha, shift, tol, gdiag=None):
        return self.base_operator._leja(v, p_out, dd, xi, alpha, shift, tol, gdiag=self.gdiag)


@dataclass
class RosenbrockStats(StepStats):
    interval: tuple = (0.0, 0.0)


class RosenbrockStepper:
    def __init__(self, problem: SemilinearProblem, tol: float, max_degree: int = 150):
        from .stencil import StencilOperator

        self._dist = hasattr(problem.operator, "comm")  # DistributedStencil (one slab per rank)
        if not (isinstance(problem.operator, StencilOperator) or self._dist):
            raise TypeError("exponential Rosenbrock needs a StencilOperator or DistributedStencil")
        if problem.jacobian is None:
            raise ValueError("exponential Rosenbrock needs the nonlinearity's Jacobian diagonal")
        self.problem, self.tol, self.max_degree = problem, tol, max_degree
        self._interp: dict = {}
        self._fused = None  # None: try the fused prologue; False: not eligible
        self._aux = None
        self._one_call = True  # es_exprb_step until it reports the grid ineligible
        self._last = None  # snapped interval of the previous step
        self._scratch = None

    def interpolant(self, lo: float, hi: float, h: float):
        key = (lo, hi, h)
        if key not in self._interp:
            if len(self._interp) > 64:
                self._interp.clear()
            self._interp[key] = make_interpolant(SpectralInterval(lo, hi), "phi1", -h, self.max_degree, self.tol)
        return self._interp[key]

    def _prologue(self, u: torch.Tensor, t: float):
        """(F, g', min g', max g').  Fused single pass for the combustion term
        (es_rosenbrock_prologue: 24 B/point instead of 72); generic path for
        other nonlinearities, boundary sources or grids the TMA kernel skips."""
        pr = self.problem
        op = pr.operator
        if pr.nonlinearity is combustion_g and pr.boundary_source is None and self._fused is not False:
            f = empty(u.numel())
            gp = empty(u.numel())
            d, keep = op.desc()
            mm = (ctypes.c_double * 2)()
            bad = ctypes.c_int64(-1)
            if self._aux is None:
                self._aux = torch.empty(4, dtype=torch.int64, device=u.device)
            hl = hh = None
            if self._dist:
                op.halo_exchange(u)
                hl, hh = op.halo_lo, op.halo_hi
            rc = _lib.load().es_rosenbrock_prologue(ctypes.byref(d), ptr(u), ptr(f), ptr(gp), mm, ctypes.byref(bad),
                                                   ptr(self._aux), ptr(hl), ptr(hh), stream_handle())
            del keep
            if rc in (_lib.ES_OK, _lib.ES_ERR_DOMAIN):
                gmin, gmax, i = mm[0], mm[1], int(bad.value)
                if self._dist:  # global interval and first bad point over all slabs
                    import torch.distributed as dist

                    c = op.comm
                    big = float(2 ** 62)
                    t3 = torch.tensor([gmin, -gmax, float(c.z_lo * c.plane + i) if i >= 0 else big],
                                      dtype=torch.float64, device=u.device)
                    c.allreduce(t3, dist.ReduceOp.MIN)
                    gmin, gmax = float(t3[0]), -float(t3[1])
                    i = int(t3[2]) if float(t3[2]) < big else -1
                if i >= 0:
                    raise DomainError(f"combustion nonlinearity undefined at index {i} (u <= 0)", index=i)
                self._fused = True
                return f, gp, gmin, gmax
            if rc != _lib.ES_ERR_ARG or self._dist:
                _lib.check(rc, "es_rosenbrock_prologue")
            self._fused = False  # not eligible (odd nx, faces, ...): generic path from now on
        g = pr.forcing(u, t)
        gp, mm = pr.jacobian(u)
        au = empty(u.numel())
        from .stencil import fused_slab

        fused_slab(op, 1.0, 0.0, u, au)
        f = _axpy(g, au, -1.0)  # F = g - b - A u
        gmin, gmax = (float(v) for v in mm.cpu())
        return f, gp, gmin, gmax

    def _one_call_step(self, u: torch.Tensor, h: float):
        """es_exprb_step: prologue, interval check, series and u + h z in one
        C call (one more, es_exprb_finish, when the snapped interval moved).
        None when the fused path does not apply (odd nx, unaligned, ...)."""
        from .device import Workspace

        pr, op, lib = self.problem, self.problem.operator, _lib.load()
        n = u.numel()
        if n != op.n:
            return None
        d, keep = op.desc()
        nbytes = lib.es_leja_stencil_workspace_bytes(ctypes.byref(d))
        ws = op._ws.get(nbytes)
        if self._scratch is None or self._scratch.numel() < 2 * n:
            self._scratch = empty(2 * n)
        if self._aux is None:
            self._aux = torch.empty(4, dtype=torch.int64, device=u.device)
        out = empty(n)
        res = _lib.StepResult()
        a, b = pr.interval.a, pr.interval.b

        def coeffs(lo, hi):
            it = self.interpolant(lo, hi, h)
            dd, xi = it.device_coeffs()
            iv = it.interval
            return it, dd, xi, 1.0 / iv.halfspan, iv.center / iv.halfspan

        lo, hi = self._last if self._last is not None else (math.nan, math.nan)
        if self._last is not None:
            it, dd, xi, alpha, shift = coeffs(lo, hi)
        else:  # no interval yet: the call stops after the prologue with ES_ERR_RANGE
            it, dd, xi, alpha, shift = None, self._aux, self._aux, 1.0, 0.0
        args = (ptr(dd), ptr(xi), dd.numel() if it is not None else 2, alpha, shift, float(self.tol), float(h))
        rc = lib.es_exprb_step(ctypes.byref(d), ptr(u), ptr(out), *args, a, b, lo, hi, ptr(self._scratch),
                               ptr(self._aux), ptr(ws), nbytes, ctypes.byref(res), stream_handle())
        if rc == _lib.ES_ERR_RANGE:
            lo, hi = res.lo, res.hi
            it, dd, xi, alpha, shift = coeffs(lo, hi)
            if len(it.dd) == 1:  # degenerate interval: newton_apply's scaling path
                return None
            rc = lib.es_exprb_finish(ctypes.byref(d), ptr(u), ptr(out), ptr(dd), ptr(xi), dd.numel(), alpha, shift,
                                     float(self.tol), float(h), ptr(self._scratch), ptr(ws), nbytes,
                                     ctypes.byref(res), stream_handle())
        del keep
        if rc == _lib.ES_ERR_DOMAIN:
            i = int(res.first_bad)
            raise DomainError(f"combustion nonlinearity undefined at index {i} (u <= 0)", index=i)
        self._last = (lo, hi)
        if rc == _lib.ES_ERR_NOT_CONVERGED:  # the halving rescue on the kept F, g'
            f, gp = self._scratch[:n], self._scratch[n:2 * n]
            z, st = _rescued(RosenbrockOperator(op, gp), it, f, self.tol, h, SpectralInterval(lo, hi),
                             self.max_degree)
            return _axpy(u, z, h), RosenbrockStats(matvecs=st.matvecs, matvecs_phi1=st.matvecs, degree_phi1=st.degree,
                                                   halvings=st.halvings, interval=(lo, hi))
        _lib.check(rc, "es_exprb_step")
        mv = int(res.phi1_series.matvecs)
        tm = timing.active()
        if tm:
            tm.add_ms(res.series_ms, mv, int(res.phi1_series.passes))
        return out, RosenbrockStats(matvecs=mv, matvecs_phi1=mv, degree_phi1=mv, interval=(lo, hi))

    def step(self, u: torch.Tensor, t: float, h: float):
        pr = self.problem
        op = pr.operator
        if (self._one_call and pr.nonlinearity is combustion_g and pr.boundary_source is None
                and _plain_stencil(op) and pr.interval.axis == "real"):
            try:
                r = self._one_call_step(u, h)
            except ValueError:  # ES_ERR_ARG: not eligible for the fused kernels
                r = None
            if r is not None:
                return r
            self._one_call = False
        f, gp, gmin, gmax = self._prologue(u, t)
        lo, hi = snap_interval(pr.interval.a - gmax, pr.interval.b - gmin, pr.interval)
        interp = self.interpolant(lo, hi, h)
        mop = RosenbrockOperator(op, gp)
        z, st = _rescued(mop, interp, f, self.tol, h, SpectralInterval(lo, hi), self.max_degree)
        stats = RosenbrockStats(matvecs=st.matvecs, matvecs_phi1=st.matvecs, degree_phi1=st.degree,
                                halvings=st.halvings, interval=(lo, hi))
        return _axpy(u, z, h), stats


def _rescued(op, interp, v, tol, h, interval, max_degree):
    try:
        y, mv = newton_apply(op, interp, v, tol)
        return y, MatfuncStats(matvecs=mv, degree=mv)
    except ConvergenceError:
        return apply_matfunc(op, v, "phi1", -h, interval, tol, max_degree)


def exponential_rosenbrock_step(problem: SemilinearProblem, u_n, h: float, tol: float, max_degree: int = 150,
                                t: float = 0.0):
    out, stats = RosenbrockStepper(problem, tol, max_degree).step(to_device(_values(u_n)), t, h)
    return _wrap(u_n, out), stats
