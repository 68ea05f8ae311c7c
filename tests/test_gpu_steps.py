"""The one-call integrator steps (es_expeuler_step, es_exprb_step /
es_exprb_finish; SURVEY.md section 8(b) stage helpers) against the
Python-orchestrated steps of the same package (integrator.py:177-189 order:
exp series, g(u) - b, phi1 series, y + h z) -- bitwise, with equal matvec
counts -- and their error paths: domain errors, exhausted series (halving
rescue), interval changes between Rosenbrock steps."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1309_4616_b200 as es  # noqa: E402
from paper_1309_4616_b200 import _lib  # noqa: E402
from paper_1309_4616_b200.device import ptr, stream_handle  # noqa: E402
from paper_1309_4616_b200.integrator import _StepWorkspace  # noqa: E402

from conftest import coeff_d  # noqa: E402


def _u0(n, seed=21):
    return torch.from_numpy(1.0 + 0.1 * np.random.default_rng(seed).random(n)).cuda()


def _euler_pair(prob, h, tol, max_degree=150):
    a = _StepWorkspace(prob, h, tol, max_degree)
    b = _StepWorkspace(prob, h, tol, max_degree)
    b._fused = False
    return a, b


@pytest.mark.parametrize("case", ["combustion", "combustion+source", "source only", "linear", "neumann+coeff"])
def test_expeuler_one_call_matches_orchestrated(case):
    g = es.Grid3D(48, 34, 21)
    bc = es.BoundaryCondition.neumann() if "neumann" in case else es.BoundaryCondition.homogeneous()
    op = es.StencilOperator(g, bc, coeff=coeff_d if "coeff" in case else None)
    src = np.random.default_rng(5).standard_normal(g.n) * 0.01 if "source" in case else None
    nl = es.combustion_g if case.startswith("combustion") or "neumann" in case else None
    u0 = _u0(g.n)
    prob = es.SemilinearProblem(operator=op, nonlinearity=nl, u0=u0, boundary_source=src)
    fused, plain = _euler_pair(prob, 1e-4, 1e-6)
    assert fused._fused
    u1, s1 = fused.step(u0, 0.0)
    u2, s2 = plain.step(u0, 0.0)
    assert (s1.matvecs_exp, s1.matvecs_phi1, s1.matvecs) == (s2.matvecs_exp, s2.matvecs_phi1, s2.matvecs)
    assert torch.equal(u1, u2), case
    if nl is None and src is None:
        assert s1.matvecs_phi1 == 0


def test_expeuler_one_call_2d_and_trajectory():
    g = es.Grid3D(256, 256, 1)  # C1 shape
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    u0 = _u0(g.n, 3)
    prob = es.SemilinearProblem(operator=op, nonlinearity=es.combustion_g, u0=u0)
    fused, plain = _euler_pair(prob, 1e-4, 1e-4)
    ua, ub = u0, u0
    for _ in range(4):
        ua, sa = fused.step(ua, 0.0)
        ub, sb = plain.step(ub, 0.0)
        assert sa.matvecs == sb.matvecs
    assert torch.equal(ua, ub)


def test_expeuler_one_call_domain_error_and_rescue():
    g = es.Grid3D(32, 16, 8)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    u0 = _u0(g.n)
    u0[99] = -1.0
    prob = es.SemilinearProblem(operator=op, nonlinearity=es.combustion_g, u0=u0)
    with pytest.raises(es.DomainError):
        _StepWorkspace(prob, 1e-4, 1e-6, 150).step(u0, 0.0)
    # too few nodes: the fused call reports the exhausted series and the step
    # falls back to the reference's orchestration (halving rescue)
    u0 = _u0(g.n)
    prob = es.SemilinearProblem(operator=op, nonlinearity=es.combustion_g, u0=u0)
    fused, plain = _euler_pair(prob, 1e-3, 1e-10, max_degree=12)
    u1, s1 = fused.step(u0, 0.0)
    u2, s2 = plain.step(u0, 0.0)
    assert s1.halvings == s2.halvings and s1.halvings > 0
    assert (s1.matvecs_exp, s1.matvecs_phi1) == (s2.matvecs_exp, s2.matvecs_phi1)
    assert torch.equal(u1, u2)


def test_exprb_one_call_matches_orchestrated_over_steps():
    g = es.Grid3D(64, 40, 24)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    u0 = _u0(g.n, 8)
    prob = es.SemilinearProblem(operator=op, nonlinearity=es.combustion_g, u0=u0)
    one = es.RosenbrockStepper(prob, 1e-6)
    orch = es.RosenbrockStepper(prob, 1e-6)
    orch._one_call = False
    ua, ub = u0, u0
    intervals = []
    for k in range(5):
        h = 2e-4 * (1 + k % 2)  # alternate h: every step rebuilds or reuses interpolants
        ua, sa = one.step(ua, 0.0, h)
        ub, sb = orch.step(ub, 0.0, h)
        assert sa.matvecs == sb.matvecs and sa.interval == sb.interval
        assert torch.equal(ua, ub), k
        intervals.append(sa.interval)
    assert one._one_call


def test_exprb_c_abi_range_then_finish():
    g = es.Grid3D(32, 24, 16)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    u = _u0(g.n, 9)
    n = g.n
    lib = _lib.load()
    d, keep = op.desc()
    nb = lib.es_leja_stencil_workspace_bytes(ctypes.byref(d))
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    scratch = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    aux = torch.empty(4, dtype=torch.int64, device="cuda")
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    a, b = es.gershgorin_bounds(op)
    res = _lib.StepResult()
    dummy = torch.zeros(2, dtype=torch.float64, device="cuda")
    rc = lib.es_exprb_step(ctypes.byref(d), ptr(u), ptr(out), ptr(dummy), ptr(dummy), 2, 1.0, 0.0, 1e-6, 2e-4,
                           a, b, 0.0, 1.0, ptr(scratch), ptr(aux), ptr(ws), nb, ctypes.byref(res), stream_handle())
    assert rc == _lib.ES_ERR_RANGE and res.first_bad == -1
    gmin, gmax = res.gprime_min, res.gprime_max
    lo, hi = es.snap_interval(a - gmax, b - gmin, es.SpectralInterval(a, b))
    assert (res.lo, res.hi) == (lo, hi)
    it = es.make_interpolant(es.SpectralInterval(lo, hi), "phi1", -2e-4, 150, 1e-6)
    dd, xi = it.device_coeffs()
    gam = it.interval.halfspan
    rc = lib.es_exprb_finish(ctypes.byref(d), ptr(u), ptr(out), ptr(dd), ptr(xi), dd.numel(), 1.0 / gam,
                             it.interval.center / gam, 1e-6, 2e-4, ptr(scratch), ptr(ws), nb, ctypes.byref(res),
                             stream_handle())
    assert rc == _lib.ES_OK and res.status_phi1 == 0 and res.series_ms > 0
    prob = es.SemilinearProblem(operator=op, nonlinearity=es.combustion_g, u0=u)
    ref = es.RosenbrockStepper(prob, 1e-6)
    ref._one_call = False
    u2, st = ref.step(u, 0.0, 2e-4)
    assert st.matvecs == res.phi1_series.matvecs and torch.equal(out, u2)
    # aliasing and unknown nonlinearity are argument errors
    rc = lib.es_expeuler_step(ctypes.byref(d), ptr(u), ptr(u), ptr(dd), dd.numel(), ptr(dd), dd.numel(), ptr(xi),
                              1.0, 0.0, 1e-6, 1e-4, 1, None, ptr(scratch), ptr(ws), ptr(ws), nb, ctypes.byref(res),
                              stream_handle())
    assert rc == _lib.ES_ERR_ARG
    del keep
