"""Parity at the BENCHMARKED sizes: every workload bench.py times (BASELINE
configs C1, C2, C3, C5) is run here through the same public-API calls the
bench makes, on the bench's own seeded inputs, and compared with the CPU
oracle (plain C, test infrastructure) or with reference-generated goldens.

Tolerances (north_star): bitwise for series without a
transcendental; 1e-12 relative per step and 1e-10 over a trajectory where
the step contains CUDA exp() (combustion g, g'); equal matvec counts always.
Also the split (Dirichlet-function boundary) path against reference goldens
(stencil.py:281-312, integrator.py:104-123).
"""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1309_4616_b200 as es  # noqa: E402
from oracle import oracle as orc  # noqa: E402

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402  (the bench's configs and seeded inputs, nothing timed)


def _relerr(a, b) -> float:
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


def test_c3_rosenbrock_512cubed_two_steps_vs_oracle():
    """The headline workload: 512^3 Dirichlet, combustion, exponential
    Rosenbrock-Euler, h = 2.5e-5, tol = 1e-4, u0 = 1 + 0.1 U[0,1) from
    default_rng(1234) -- two chained steps of bench.Stepper's call."""
    cfg = bench.CONFIGS["C3"]
    nx, ny, nz = cfg["dims"]
    g = es.Grid3D(nx, ny, nz)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    u0 = bench.initial_state(g.n)
    ud = torch.from_numpy(u0).cuda()
    prob = es.SemilinearProblem(operator=op, nonlinearity=es.combustion_g, u0=ud)
    assert op.two_node_passes()  # the benchmarked kernel (k_node_tb, multi-chunk)
    ros = es.RosenbrockStepper(prob, cfg["tol"])
    h = cfg["h"]
    u1, st1 = ros.step(ud, 0.0, h)
    u2, st2 = ros.step(u1, h, h)
    u1h, u2h = u1.cpu().numpy(), u2.cpu().numpy()
    del u1, u2, ud, ros, prob
    torch.cuda.empty_cache()
    spec = orc.StencilSpec(nx, ny, nz)
    r1, m1 = orc.rosenbrock_step(spec, u0, h, cfg["tol"])
    assert st1.matvecs == m1
    assert _relerr(u1h, r1) <= 1e-12
    r2, m2 = orc.rosenbrock_step(spec, r1, h, cfg["tol"])
    assert st2.matvecs == m2
    assert _relerr(u2h, r2) <= 1e-12


def test_c1_256sq_ten_steps_vs_reference_golden(golden):
    """C1 at full size: 256^2 exponential Euler, 10 steps; the golden is the
    reference's own integrate() (integrator.py:209-239) with its observer."""
    d = golden("c1_trajectory")
    h, tol, nsteps = d["params"]
    cfg = bench.CONFIGS["C1"]
    assert (h, tol, tuple(int(v) for v in d["dims"])) == (cfg["h"], cfg["tol"], cfg["dims"])
    assert np.array_equal(d["u0"], bench.initial_state(256 * 256))
    g = es.Grid3D(256, 256, 1)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    obs = []
    prob = es.SemilinearProblem(operator=op, nonlinearity=es.combustion_g, u0=d["u0"])
    u = es.integrate(prob, es.StepperConfig(h=h, t_end=h * nsteps, tol=tol),
                     observer=lambda k, t, mv, mx: obs.append((k, t, mv, mx)))
    ref_obs = d["obs"]
    assert [o[2] for o in obs] == [int(v) for v in ref_obs[:, 2]]
    np.testing.assert_allclose([o[3] for o in obs], ref_obs[:, 3], rtol=1e-12)
    assert _relerr(u, d["u"]) <= 1e-10
    # the bench's loop: bench.Stepper (one fused C call per step), same steps
    step = bench.Stepper(cfg, es, es.SemilinearProblem(operator=op, nonlinearity=es.combustion_g,
                                                        u0=torch.from_numpy(d["u0"]).cuda()))
    ub = torch.from_numpy(d["u0"]).cuda()
    for k in range(int(nsteps)):
        ub, st = step(ub, k * h)
        assert st.matvecs == int(ref_obs[k, 2]), k
    assert _relerr(ub.cpu().numpy(), d["u"]) <= 1e-10


def test_c2_4096sq_benchmarked_series_vs_oracle():
    """C2 exactly as benched: exp(-hA) v, 4096^2 Neumann, radial D (streamed
    sample), h = 6e-7, tol = 1e-4, v ~ N(0,1) default_rng(1234)."""
    cfg = bench.CONFIGS["C2"]
    g = es.Grid3D(*cfg["dims"])
    op = es.StencilOperator(g, es.BoundaryCondition.neumann(), coeff=es.radial_coeff)
    v = np.random.default_rng(1234).standard_normal(g.n)
    prob = es.SemilinearProblem(operator=op, nonlinearity=None, u0=torch.from_numpy(v).cuda())
    step = bench.Stepper(cfg, es, prob)
    p, st = step(prob.u0, 0.0)
    spec = orc.StencilSpec(*cfg["dims"], mode=orc.MODE_NEUMANN, coeff_kind=orc.COEFF_RADIAL)
    lo, hi = spec.gershgorin()
    it = orc.interpolant(lo, hi, "exp", -cfg["h"], 150)
    ref, mv = orc.newton_stencil(spec, it, v, cfg["tol"])
    assert st.matvecs == mv
    assert p.cpu().numpy().tobytes() == ref.tobytes()


def test_c5_csr_2pow22_benchmarked_series_vs_oracle():
    """C5 exactly as benched: phi1(-A) v on the seeded n = 2^22 symmetric CSR
    matrix (5.45e7 nonzeros), tol = 1e-8 -- bitwise with equal matvecs."""
    cfg = bench.CONFIGS["C5"]
    a = bench.csr_matrix(cfg)
    v = np.random.default_rng(1234).standard_normal(a.nrows)
    step = bench.CsrStepper(cfg, es, a)
    p, st = step(torch.from_numpy(v).cuda(), 0.0)
    oc = orc.Csr(a.nrows, a.row_ptr, a.col_idx, a.vals)
    lo, hi = oc.gershgorin()
    it = orc.interpolant(lo, hi, "phi1", -cfg["h"], 150)
    assert np.array_equal(it.dd, step.it.dd)
    ref, mv = orc.newton_csr(oc, it, v, cfg["tol"])
    assert st.matvecs == mv
    assert p.cpu().numpy().tobytes() == ref.tobytes()


# ---------------------------------------------------------------------------
# Dirichlet-function boundaries: the affine split (reference goldens)


def _bc_fn(name):
    # the same expressions the golden's reference parse_expression evaluated
    if name == "poly":
        return es.BoundaryCondition.function(lambda x, y, z: z * (1 - z) * x * y, "z*(1-z)*x*y")
    return es.BoundaryCondition.function(lambda x, y, z: np.sin(np.pi * z) * np.exp(-x * y),
                                         "sin(pi*z)*exp(-x*y)")


def _split_op(d, p):
    g = es.Grid3D(*(int(v) for v in d[f"{p}_dims"]))
    coeff = es.radial_coeff if bool(d[f"{p}_coeff"]) else None
    return es.StencilOperator(g, _bc_fn(str(d[f"{p}_bc"])), coeff=coeff)


def test_affine_split_pieces_bitwise(golden):
    d = golden("split")
    for i in range(int(d["ncases"])):
        p = f"s{i}"
        op = _split_op(d, p)
        for j, f in enumerate(es.boundary_faces(op)):
            assert f.tobytes() == d[f"{p}_face{j}"].tobytes(), (p, j)
        x = es.Field(op.grid, d[f"{p}_x"])
        hom, b = es.apply_affine_split(op, x)
        assert np.asarray(hom.values).tobytes() == d[f"{p}_hom"].tobytes(), p
        assert np.asarray(b.values).tobytes() == d[f"{p}_b"].tobytes(), p
        bs = es.boundary_source_field(op)
        assert np.asarray(bs.values).tobytes() == d[f"{p}_bsrc"].tobytes(), p
        y = es.homogeneous_part(op).fused_apply_flat(0.75, -0.5, d[f"{p}_x"])
        assert y.tobytes() == d[f"{p}_hp_y"].tobytes(), p
        full = es.apply(op, x)
        assert np.asarray(full.values).tobytes() == d[f"{p}_full"].tobytes(), p


def test_split_problem_trajectories(golden):
    d = golden("split")
    for i in range(int(d["ntraj"])):
        p = f"t{i}"
        op = _split_op(d, p)
        h, tol, nsteps = d[f"{p}_params"]
        b = es.boundary_source_field(op).values
        assert np.asarray(b).tobytes() == d[f"{p}_b"].tobytes(), p
        nl = es.combustion_g if bool(d[f"{p}_nonlin"]) else None
        prob = es.SemilinearProblem(operator=es.homogeneous_part(op), nonlinearity=nl, u0=d[f"{p}_u0"],
                                    boundary_source=b)
        obs = []
        u = es.integrate(prob, es.StepperConfig(h=h, t_end=h * nsteps, tol=tol),
                         observer=lambda k, t, mv, mx: obs.append((k, t, mv, mx)))
        ref_obs = d[f"{p}_obs"]
        assert [o[2] for o in obs] == [int(v) for v in ref_obs[:, 2]], p
        np.testing.assert_allclose([o[3] for o in obs], ref_obs[:, 3], rtol=1e-12)
        tol_u = 0.0 if nl is None else 1e-10
        assert _relerr(u, d[f"{p}_u"]) <= tol_u, p
