"""The reference package itself, running on the B200 kernels.

``integration/expstencil_b200_backend.py`` is installed into the unmodified
reference (``oracle/_ref``, built by ``oracle/build_ref.sh``) through its own
seam, ``expstencil._kernels.get_kernels`` / ``available_backends``
(reference ``_kernels.py:31-53``).  Then the reference's operator contracts
(restated from ``pkg/tests/test_stencil.py:48-151`` and ``:190-262``: dense
equivalence, known answers, traversal invariance over every available
backend, affine split, complex fields) run through
``StencilOperator(..., backend="b200")``, and every kernel-module call is
compared bit for bit with the reference's own compiled core on the same
inputs.  Finally the whole reference (integrator, Newton-Leja series,
partitioned wrappers, CSR) runs with "b200" as its default backend.
"""

import math
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "oracle", "_ref")
if not os.path.isdir(os.path.join(REF, "expstencil")):  # pragma: no cover
    pytest.skip("reference not built (oracle/build_ref.sh)", allow_module_level=True)
sys.path.insert(0, REF)
sys.path.insert(0, os.path.join(REPO, "integration"))
os.environ.setdefault("EXPSTENCIL_KERNELS", "compiled")

import expstencil as ref  # noqa: E402
import expstencil_b200_backend as b200  # noqa: E402
from expstencil import _kernels  # noqa: E402
from expstencil.expr import parse_expression  # noqa: E402
from expstencil.grid import Field, Grid3D, eval_on_grid, linear_index, zeros_field  # noqa: E402
from expstencil.sparse import CsrMatrix, fused_spmv, spmv  # noqa: E402
from expstencil.stencil import (  # noqa: E402
    BoundaryCondition,
    StencilOperator,
    apply,
    apply_affine_split,
    boundary_source_field,
    fused_apply,
)

b200.install(_kernels)
core = _kernels.get_kernels("compiled")

BCS = {
    "none": BoundaryCondition.none(),
    "homogeneous": BoundaryCondition.homogeneous(),
    "poly": BoundaryCondition.function(parse_expression("z*(1-z)*x*y"), "z*(1-z)*x*y"),
    "trig": BoundaryCondition.function(parse_expression("sin(pi*z)*exp(-x*y)"), "sin(pi*z)*exp(-x*y)"),
}


def coeff_d(x, y, z):
    return 1.0 / np.sqrt(1.0 + x * x + y * y)


def test_seam_lists_and_resolves_b200():
    assert "b200" in _kernels.available_backends()
    assert _kernels.get_kernels("b200") is b200
    assert _kernels.get_kernels("b200").backend_name == "b200"
    with pytest.raises(ValueError):
        _kernels.get_kernels("nope")


# ---------------------------------------------------------------------------
# bitwise against the reference's compiled core, through the reference API


@pytest.mark.parametrize("kind", ["f64", "f32"])
@pytest.mark.parametrize("bc", list(BCS))
def test_apply_bitwise_equals_compiled_core(bc, kind):
    rng = np.random.default_rng(41)
    dt = np.float64 if kind == "f64" else np.float32
    for dims in [(5, 5, 5), (9, 9, 9), (7, 5, 3), (9, 7, 5), (33, 17, 1), (3, 1, 1), (1, 4, 6), (16, 12, 10)]:
        g = Grid3D(*dims)
        for coeff in (None, coeff_d):
            u = Field(g, rng.standard_normal(g.n).astype(dt))
            for trav in ("naive", "tiled"):
                got = apply(StencilOperator(g, BCS[bc], coeff=coeff, traversal=trav, tile=(4, 3), backend="b200"), u)
                exp = apply(StencilOperator(g, BCS[bc], coeff=coeff, backend="compiled"), u)
                assert got.values.dtype == exp.values.dtype == dt
                assert got.values.tobytes() == exp.values.tobytes(), (dims, bc, coeff is not None, trav)


def test_fused_apply_flat_bitwise_equals_compiled_core():
    rng = np.random.default_rng(42)
    for dims in [(11, 9, 12), (64, 48, 1), (20, 18, 16)]:
        g = Grid3D(*dims)
        for bc in ("none", "homogeneous"):
            for coeff in (None, coeff_d):
                x = rng.standard_normal(g.n)
                a, b = float(rng.uniform(0.1, 3)), float(rng.uniform(-2, 2))
                got = StencilOperator(g, BCS[bc], coeff=coeff, backend="b200").fused_apply_flat(a, b, x)
                exp = StencilOperator(g, BCS[bc], coeff=coeff, backend="compiled").fused_apply_flat(a, b, x)
                assert got.tobytes() == exp.tobytes(), (dims, bc)


def test_slab_with_halos_bitwise_equals_compiled_core():
    rng = np.random.default_rng(43)
    g = Grid3D(11, 9, 12)
    op = StencilOperator(g, BCS["homogeneous"], coeff=coeff_d)
    for dt in (np.float64, np.float32):
        x3 = rng.standard_normal(g.n).astype(dt).reshape(g.shape)
        c3 = op.coeff_values("f64" if dt == np.float64 else "f32")
        for z0, lz in ((0, 5), (5, 4), (9, 3)):
            lo = x3[z0 - 1].copy() if z0 > 0 else None
            hi = x3[z0 + lz].copy() if z0 + lz < g.nz else None
            outs = []
            for k in (b200, core):
                o3 = np.empty((lz, g.ny, g.nx), dtype=dt)
                k.stencil_fused_slab(x3[z0:z0 + lz].copy(), o3, 1.5, -0.25, op.weights(), 0, halo_lo=lo, halo_hi=hi,
                                     z0=z0, nz_total=g.nz, coeff3=c3[z0:z0 + lz].copy())
                outs.append(o3)
            assert outs[0].tobytes() == outs[1].tobytes(), (dt, z0, lz)


def test_stencil_kernel_rejects_other_dtypes():
    u = np.zeros((2, 2, 2), dtype=np.int64)
    with pytest.raises(TypeError):
        b200.stencil_fused_slab(u, np.empty_like(u), 1.0, 0.0, (1.0, 1.0, 1.0), 0)


@pytest.mark.parametrize("combo", ["f64", "f32", "f64-c128", "c128", "f64-i64", "c128-i64", "f32-i64"])
def test_csr_rows_bitwise_equals_compiled_core(combo):
    rng = np.random.default_rng(44)
    n = 3000
    dense = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.004)
    dense[7, :] = 0.0  # an empty row
    dense[11, :] = rng.standard_normal(n)  # a long row
    a = CsrMatrix.from_dense(dense)
    vals, x = a.vals, rng.standard_normal(n)
    alpha, beta = 0.7, -1.3
    if combo.startswith("f32"):
        vals, x = vals.astype(np.float32), x.astype(np.float32)
    if "c128" in combo:
        x = x + 1j * rng.standard_normal(n)
        alpha, beta = 0.7 - 0.2j, -1.3 + 0.5j
        if combo.startswith("c128"):
            vals = vals + 1j * rng.standard_normal(vals.shape[0])
    col = a.col_idx.astype(np.int64) if combo.endswith("i64") else a.col_idx
    for lo, hi in ((0, n), (5, 1777)):
        y0 = np.full(n, 9.0, dtype=x.dtype)
        y1 = y0.copy()
        b200.csr_fused_rows(lo, hi, a.row_ptr, col, vals, x, y0, alpha, beta, True)
        core.csr_fused_rows(lo, hi, a.row_ptr, col, vals, x, y1, alpha, beta, True)
        assert y0.tobytes() == y1.tobytes(), (combo, lo, hi)
    y0, y1 = np.empty(n, dtype=x.dtype), np.empty(n, dtype=x.dtype)
    b200.csr_fused(n, a.row_ptr, col, vals, x, y0, alpha, beta, False)
    core.csr_fused(n, a.row_ptr, col, vals, x, y1, alpha, beta, False)
    assert y0.tobytes() == y1.tobytes(), combo


def test_csr_public_api_bitwise():
    rng = np.random.default_rng(45)
    n = 2000
    dense = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.01)
    a = CsrMatrix.from_dense(dense)
    x = rng.standard_normal(n)
    assert spmv(a, x, backend="b200").tobytes() == spmv(a, x, backend="compiled").tobytes()
    assert fused_spmv(a, 0.5, 2.0, x, backend="b200").tobytes() == fused_spmv(a, 0.5, 2.0, x,
                                                                              backend="compiled").tobytes()
    with pytest.raises(TypeError):
        b200.csr_fused(n, a.row_ptr, a.col_idx.astype(np.int16), a.vals, x, np.empty(n), 1.0, 0.0, False)


def test_combustion_through_the_backend():
    from expstencil.errors import DomainError
    from expstencil.integrator import combustion_g

    u = np.random.default_rng(46).uniform(0.05, 2.5, 20000)
    got, exp = combustion_g(u, backend="b200"), combustion_g(u, backend="compiled")
    np.testing.assert_allclose(got, exp, rtol=2e-16 * 4, atol=0)  # CUDA exp vs libm: <= 1 ulp per op
    u32 = u.astype(np.float32)
    np.testing.assert_allclose(combustion_g(u32, backend="b200"), combustion_g(u32, backend="compiled"),
                               rtol=4 * 1.2e-7, atol=float(np.finfo(np.float32).tiny))  # subnormals: absolute
    with pytest.raises(DomainError):
        combustion_g(np.array([1.0, 0.0]), backend="b200")


# ---------------------------------------------------------------------------
# the reference's operator contracts, run on backend="b200"


def dense_laplacian(g: Grid3D, kind: str, fn=None, coeff=None):
    """(M, b) with A u = M u + b assembled point by point from the 7-point rule
    (independent of every kernel): periodic wrap for kind "none", zero ghosts
    for "homogeneous", ghosts f(x, y, z) on the boundary for "function"."""
    n = g.n
    m = np.zeros((n, n))
    b = np.zeros(n)
    dims = (g.nx, g.ny, g.nz)
    w = [0.0 if k == 1 else float((k + 1) ** 2) for k in dims]
    d = None if coeff is None else eval_on_grid(g, coeff).values
    for iz in range(g.nz):
        for iy in range(g.ny):
            for ix in range(g.nx):
                i = linear_index(g, ix, iy, iz)
                pos = [ix, iy, iz]
                for ax in range(3):
                    if w[ax] == 0.0:
                        continue
                    m[i, i] += 2.0 * w[ax]
                    for st in (-1, 1):
                        q = list(pos)
                        q[ax] += st
                        if 0 <= q[ax] < dims[ax]:
                            m[i, linear_index(g, *q)] -= w[ax]
                        elif kind == "none":
                            q[ax] %= dims[ax]
                            m[i, linear_index(g, *q)] -= w[ax]
                        elif kind == "function":
                            xyz = [(q[k] + 1) / (dims[k] + 1) for k in range(3)]
                            b[i] -= w[ax] * float(fn(*xyz))
                if d is not None:
                    m[i, :] *= d[i]
                    b[i] *= d[i]
    return m, b


@pytest.mark.parametrize("dims", [(5, 5, 5), (7, 5, 3), (6, 1, 4)])
@pytest.mark.parametrize("bc", list(BCS))
def test_dense_equivalence_on_b200(dims, bc):
    g = Grid3D(*dims)
    m, b = dense_laplacian(g, BCS[bc].kind, BCS[bc].fn)
    u = np.random.default_rng(47).standard_normal(g.n)
    exp = m @ u + b
    got = apply(StencilOperator(g, BCS[bc], backend="b200"), Field(g, u)).values
    assert np.max(np.abs(got - exp)) <= 1e-13 * np.max(np.abs(exp))
    u32 = u.astype(np.float32)
    got32 = apply(StencilOperator(g, BCS[bc], backend="b200"), Field(g, u32)).values
    assert got32.dtype == np.float32
    exp32 = m @ u32.astype(np.float64) + b
    assert np.max(np.abs(got32 - exp32)) <= 1e-5 * np.max(np.abs(exp32))


def test_dense_equivalence_with_coefficient_on_b200():
    g = Grid3D(6, 5, 4)
    m, _ = dense_laplacian(g, "homogeneous", coeff=coeff_d)
    u = np.random.default_rng(48).standard_normal(g.n)
    got = apply(StencilOperator(g, BCS["homogeneous"], coeff=coeff_d, backend="b200"), Field(g, u)).values
    assert np.max(np.abs(got - m @ u)) <= 1e-13 * np.max(np.abs(m @ u))


def _impulse(g):
    u = zeros_field(g)
    u.values[linear_index(g, g.nx // 2, g.ny // 2, g.nz // 2)] = 1.0
    return u


def test_known_answers_on_b200():
    g = Grid3D(3, 3, 3)  # dx = 1/4: centre 6/dx^2 = 96, neighbours -1/dx^2 = -16
    op = StencilOperator(g, BCS["homogeneous"], backend="b200")
    y = apply(op, _impulse(g)).values
    assert y[linear_index(g, 1, 1, 1)] == 96.0 and np.count_nonzero(y) == 7
    for nb in [(0, 1, 1), (2, 1, 1), (1, 0, 1), (1, 2, 1), (1, 1, 0), (1, 1, 2)]:
        assert y[linear_index(g, *nb)] == -16.0
    assert fused_apply(op, 2.0, 1.0, _impulse(g)).values[linear_index(g, 1, 1, 1)] == 193.0
    sc = apply(StencilOperator(g, BCS["homogeneous"], coeff=coeff_d, backend="b200"), _impulse(g)).values
    assert sc[linear_index(g, 1, 1, 1)] == pytest.approx(96.0 / math.sqrt(1.5), rel=1e-14)
    assert np.all(apply(op, zeros_field(g)).values == 0.0)
    g1 = Grid3D(3, 1, 1)  # a 3x1x1 grid is the 1D rule tridiag(32, -16)
    y1 = apply(StencilOperator(g1, BCS["homogeneous"], backend="b200"), Field(g1, np.array([1.0, 0.0, 0.0])))
    assert np.array_equal(y1.values, [32.0, -16.0, 0.0])
    # affine split at the corner: b = -(1/dx^2) (f at the three ghost positions)
    fn = BCS["poly"].fn
    b = boundary_source_field(StencilOperator(g, BCS["poly"], backend="b200")).values
    dx = g.dx
    assert b[0] == pytest.approx(-(fn(0.0, dx, dx) + fn(dx, 0.0, dx) + fn(dx, dx, 0.0)) / dx**2, rel=1e-14)


@pytest.mark.parametrize("bc", list(BCS))
def test_traversal_invariance_over_every_backend(bc):
    g = Grid3D(9, 7, 5)
    u = Field(g, np.random.default_rng(49).standard_normal(g.n))
    results = []
    for backend in _kernels.available_backends():
        for t in ("naive", "tiled"):
            results.append(apply(StencilOperator(g, BCS[bc], traversal=t, tile=(4, 2), backend=backend), u).values)
    assert len(results) >= 4
    assert all(np.array_equal(results[0], r) for r in results)


def test_affine_split_contract_on_b200():
    g = Grid3D(5, 4, 3)
    rng = np.random.default_rng(50)
    for name in ("poly", "trig"):
        op = StencilOperator(g, BCS[name], backend="b200")
        u = Field(g, rng.standard_normal(g.n))
        hom, b = apply_affine_split(op, u)
        full = apply(op, u)
        assert np.max(np.abs(hom.values + b.values - full.values)) <= 1e-12 * np.max(np.abs(full.values))
        _, b2 = apply_affine_split(op, Field(g, rng.standard_normal(g.n)))
        assert np.array_equal(b.values, b2.values)
    opz = StencilOperator(g, BoundaryCondition.function(lambda x, y, z: 0.0 * x, "0"), backend="b200")
    assert np.all(apply_affine_split(opz, zeros_field(g))[1].values == 0.0)


def test_complex_field_apply_on_b200():
    g = Grid3D(4, 4, 4)
    op = StencilOperator(g, BCS["homogeneous"], backend="b200")
    rng = np.random.default_rng(51)
    z = rng.standard_normal(g.n) + 1j * rng.standard_normal(g.n)
    got = op.fused_apply_flat(2.0, 0.5, z)
    re = op.fused_apply_flat(1.0, 0.0, z.real.copy())
    im = op.fused_apply_flat(1.0, 0.0, z.imag.copy())
    assert np.array_equal(got, 2.0 * (re + 1j * im) + 0.5 * z)


# ---------------------------------------------------------------------------
# the whole reference on the B200 kernels ("b200" as the default backend)


@pytest.fixture
def b200_default():
    b200.install(_kernels, default=True)
    yield
    _kernels._DEFAULT = _kernels._b200_saved_default
    del _kernels._b200_saved_default


def _run_reference_flows():
    from expstencil.decomp import PartitionedCsr, PartitionedStencil, make_partition
    from expstencil.integrator import SemilinearProblem, StepperConfig, combustion_g, integrate
    from expstencil.matfunc import gershgorin_interval, make_interpolant, newton_apply

    out = {}
    g = Grid3D(24, 20, 16)
    op = StencilOperator(g, BCS["homogeneous"], coeff=coeff_d)
    rng = np.random.default_rng(52)
    v = rng.standard_normal(g.n)
    it = make_interpolant(gershgorin_interval(op), "phi1", -3e-4, 150, 1e-8)
    out["newton"] = newton_apply(op, it, v, 1e-8)
    pop = PartitionedStencil(op, make_partition(g, 3))
    out["partitioned"] = newton_apply(pop, it, v, 1e-8)
    pop.close()
    u0 = 1.0 + 0.1 * rng.random(g.n)
    obs = []
    prob = SemilinearProblem(operator=StencilOperator(g, BCS["homogeneous"]),
                             nonlinearity=lambda u: combustion_g(u), u0=u0)
    out["trajectory"] = integrate(prob, StepperConfig(h=1e-4, t_end=3e-4, tol=1e-6),
                                  observer=lambda k, t, mv, mx: obs.append(mv))
    out["obs"] = obs
    dense = rng.standard_normal((900, 900)) * (rng.random((900, 900)) < 0.02)
    a = CsrMatrix.from_dense(dense + dense.T + 40 * np.eye(900))
    ita = make_interpolant(gershgorin_interval(a), "exp", -1e-2, 150, 1e-10)
    x = rng.standard_normal(900)
    out["csr"] = newton_apply(a, ita, x, 1e-10)
    pa = PartitionedCsr(a, make_partition(a, 3))
    out["partitioned_csr"] = newton_apply(pa, ita, x, 1e-10)
    pa.close()
    return out


def test_reference_flows_on_b200_match_compiled(b200_default):
    on_b200 = _run_reference_flows()
    _kernels._DEFAULT = "compiled"
    on_core = _run_reference_flows()
    for key in ("newton", "partitioned", "csr", "partitioned_csr"):
        (p0, m0), (p1, m1) = on_b200[key], on_core[key]
        assert m0 == m1 and p0.tobytes() == p1.tobytes(), key
    assert on_b200["obs"] == on_core["obs"]
    t0, t1 = on_b200["trajectory"], on_core["trajectory"]
    assert np.max(np.abs(t0 - t1)) <= 1e-12 * np.max(np.abs(t1))  # CUDA exp vs libm inside g(u)
