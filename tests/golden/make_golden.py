"""Generate the golden fixtures in tests/golden/*.npz FROM THE REFERENCE ITSELF.

Run in the build container only (needs the reference built by
``oracle/build_ref.sh`` into ``oracle/_ref``):

    ./oracle/build_ref.sh && python tests/golden/make_golden.py

Every fixture stores its inputs next to the reference outputs, so the tests
never depend on RNG streams.  Calls go through the reference's public API
(StencilOperator.fused_apply_flat / apply, the kernel module's
stencil_fused_slab for slab + halo cases, newton_apply, make_interpolant,
apply_matfunc, integrate, CsrMatrix, combustion_g) with its compiled (Cython)
backend.  The reference's combustion stepper bug is
worked around by passing a one-argument nonlinearity.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref"))

os.environ.setdefault("EXPSTENCIL_KERNELS", "compiled")

import expstencil  # noqa: E402
from expstencil import _kernels  # noqa: E402
from expstencil.expr import parse_expression  # noqa: E402
from expstencil.grid import Field, Grid3D  # noqa: E402
from expstencil.integrator import SemilinearProblem, StepperConfig, combustion_g, integrate  # noqa: E402
from expstencil.matfunc import (  # noqa: E402
    apply_matfunc,
    canonical_leja_points,
    gershgorin_interval,
    make_interpolant,
    newton_apply,
)
from expstencil.sparse import CsrMatrix  # noqa: E402
from expstencil.stencil import BoundaryCondition, StencilOperator, apply, boundary_faces  # noqa: E402

assert _kernels.default_backend() == "compiled", "golden vectors must come from the compiled core"


def coeff_d(x, y, z):
    return 1.0 / np.sqrt(1.0 + x * x + y * y)


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) // 1024} KiB)")


def bc_of(name):
    return {
        "none": BoundaryCondition.none(),
        "homogeneous": BoundaryCondition.homogeneous(),
        "poly": BoundaryCondition.function(parse_expression("z*(1-z)*x*y"), "z*(1-z)*x*y"),
        "trig": BoundaryCondition.function(parse_expression("sin(pi*z)*exp(-x*y)"), "sin(pi*z)*exp(-x*y)"),
    }[name]


def stencil_cases():
    """Single fused applies: grids x BCs x coefficient, plus slab/halo calls."""
    rng = np.random.default_rng(101)
    out = {}
    cases = []
    grids = [(5, 5, 5), (9, 9, 9), (7, 5, 3), (9, 7, 5), (37, 23, 19), (33, 17, 1), (3, 1, 1), (1, 4, 6)]
    for dims in grids:
        for bc in ("none", "homogeneous", "poly", "trig"):
            for coeff in (False, True):
                if coeff and bc in ("poly", "trig") and dims != (9, 7, 5):
                    continue
                cases.append((dims, bc, coeff))
    for i, (dims, bc, coeff) in enumerate(cases):
        g = Grid3D(*dims)
        op = StencilOperator(g, bc_of(bc), coeff=coeff_d if coeff else None)
        x = rng.standard_normal(g.n)
        if bc in ("poly", "trig"):
            y = apply(op, Field(g, x)).values
            alpha, beta = 1.0, 0.0
            faces = boundary_faces(op, np.float64)
            for j, f in enumerate(faces):
                out[f"c{i}_face{j}"] = f
        else:
            alpha, beta = float(rng.uniform(0.1, 3.0)), float(rng.uniform(-2.0, 2.0))
            y = op.fused_apply_flat(alpha, beta, x)
        out[f"c{i}_dims"] = np.array(dims)
        out[f"c{i}_bc"] = np.array(bc)
        out[f"c{i}_coeff"] = np.array(coeff)
        out[f"c{i}_ab"] = np.array([alpha, beta])
        out[f"c{i}_x"] = x
        out[f"c{i}_y"] = y
    out["ncases"] = np.array(len(cases))
    save("stencil_apply", **out)


def slab_cases():
    """Kernel-module calls on one z-slab with halo planes (decomp.py:207-232)."""
    k = _kernels.get_kernels("compiled")
    rng = np.random.default_rng(102)
    out = {}
    cases = [((11, 9, 12), 0, 5), ((11, 9, 12), 5, 4), ((11, 9, 12), 9, 3), ((16, 16, 8), 2, 4)]
    for i, (dims, z0, lz) in enumerate(cases):
        g = Grid3D(*dims)
        op = StencilOperator(g, BoundaryCondition.homogeneous(), coeff=coeff_d if i % 2 else None)
        x = rng.standard_normal(g.n)
        x3 = x.reshape(g.shape)
        lo = x3[z0 - 1].copy() if z0 > 0 else None
        hi = x3[z0 + lz].copy() if z0 + lz < g.nz else None
        o3 = np.empty((lz, g.ny, g.nx))
        coeff3 = op.coeff_values("f64")
        k.stencil_fused_slab(x3[z0:z0 + lz].copy(), o3, 1.5, -0.25, op.weights(), 0,
                             halo_lo=lo, halo_hi=hi, z0=z0, nz_total=g.nz,
                             coeff3=None if coeff3 is None else coeff3[z0:z0 + lz].copy())
        out[f"s{i}_dims"] = np.array(dims)
        out[f"s{i}_z"] = np.array([z0, lz])
        out[f"s{i}_coeff"] = np.array(coeff3 is not None)
        out[f"s{i}_x"] = x
        out[f"s{i}_y"] = o3.reshape(-1)
    out["ncases"] = np.array(len(cases))
    save("stencil_slab", **out)


def leja_cases():
    """Canonical Leja nodes and divided differences (matfunc.py:122-268)."""
    out = {"canonical": canonical_leja_points(151)}
    specs = [
        (0.0, 5.284e5, "exp", -1e-4), (0.0, 5.284e5, "phi1", -1e-4),
        (0.0, 3.158e6, "exp", -2.5e-5), (0.0, 3.158e6, "phi1", -2.5e-5),
        (0.0, 64.0, "exp", -0.1), (-2.85, 26.85, "phi1", -1.0), (3.0, 3.0, "phi1", -0.5),
    ]
    for i, (a, b, tgt, s) in enumerate(specs):
        it = make_interpolant(expstencil.SpectralInterval(a, b), tgt, s, 150, 1e-8)
        out[f"i{i}_spec"] = np.array([a, b, s])
        out[f"i{i}_target"] = np.array(tgt)
        out[f"i{i}_xi"] = it.xi
        out[f"i{i}_dd"] = it.dd
    out["ncases"] = np.array(len(specs))
    save("leja", **out)


def newton_cases():
    """newton_apply on stencil operators: fixed degree (tol=0) and truncated."""
    rng = np.random.default_rng(103)
    out = {}
    cases = [
        ((37, 23, 19), "homogeneous", False, "phi1", -3e-4, 0.0, 25),
        ((37, 23, 19), "homogeneous", True, "phi1", -3e-4, 0.0, 25),
        ((37, 23, 19), "homogeneous", False, "exp", -3e-4, 1e-8, 150),
        ((37, 23, 19), "homogeneous", True, "phi1", -3e-4, 1e-6, 150),
        ((64, 48, 1), "homogeneous", False, "exp", -1e-4, 1e-4, 150),
        ((64, 48, 1), "homogeneous", True, "phi1", -1e-4, 1e-8, 150),
        ((16, 16, 16), "none", False, "exp", -1e-3, 1e-8, 150),
        ((40, 30, 20), "homogeneous", False, "exp", -1e-2, 1e-8, 40),  # exhausts -> ConvergenceError
    ]
    for i, (dims, bc, coeff, tgt, s, tol, maxdeg) in enumerate(cases):
        g = Grid3D(*dims)
        op = StencilOperator(g, bc_of(bc), coeff=coeff_d if coeff else None)
        iv = gershgorin_interval(op)
        it = make_interpolant(iv, tgt, s, maxdeg, tol if tol > 0 else 1e-8)
        v = rng.standard_normal(g.n)
        try:
            p, mv = newton_apply(op, it, v, tol)
            err = np.array([0.0, 0.0])
        except expstencil.errors.ConvergenceError as e:
            p, mv = np.zeros(0), -1
            err = np.array([e.residual, e.degree])
        out[f"n{i}_dims"] = np.array(dims)
        out[f"n{i}_bc"] = np.array(bc)
        out[f"n{i}_coeff"] = np.array(coeff)
        out[f"n{i}_target"] = np.array(tgt)
        out[f"n{i}_params"] = np.array([s, tol, maxdeg, iv.a, iv.b])
        out[f"n{i}_xi"] = it.xi
        out[f"n{i}_dd"] = it.dd
        out[f"n{i}_v"] = v
        out[f"n{i}_p"] = p
        out[f"n{i}_mv"] = np.array(mv)
        out[f"n{i}_err"] = err
    out["ncases"] = np.array(len(cases))
    save("newton", **out)


def step_cases():
    """Exponential Euler trajectories with the combustion term (C1 scaled down)."""
    rng = np.random.default_rng(104)
    out = {}
    cases = [((32, 32, 1), 1e-4, 1e-4, 3), ((17, 17, 17), 1e-4, 1e-4, 2), ((24, 20, 1), 1e-3, 1e-6, 2),
             ((64, 64, 1), 2e-3, 1e-4, 3), ((24, 22, 20), 1e-3, 1e-4, 2)]
    for i, (dims, h, tol, nsteps) in enumerate(cases):
        g = Grid3D(*dims)
        op = StencilOperator(g, BoundaryCondition.homogeneous())
        u0 = 1.0 + 0.1 * rng.random(g.n)
        obs = []
        prob = SemilinearProblem(operator=op, nonlinearity=lambda u: combustion_g(u), u0=u0)
        u = integrate(prob, StepperConfig(h=h, t_end=h * nsteps, tol=tol),
                      observer=lambda k, t, mv, mx: obs.append((k, t, mv, mx)))
        out[f"t{i}_dims"] = np.array(dims)
        out[f"t{i}_params"] = np.array([h, tol, nsteps])
        out[f"t{i}_u0"] = u0
        out[f"t{i}_u"] = u
        out[f"t{i}_obs"] = np.array(obs)
    out["ncases"] = np.array(len(cases))
    save("expeuler", **out)


def rescue_cases():
    """apply_matfunc halving rescue (matfunc.py:328-373)."""
    rng = np.random.default_rng(105)
    g = Grid3D(20, 18, 16)
    op = StencilOperator(g, BoundaryCondition.homogeneous())
    out = {}
    for i, tgt in enumerate(("exp", "phi1")):
        v = rng.standard_normal(g.n)
        y, st = apply_matfunc(op, v, tgt, -3e-2, tol=1e-8, max_degree=40)
        out[f"r{i}_target"] = np.array(tgt)
        out[f"r{i}_v"] = v
        out[f"r{i}_y"] = y
        out[f"r{i}_stats"] = np.array([st.matvecs, st.degree, st.halvings])
    out["dims"] = np.array([20, 18, 16])
    out["params"] = np.array([-3e-2, 1e-8, 40])
    save("rescue", **out)


def csr_cases():
    """CSR fused SpMV (sequential row sums) and a phi1 series (sparse.py:185-192)."""
    rng = np.random.default_rng(106)
    n, r = 3000, 5
    rows = np.repeat(np.arange(n), r)
    cols = rng.integers(0, n, size=n * r)
    vals = -rng.random(n * r)
    rr = np.concatenate([rows, cols, np.arange(n)])
    cc = np.concatenate([cols, rows, np.arange(n)])
    vv = np.concatenate([vals, vals, np.full(n, 12.0)])
    a = CsrMatrix.from_coo(n, n, rr, cc, vv, sum_duplicates=True)
    x = rng.standard_normal(n)
    y = a.fused_apply_flat(0.7, -1.3, x)
    iv = gershgorin_interval(a)
    it = make_interpolant(iv, "phi1", -1.0, 150, 1e-8)
    p, mv = newton_apply(a, it, x, 1e-8)
    p0, mv0 = newton_apply(a, it, x, 0.0)
    save("csr", n=np.array(n), row_ptr=a.row_ptr, col=a.col_idx, vals=a.vals, x=x, y=y,
         interval=np.array([iv.a, iv.b]), xi=it.xi, dd=it.dd, p=p, mv=np.array(mv), p0=p0,
         mv0=np.array(mv0))


MM_GOOD = {
    "sym": "%%MatrixMarket matrix coordinate real symmetric\n% comment\n4 4 5\n1 1 2.5\n2 1 -1\n3 2 -0.5\n"
           "4 4 3\n4 3 1e-3\n",
    "herm": "%%MatrixMarket matrix coordinate complex hermitian\n3 3 4\n1 1 1 0\n2 1 0.5 -0.25\n3 3 2 0\n"
            "3 2 0 1\n",
    "skew": "%%MatrixMarket matrix coordinate real skew-symmetric\n3 3 2\n2 1 1.5\n3 1 -2\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n\n3 4 3\n1 2\n3 4 7.5\n2 1\n",
    "general": "%%MatrixMarket matrix coordinate integer general\n2 3 3\n2 3 4\n1 1 -2\n1 3 5\n",
}
MM_BAD = {
    "header": "%%MatrixMarket matrix array real general\n2 2 1\n1 1 1\n",
    "field": "%%MatrixMarket matrix coordinate quaternion general\n2 2 1\n1 1 1\n",
    "size": "%%MatrixMarket matrix coordinate real general\n% c\n2 2\n1 1 1\n",
    "bounds": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n3 1 2\n",
    "value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 x\n",
    "upper": "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1\n1 2 3\n",
    "hdiag": "%%MatrixMarket matrix coordinate complex hermitian\n2 2 1\n1 1 1 2\n",
    "dup": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n2 2 1\n1 1 4\n",
    "count": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n2 2 1\n",
    "extra": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n2 2 1\n",
    "square": "%%MatrixMarket matrix coordinate real symmetric\n2 3 1\n1 1 1\n",
}


def csr_complex_cases():
    """The propagate path (cli.py:304-357): complex CSR rows for real and
    Hermitian matrices (_core.pyx:263-278), complex Newton series on real-
    and imaginary-axis intervals, exp(-i t H) psi0 through apply_matfunc with
    halving, and Matrix Market parsing (sparse.py:292-428)."""
    import tempfile

    from expstencil.errors import MatrixMarketError
    from expstencil.matfunc import SpectralInterval
    from expstencil.sparse import read_matrix_market, spmv

    rng = np.random.default_rng(108)
    out = {}
    n = 700
    mats = {}
    d = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.02)
    d = d + d.T + np.diag(rng.random(n) * 4.0)
    mats["real"] = CsrMatrix.from_dense(d)
    hmat = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * (rng.random((n, n)) < 0.02)
    hmat = hmat + hmat.conj().T + np.diag(rng.random(n))
    mats["herm"] = CsrMatrix.from_dense(hmat)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    out["x"] = x
    for name, m in mats.items():
        out[f"{name}_row_ptr"], out[f"{name}_col"], out[f"{name}_vals"] = m.row_ptr, m.col_idx, m.vals
        out[f"{name}_y"] = m.fused_apply_flat(0.7 - 0.2j, -1.3, x)
        out[f"{name}_spmv"] = spmv(m, x)
        k = 0
        for axis, target, scale in (("real", "exp", -0.8j), ("real", "phi1", -0.5j), ("imag", "exp", -0.8)):
            iv = gershgorin_interval(m, axis)
            it = make_interpolant(iv, target, scale, 100, 1e-10)
            for tol in (0.0, 1e-10):
                p, mv = newton_apply(m, it, x, tol)
                key = f"{name}_s{k}"
                out[key + "_meta"] = np.array([iv.a, iv.b, tol, mv])
                out[key + "_axis"] = np.array(axis)
                out[key + "_target"] = np.array(target)
                out[key + "_scale"] = np.array(scale, dtype=np.complex128)
                out[key + "_dd"], out[key + "_xi"], out[key + "_p"] = it.dd, it.xi, p
                k += 1
        out[f"{name}_nseries"] = np.array(k)
        # exp(-i t H) psi0 with a degree cap that forces the halving rescue
        psi0 = np.full(n, 1.0 / np.sqrt(n), dtype=np.complex128)
        iv = gershgorin_interval(m)
        psi, st = apply_matfunc(m, psi0, "exp", scale=-1j * 3.0, interval=iv, tol=1e-8, max_degree=40)
        out[f"{name}_psi"] = psi
        out[f"{name}_prop_stats"] = np.array([st.matvecs, st.degree, st.halvings])
    # Matrix Market
    with tempfile.TemporaryDirectory() as tmp:
        for name, text in MM_GOOD.items():
            path = os.path.join(tmp, name + ".mtx")
            with open(path, "w") as fh:
                fh.write(text)
            a = read_matrix_market(path)
            out[f"mm_{name}_text"] = np.array(text)
            out[f"mm_{name}"] = np.array([a.nrows, a.ncols])
            out[f"mm_{name}_row_ptr"], out[f"mm_{name}_col"], out[f"mm_{name}_vals"] = a.row_ptr, a.col_idx, a.vals
        for name, text in MM_BAD.items():
            path = os.path.join(tmp, name + ".mtx")
            with open(path, "w") as fh:
                fh.write(text)
            try:
                read_matrix_market(path)
                raise AssertionError(f"{name} parsed")
            except MatrixMarketError as err:
                out[f"mmbad_{name}_text"] = np.array(text)
                out[f"mmbad_{name}_line"] = np.array(err.line)
                out[f"mmbad_{name}_msg"] = np.array(str(err))
    out["mm_good"] = np.array(sorted(MM_GOOD))
    out["mm_bad"] = np.array(sorted(MM_BAD))
    save("csr_complex", **out)


def combustion_cases():
    rng = np.random.default_rng(107)
    u = rng.uniform(0.05, 2.5, 5000)
    save("combustion", u=u, g=combustion_g(u))


def field_cases():
    """Field binary files as the reference writes them (grid.py:178-206)."""
    import tempfile

    from expstencil.grid import write_field_binary

    rng = np.random.default_rng(109)
    out = {}
    cases = {"f64": (Grid3D(5, 4, 3), rng.standard_normal(60)),
             "f32": (Grid3D(7, 1, 2), rng.standard_normal(14).astype(np.float32)),
             "c128": (Grid3D(3, 3, 1), rng.standard_normal(9) + 1j * rng.standard_normal(9))}
    with tempfile.TemporaryDirectory() as tmp:
        for kind, (g, v) in cases.items():
            path = os.path.join(tmp, kind + ".bin")
            write_field_binary(Field(g, v), path)
            out[f"{kind}_dims"] = np.array([g.nx, g.ny, g.nz])
            out[f"{kind}_values"] = v
            out[f"{kind}_bytes"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
    save("field_binary", **out)


def f32_cases():
    """The reference's float kernels: fused stencil applies on f32 fields
    (all boundary kinds, coefficient, slab + halos through the kernel
    module), combustion on f32, and a float32 CSR matrix (promoted to f64)."""
    from expstencil.sparse import fused_spmv

    k = _kernels.get_kernels("compiled")
    rng = np.random.default_rng(110)
    out = {}
    cases = []
    for dims in ((12, 10, 8), (16, 16, 1), (7, 5, 3), (1, 4, 6)):
        for bc in ("none", "homogeneous", "poly"):
            for coeff in (False, True):
                cases.append((dims, bc, coeff))
    for i, (dims, bc, coeff) in enumerate(cases):
        g = Grid3D(*dims)
        op = StencilOperator(g, bc_of(bc), coeff=coeff_d if coeff else None)
        x = rng.standard_normal(g.n).astype(np.float32)
        if bc == "poly":
            y = apply(op, Field(g, x)).values
            ab = (1.0, 0.0)
        else:
            ab = (float(rng.uniform(0.1, 3.0)), float(rng.uniform(-2.0, 2.0)))
            y = op.fused_apply_flat(ab[0], ab[1], x)
        assert y.dtype == np.float32
        out[f"c{i}_dims"], out[f"c{i}_bc"], out[f"c{i}_coeff"] = np.array(dims), np.array(bc), np.array(coeff)
        out[f"c{i}_ab"], out[f"c{i}_x"], out[f"c{i}_y"] = np.array(ab), x, y
    out["ncases"] = np.array(len(cases))
    # slab with halos, float
    g = Grid3D(11, 9, 12)
    op = StencilOperator(g, BoundaryCondition.homogeneous(), coeff=coeff_d)
    x = rng.standard_normal(g.n).astype(np.float32)
    x3 = x.reshape(g.shape)
    z0, lz = 5, 4
    o3 = np.empty((lz, g.ny, g.nx), dtype=np.float32)
    c3 = op.coeff_values("f32")[z0:z0 + lz].copy()
    k.stencil_fused_slab(x3[z0:z0 + lz].copy(), o3, 1.5, -0.25, op.weights(), 0, halo_lo=x3[z0 - 1].copy(),
                         halo_hi=x3[z0 + lz].copy(), z0=z0, nz_total=g.nz, coeff3=c3)
    out["slab_x"], out["slab_y"] = x, o3.reshape(-1)
    # combustion on float32
    u = rng.uniform(0.05, 2.5, 4000).astype(np.float32)
    out["comb_u"], out["comb_g"] = u, combustion_g(u)
    # float32 CSR values
    n = 500
    dense = (rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.03)).astype(np.float32)
    a = CsrMatrix.from_dense(dense)
    xv = rng.standard_normal(n)
    out["csr_row_ptr"], out["csr_col"], out["csr_vals"], out["csr_x"] = a.row_ptr, a.col_idx, a.vals, xv
    out["csr_y"] = fused_spmv(a, 0.7, -1.3, xv)
    save("f32", **out)


def c1_trajectory_case():
    """BASELINE config 1 at full size: 256x256 homogeneous Dirichlet,
    combustion, exponential Euler h=1e-4, tol=1e-4, 10 steps through
    integrate() with its observer (integrator.py:209-239).  u0 = 1 + 0.1 U[0,1)
    from default_rng(1234), the bench's seeding."""
    g = Grid3D(256, 256, 1)
    op = StencilOperator(g, BoundaryCondition.homogeneous())
    u0 = 1.0 + 0.1 * np.random.default_rng(1234).random(g.n)
    h, tol, nsteps = 1e-4, 1e-4, 10
    obs = []
    prob = SemilinearProblem(operator=op, nonlinearity=lambda u: combustion_g(u), u0=u0)
    u = integrate(prob, StepperConfig(h=h, t_end=h * nsteps, tol=tol),
                  observer=lambda k, t, mv, mx: obs.append((k, t, mv, mx)))
    save("c1_trajectory", u0=u0, u=u, obs=np.array(obs), params=np.array([h, tol, nsteps]),
         dims=np.array([256, 256, 1]))


def split_cases():
    """Dirichlet-function boundaries through the affine split
    (stencil.py:281-312): apply_affine_split, homogeneous_part applies,
    boundary_source_field, and exponential-Euler trajectories on the split
    problem (forcing g - b, integrator.py:104-123)."""
    from expstencil.grid import Field as RField
    from expstencil.stencil import apply_affine_split, boundary_source_field, homogeneous_part

    rng = np.random.default_rng(106)
    out = {}
    cases = [((9, 7, 5), "poly", False), ((9, 7, 5), "trig", True), ((33, 17, 1), "trig", False),
             ((24, 20, 16), "poly", True), ((40, 36, 1), "trig", True)]
    for i, (dims, bc, coeff) in enumerate(cases):
        g = Grid3D(*dims)
        op = StencilOperator(g, bc_of(bc), coeff=coeff_d if coeff else None)
        x = rng.standard_normal(g.n)
        hom, b = apply_affine_split(op, RField(g, x))
        bs = boundary_source_field(op)
        hp = homogeneous_part(op)
        y = hp.fused_apply_flat(0.75, -0.5, x)
        full = apply(op, RField(g, x)).values
        out[f"s{i}_dims"], out[f"s{i}_bc"], out[f"s{i}_coeff"] = np.array(dims), np.array(bc), np.array(coeff)
        out[f"s{i}_x"] = x
        out[f"s{i}_hom"], out[f"s{i}_b"], out[f"s{i}_bsrc"] = hom.values, b.values, bs.values
        out[f"s{i}_hp_y"], out[f"s{i}_full"] = y, full
        for j, f in enumerate(boundary_faces(op, np.float64)):
            out[f"s{i}_face{j}"] = f
    out["ncases"] = np.array(len(cases))
    # trajectories on the split problem: du/dt + A_hom u = g(u) - b
    traj = [((32, 32, 1), "trig", False, True, 2e-4, 1e-6, 3), ((20, 18, 16), "poly", True, True, 2e-4, 1e-6, 2),
            ((48, 40, 1), "poly", False, False, 1e-3, 1e-8, 2)]
    for i, (dims, bc, coeff, nonlin, h, tol, nsteps) in enumerate(traj):
        g = Grid3D(*dims)
        op = StencilOperator(g, bc_of(bc), coeff=coeff_d if coeff else None)
        b = boundary_source_field(op).values
        u0 = 1.0 + 0.1 * rng.random(g.n)
        obs = []
        prob = SemilinearProblem(operator=homogeneous_part(op),
                                 nonlinearity=(lambda u: combustion_g(u)) if nonlin else None, u0=u0,
                                 boundary_source=b)
        u = integrate(prob, StepperConfig(h=h, t_end=h * nsteps, tol=tol),
                      observer=lambda k, t, mv, mx: obs.append((k, t, mv, mx)))
        out[f"t{i}_dims"], out[f"t{i}_bc"], out[f"t{i}_coeff"] = np.array(dims), np.array(bc), np.array(coeff)
        out[f"t{i}_nonlin"] = np.array(nonlin)
        out[f"t{i}_params"] = np.array([h, tol, nsteps])
        out[f"t{i}_u0"], out[f"t{i}_b"], out[f"t{i}_u"], out[f"t{i}_obs"] = u0, b, u, np.array(obs)
        for j, f in enumerate(boundary_faces(op, np.float64)):
            out[f"t{i}_face{j}"] = f
    out["ntraj"] = np.array(len(traj))
    save("split", **out)


if __name__ == "__main__":
    if len(sys.argv) > 1:  # regenerate selected fixtures only: make_golden.py split c1_trajectory
        for name in sys.argv[1:]:
            globals()[name + ("_case" if name == "c1_trajectory" else "_cases")]()
        sys.exit(0)
    c1_trajectory_case()
    split_cases()
    stencil_cases()
    slab_cases()
    leja_cases()
    newton_cases()
    step_cases()
    rescue_cases()
    csr_cases()
    combustion_cases()
    csr_complex_cases()
    field_cases()
    f32_cases()
