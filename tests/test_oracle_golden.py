"""Pin the CPU oracle (oracle/) against golden vectors the reference produced.

Bitwise where the reference arithmetic is reproducible (stencil points, the
Newton-Leja recurrence for equal matvec counts, sequential CSR rows); within
1 ulp-scale tolerances where the reference calls libm/numpy transcendental
functions that the oracle also calls (combustion exp) or where stepping
composes several series.
"""

import numpy as np
import pytest

from oracle import oracle as orc

MODES = {"none": orc.MODE_PERIODIC, "homogeneous": orc.MODE_ZERO, "poly": orc.MODE_FACES,
         "trig": orc.MODE_FACES}


def _spec(dims, bc, coeff, faces=None):
    nx, ny, nz = (int(d) for d in dims)
    return orc.StencilSpec(nx, ny, nz, mode=MODES[str(bc)],
                           coeff_kind=orc.COEFF_RADIAL if bool(coeff) else orc.COEFF_NONE,
                           faces=faces)


def test_stencil_apply_bitwise(golden, oracle):
    d = golden("stencil_apply")
    for i in range(int(d["ncases"])):
        faces = None
        if str(d[f"c{i}_bc"]) in ("poly", "trig"):
            faces = tuple(d[f"c{i}_face{j}"] for j in range(6))
        spec = _spec(d[f"c{i}_dims"], d[f"c{i}_bc"], d[f"c{i}_coeff"], faces)
        a, b = d[f"c{i}_ab"]
        got = oracle.stencil_fused(spec, a, b, d[f"c{i}_x"])
        assert np.array_equal(got, d[f"c{i}_y"]), f"case {i}"
        # sign of zero too (sha256-level identity)
        assert got.tobytes() == d[f"c{i}_y"].tobytes(), f"case {i} bytes"


def test_stencil_slab_halo_bitwise(golden, oracle):
    d = golden("stencil_slab")
    for i in range(int(d["ncases"])):
        nx, ny, nz = (int(v) for v in d[f"s{i}_dims"])
        z0, lz = (int(v) for v in d[f"s{i}_z"])
        spec = orc.StencilSpec(nx, ny, nz, coeff_kind=orc.COEFF_RADIAL if bool(d[f"s{i}_coeff"]) else 0)
        x3 = d[f"s{i}_x"].reshape(nz, ny, nx)
        lo = x3[z0 - 1] if z0 > 0 else None
        hi = x3[z0 + lz] if z0 + lz < nz else None
        coeff = None
        if spec.coeff_kind:
            spec = orc.StencilSpec(nx, ny, nz, coeff_kind=orc.COEFF_ARRAY,
                                   coeff=spec.coeff_grid()[z0:z0 + lz].copy())
        got = oracle.stencil_fused(spec, 1.5, -0.25, x3[z0:z0 + lz].reshape(-1), z0=z0,
                                   halo_lo=lo, halo_hi=hi, coeff=coeff)
        assert got.tobytes() == d[f"s{i}_y"].tobytes(), f"slab case {i}"


def test_radial_coefficient_matches_eval_on_grid(oracle):
    # in-kernel D formula == the numpy-sampled coefficient, bit for bit
    spec = orc.StencilSpec(4096, 64, 1, coeff_kind=orc.COEFF_RADIAL)
    x = np.arange(1, 4097, dtype=np.float64) / 4097
    y = np.arange(1, 65, dtype=np.float64) / 65
    X, Y = np.meshgrid(x, y)
    ref = 1.0 / np.sqrt(1.0 + X * X + Y * Y)
    assert np.array_equal(spec.coeff_grid()[0], ref)


def test_leja_points_and_divided_differences(golden):
    d = golden("leja")
    assert np.array_equal(orc.canonical_leja(151), d["canonical"])
    for i in range(int(d["ncases"])):
        a, b, s = d[f"i{i}_spec"]
        it = orc.interpolant(a, b, str(d[f"i{i}_target"]), s, 150)
        assert np.array_equal(it.xi, d[f"i{i}_xi"])
        # same numpy ops in the same order: bitwise on the same BLAS build
        np.testing.assert_allclose(it.dd, d[f"i{i}_dd"], rtol=1e-13, atol=0)


def test_newton_series(golden, oracle):
    d = golden("newton")
    for i in range(int(d["ncases"])):
        spec = _spec(d[f"n{i}_dims"], d[f"n{i}_bc"], d[f"n{i}_coeff"])
        s, tol, maxdeg, a, b = d[f"n{i}_params"]
        it = orc.Interp(a, b, str(d[f"n{i}_target"]), s, d[f"n{i}_xi"], d[f"n{i}_dd"])
        if int(d[f"n{i}_mv"]) < 0:
            with pytest.raises(orc.OracleConvergenceError) as ei:
                oracle.newton_stencil(spec, it, d[f"n{i}_v"], tol)
            res, deg = d[f"n{i}_err"]
            assert ei.value.degree == int(deg)
            assert ei.value.residual == pytest.approx(res, rel=1e-10)
            continue
        p, mv = oracle.newton_stencil(spec, it, d[f"n{i}_v"], tol)
        assert mv == int(d[f"n{i}_mv"]), f"case {i}"
        assert p.tobytes() == d[f"n{i}_p"].tobytes(), f"case {i}"


def test_expeuler_trajectory(golden, oracle):
    d = golden("expeuler")
    for i in range(int(d["ncases"])):
        nx, ny, nz = (int(v) for v in d[f"t{i}_dims"])
        h, tol, nsteps = d[f"t{i}_params"]
        spec = orc.StencilSpec(nx, ny, nz)
        u = d[f"t{i}_u0"]
        obs = d[f"t{i}_obs"]
        for k in range(int(nsteps)):
            u, (m1, m2) = oracle.expeuler_step(spec, u, h, tol)
            assert m1 + m2 == int(obs[k, 2]), f"case {i} step {k}"
        ref = d[f"t{i}_u"]
        # exp() in the combustion term is libm on both sides: bitwise here,
        # 1e-12 is the documented cross-platform bound
        assert np.max(np.abs(u - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_csr_rows_and_series(golden, oracle):
    d = golden("csr")
    a = orc.Csr(int(d["n"]), d["row_ptr"], d["col"], d["vals"])
    y = oracle.csr_fused(a, 0.7, -1.3, d["x"])
    assert y.tobytes() == d["y"].tobytes()
    lo, hi = a.gershgorin()
    assert (lo, hi) == tuple(d["interval"])
    it = orc.Interp(lo, hi, "phi1", -1.0, d["xi"], d["dd"])
    p0, mv0 = oracle.newton_csr(a, it, d["x"], 0.0)
    assert mv0 == int(d["mv0"]) and p0.tobytes() == d["p0"].tobytes()
    p, mv = oracle.newton_csr(a, it, d["x"], 1e-8)
    assert mv == int(d["mv"]) and p.tobytes() == d["p"].tobytes()


def test_combustion(golden, oracle):
    d = golden("combustion")
    got = oracle.combustion(d["u"])
    np.testing.assert_allclose(got, d["g"], rtol=2e-16 * 4, atol=0)
    with pytest.raises(ValueError, match="index 3"):
        oracle.combustion(np.array([1.0, 1.0, 2.0, 0.0, -1.0]))


def test_neumann_matches_dense_oracle(oracle):
    # build-defined Neumann ghost (ghost = adjacent interior value) against a
    # brute-force dense assembly of the same rule
    nx, ny, nz = 6, 5, 4
    spec = orc.StencilSpec(nx, ny, nz, mode=orc.MODE_NEUMANN, coeff_kind=orc.COEFF_RADIAL)
    wx, wy, wz = spec.weights()
    n = spec.n
    mat = np.zeros((n, n))
    d = spec.coeff_grid().reshape(-1)
    for iz in range(nz):
        for iy in range(ny):
            for ix in range(nx):
                i = ix + nx * (iy + ny * iz)
                for (sx, sy, sz), w, m in (((1, 0, 0), wx, nx), ((0, 1, 0), wy, ny), ((0, 0, 1), wz, nz)):
                    for st in (-1, 1):
                        jx, jy, jz = ix + st * sx, iy + st * sy, iz + st * sz
                        if 0 <= jx < nx and 0 <= jy < ny and 0 <= jz < nz:
                            mat[i, i] += w * d[i]
                            mat[i, jx + nx * (jy + ny * jz)] -= w * d[i]
    x = np.random.default_rng(5).standard_normal(n)
    got = oracle.stencil_fused(spec, 1.0, 0.0, x)
    ref = mat @ x
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
    lo, hi = spec.gershgorin()
    ev = np.linalg.eigvals(mat)
    assert lo <= ev.real.min() + 1e-9 and ev.real.max() <= hi + 1e-9
    assert lo == 0.0


def test_c1_full_size_trajectory(golden, oracle):
    # BASELINE config 1 at full size (256^2, 10 steps, reference integrate())
    d = golden("c1_trajectory")
    h, tol, nsteps = d["params"]
    nx, ny, nz = (int(v) for v in d["dims"])
    u, obs = oracle.integrate(orc.StencilSpec(nx, ny, nz), d["u0"], h, h * nsteps, tol)
    ref_obs = d["obs"]
    assert [o[2] for o in obs] == [int(m) for m in ref_obs[:, 2]]
    np.testing.assert_allclose([o[3] for o in obs], ref_obs[:, 3], rtol=1e-12, atol=0)
    ref = d["u"]
    assert np.max(np.abs(u - ref)) <= 1e-10 * np.max(np.abs(ref))


def _split_spec(d, p, faces=True):
    nx, ny, nz = (int(v) for v in d[f"{p}_dims"])
    ck = orc.COEFF_RADIAL if bool(d[f"{p}_coeff"]) else orc.COEFF_NONE
    if not faces:
        return orc.StencilSpec(nx, ny, nz, coeff_kind=ck)
    return orc.StencilSpec(nx, ny, nz, mode=orc.MODE_FACES, coeff_kind=ck,
                           faces=tuple(d[f"{p}_face{j}"] for j in range(6)))


def test_affine_split_pieces(golden, oracle):
    # apply_affine_split / homogeneous_part / boundary_source_field
    # (stencil.py:281-312): A u = A_hom u + b, bitwise
    d = golden("split")
    for i in range(int(d["ncases"])):
        p = f"s{i}"
        x = d[f"{p}_x"]
        full = _split_spec(d, p)
        hom = _split_spec(d, p, faces=False)
        b = oracle.stencil_fused(full, 1.0, 0.0, np.zeros_like(x))
        assert b.tobytes() == d[f"{p}_b"].tobytes() == d[f"{p}_bsrc"].tobytes(), p
        assert oracle.stencil_fused(hom, 1.0, 0.0, x).tobytes() == d[f"{p}_hom"].tobytes(), p
        assert oracle.stencil_fused(hom, 0.75, -0.5, x).tobytes() == d[f"{p}_hp_y"].tobytes(), p
        assert oracle.stencil_fused(full, 1.0, 0.0, x).tobytes() == d[f"{p}_full"].tobytes(), p


def test_split_problem_trajectories(golden, oracle):
    # du/dt + A_hom u = g(u) - b (SemilinearProblem.forcing, integrator.py:104-123)
    d = golden("split")
    for i in range(int(d["ntraj"])):
        p = f"t{i}"
        h, tol, nsteps = d[f"{p}_params"]
        u, obs = oracle.integrate(_split_spec(d, p, faces=False), d[f"{p}_u0"], h, h * nsteps, tol,
                                  nonlinear=bool(d[f"{p}_nonlin"]), source=d[f"{p}_b"])
        assert [o[2] for o in obs] == [int(m) for m in d[f"{p}_obs"][:, 2]], p
        ref = d[f"{p}_u"]
        assert np.max(np.abs(u - ref)) <= 1e-12 * np.max(np.abs(ref)), p
