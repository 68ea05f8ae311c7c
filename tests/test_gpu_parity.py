"""Parity of the B200 path (through the C ABI) with the reference's golden
vectors and the CPU oracle.  Bitwise for stencil applies and Newton-Leja
series (equal matvec counts asserted); 1e-12 relative for steps that contain
CUDA exp(); 1e-10 over trajectories."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1309_4616_b200 as es  # noqa: E402
from oracle import oracle as orc  # noqa: E402

from conftest import coeff_d, fresh_stream  # noqa: E402

BCS = {"none": es.BoundaryCondition.none(), "homogeneous": es.BoundaryCondition.homogeneous(),
       "neumann": es.BoundaryCondition.neumann()}
ORC_MODE = {"none": orc.MODE_PERIODIC, "homogeneous": orc.MODE_ZERO, "neumann": orc.MODE_NEUMANN}


def _faces_bc(i, d):
    faces = tuple(d[f"c{i}_face{j}"] for j in range(6))
    return es.BoundaryCondition.function(lambda x, y, z: 0.0 * x, "golden"), faces


def test_stencil_apply_matches_reference_bitwise(golden):
    d = golden("stencil_apply")
    for i in range(int(d["ncases"])):
        g = es.Grid3D(*(int(v) for v in d[f"c{i}_dims"]))
        bc = str(d[f"c{i}_bc"])
        coeff = coeff_d if bool(d[f"c{i}_coeff"]) else None
        x = d[f"c{i}_x"]
        if bc in ("poly", "trig"):
            bcobj, faces = _faces_bc(i, d)
            op = es.StencilOperator(g, bcobj, coeff=coeff)
            out = torch.empty(g.n, dtype=torch.float64, device="cuda")
            xd = torch.from_numpy(x).cuda()
            es.fused_slab(op, 1.0, 0.0, xd.view(g.shape), out.view(g.shape), faces=faces)
            got = out.cpu().numpy()
        else:
            op = es.StencilOperator(g, BCS[bc], coeff=coeff)
            a, b = d[f"c{i}_ab"]
            got = op.fused_apply_flat(a, b, x)
        assert got.tobytes() == d[f"c{i}_y"].tobytes(), f"case {i} {tuple(d[f'c{i}_dims'])} {bc}"


def test_slab_with_halos_bitwise(golden):
    d = golden("stencil_slab")
    for i in range(int(d["ncases"])):
        g = es.Grid3D(*(int(v) for v in d[f"s{i}_dims"]))
        z0, lz = (int(v) for v in d[f"s{i}_z"])
        op = es.StencilOperator(g, es.BoundaryCondition.homogeneous(),
                                coeff=coeff_d if bool(d[f"s{i}_coeff"]) else None)
        x3 = torch.from_numpy(d[f"s{i}_x"]).cuda().view(g.shape)
        lo = x3[z0 - 1].clone() if z0 > 0 else None
        hi = x3[z0 + lz].clone() if z0 + lz < g.nz else None
        out = torch.empty((lz, g.ny, g.nx), dtype=torch.float64, device="cuda")
        es.fused_slab(op, 1.5, -0.25, x3[z0:z0 + lz].clone(), out, halo_lo=lo, halo_hi=hi, z0=z0)
        assert out.cpu().numpy().reshape(-1).tobytes() == d[f"s{i}_y"].tobytes(), f"slab {i}"


def _interp(d, i):
    s, tol, maxdeg, a, b = d[f"n{i}_params"]
    iv = es.SpectralInterval(a, b)
    return es.LejaInterpolant(iv, str(d[f"n{i}_target"]), s, int(maxdeg), tol if tol > 0 else 1e-8,
                              iv.center + iv.halfspan * d[f"n{i}_xi"], d[f"n{i}_xi"], d[f"n{i}_dd"]), tol


@pytest.mark.parametrize("graph", [True, False])
def test_newton_series_matches_reference_bitwise(golden, graph, monkeypatch):
    if not graph:
        monkeypatch.setenv("ES_NO_GRAPH", "1")
    d = golden("newton")
    for i in range(int(d["ncases"])):
        g = es.Grid3D(*(int(v) for v in d[f"n{i}_dims"]))
        op = es.StencilOperator(g, BCS[str(d[f"n{i}_bc"])], coeff=coeff_d if bool(d[f"n{i}_coeff"]) else None)
        it, tol = _interp(d, i)
        if int(d[f"n{i}_mv"]) < 0:
            with pytest.raises(es.ConvergenceError) as ei:
                es.newton_apply(op, it, d[f"n{i}_v"], tol)
            res, deg = d[f"n{i}_err"]
            assert ei.value.degree == int(deg)
            assert ei.value.residual == pytest.approx(res, rel=1e-9)
            continue
        p, mv = es.newton_apply(op, it, d[f"n{i}_v"], tol)
        assert mv == int(d[f"n{i}_mv"]), f"case {i}"
        assert p.tobytes() == d[f"n{i}_p"].tobytes(), f"case {i}"


def test_newton_device_resident_matches_host(golden):
    d = golden("newton")
    g = es.Grid3D(*(int(v) for v in d["n1_dims"]))
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous(), coeff=coeff_d)
    it, tol = _interp(d, 1)
    v = torch.from_numpy(d["n1_v"]).cuda()
    p, mv = es.newton_apply(op, it, v, tol)
    assert isinstance(p, torch.Tensor) and p.is_cuda
    assert p.cpu().numpy().tobytes() == d["n1_p"].tobytes()
    assert torch.equal(v.cpu(), torch.from_numpy(d["n1_v"]))  # input untouched


def test_expeuler_trajectories(golden):
    d = golden("expeuler")
    for i in range(int(d["ncases"])):
        g = es.Grid3D(*(int(v) for v in d[f"t{i}_dims"]))
        h, tol, nsteps = d[f"t{i}_params"]
        op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
        obs = []
        prob = es.SemilinearProblem(operator=op, nonlinearity=es.combustion_g, u0=d[f"t{i}_u0"])
        u = es.integrate(prob, es.StepperConfig(h=h, t_end=h * nsteps, tol=tol),
                         observer=lambda k, t, mv, mx: obs.append((k, t, mv, mx)))
        ref_obs = d[f"t{i}_obs"]
        assert [o[2] for o in obs] == [int(v) for v in ref_obs[:, 2]], f"case {i} matvecs"
        ref = d[f"t{i}_u"]
        assert np.max(np.abs(u - ref)) <= 1e-10 * np.max(np.abs(ref)), f"case {i}"
        np.testing.assert_allclose([o[3] for o in obs], ref_obs[:, 3], rtol=1e-12)


def test_rescue_halving(golden):
    d = golden("rescue")
    g = es.Grid3D(*(int(v) for v in d["dims"]))
    s, tol, maxdeg = d["params"]
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    for i in range(2):
        y, st = es.apply_matfunc(op, d[f"r{i}_v"], str(d[f"r{i}_target"]), s, tol=tol, max_degree=int(maxdeg))
        assert [st.matvecs, st.degree, st.halvings] == [int(v) for v in d[f"r{i}_stats"]]
        ref = d[f"r{i}_y"]
        assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_csr_bitwise(golden):
    d = golden("csr")
    n = int(d["n"])
    a = es.CsrMatrix(n, n, d["row_ptr"], d["col"], d["vals"])
    y = a.fused_apply_flat(0.7, -1.3, d["x"])
    assert y.tobytes() == d["y"].tobytes()
    iv = es.gershgorin_interval(a)
    assert (iv.a, iv.b) == tuple(d["interval"])
    it = es.LejaInterpolant(iv, "phi1", -1.0, 150, 1e-8, iv.center + iv.halfspan * d["xi"], d["xi"], d["dd"])
    p0, mv0 = es.newton_apply(a, it, d["x"], 0.0)
    assert mv0 == int(d["mv0"]) and p0.tobytes() == d["p0"].tobytes()
    p, mv = es.newton_apply(a, it, d["x"], 1e-8)
    assert mv == int(d["mv"]) and p.tobytes() == d["p"].tobytes()


def test_combustion_and_domain_error(golden):
    d = golden("combustion")
    got = es.combustion_g(d["u"])
    np.testing.assert_allclose(got, d["g"], rtol=1e-15, atol=0)
    with pytest.raises(es.DomainError) as ei:
        es.combustion_g(np.array([1.0, 1.0, 2.0, 0.0, -1.0, 0.0]))
    assert ei.value.index == 3


@pytest.mark.parametrize("dims", [(64, 48, 1), (63, 47, 1), (40, 36, 28), (39, 17, 9), (1, 4, 6), (1030, 5, 1),
                                  (130, 20, 19)])
@pytest.mark.parametrize("bc", ["homogeneous", "neumann", "none"])
@pytest.mark.parametrize("coeff", ["none", "radial", "array"])
@pytest.mark.parametrize("kernel", ["tma", "v1"])
def test_apply_and_series_vs_oracle(dims, bc, coeff, kernel, monkeypatch):
    if kernel == "v1":
        monkeypatch.setenv("ES_KERNEL", "v1")
    nx, ny, nz = dims
    g = es.Grid3D(nx, ny, nz)
    cfun = {"none": None, "radial": es.radial_coeff, "array": lambda x, y, z: 1.0 + 0.5 * x * y + 0.25 * z}[coeff]
    op = es.StencilOperator(g, BCS[bc], coeff=cfun)
    ck = {"none": orc.COEFF_NONE, "radial": orc.COEFF_RADIAL, "array": orc.COEFF_ARRAY}[coeff]
    spec = orc.StencilSpec(nx, ny, nz, mode=ORC_MODE[bc], coeff_kind=ck,
                           coeff=op.coeff_values("f64") if coeff == "array" else None)
    rng = np.random.default_rng(hash(dims) % 1000)
    x = rng.standard_normal(g.n)
    assert op.fused_apply_flat(0.37, -1.25, x).tobytes() == orc.stencil_fused(spec, 0.37, -1.25, x).tobytes()
    lo, hi = es.gershgorin_bounds(op)
    assert (lo, hi) == spec.gershgorin()
    iv = es.SpectralInterval(lo, hi)
    it = es.make_interpolant(iv, "exp", -3.0 / max(hi, 1.0), 20, 1e-8)
    p, mv = es.newton_apply(op, it, x, 0.0)
    ref, mvr = orc.newton_stencil(spec, orc.Interp(lo, hi, "exp", it.scale, it.xi, it.dd), x, 0.0)
    assert mv == mvr == 20
    assert p.tobytes() == ref.tobytes()


def test_partition_invariance_bitwise():
    g = es.Grid3D(17, 17, 17)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    x = np.random.default_rng(3).standard_normal(g.n)
    ref = op.fused_apply_flat(2.0, 1.0, x)
    for m in (1, 2, 3, 4):
        w = es.PartitionedStencil(op, es.make_partition(g, m))
        assert w.fused_apply_flat(2.0, 1.0, x).tobytes() == ref.tobytes()
        assert w.ledger.last_scalars() == 2 * (m - 1) * 17 * 17


@pytest.mark.parametrize("kernel", ["tma", "v1"])
def test_rosenbrock_step_vs_oracle(kernel, monkeypatch):
    if kernel == "v1":
        monkeypatch.setenv("ES_KERNEL", "v1")
    g = es.Grid3D(40, 36, 32)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    u0 = 1.0 + 0.1 * np.random.default_rng(11).random(g.n)
    prob = es.SemilinearProblem(operator=op, nonlinearity=es.combustion_g, u0=u0)
    h, tol = 2e-4, 1e-6
    u1, st = es.exponential_rosenbrock_step(prob, u0, h, tol)
    spec = orc.StencilSpec(40, 36, 32)
    ref, m = orc.rosenbrock_step(spec, u0, h, tol)
    assert st.matvecs == m
    assert np.max(np.abs(u1 - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_large_2d_neumann_radial_series_vs_oracle():
    # C2-shaped (4096 x 4096 Neumann + in-kernel D), fixed degree
    g = es.Grid3D(4096, 4096, 1)
    op = es.StencilOperator(g, es.BoundaryCondition.neumann(), coeff=es.radial_coeff)
    lo, hi = es.gershgorin_bounds(op)
    it = es.make_interpolant(es.SpectralInterval(lo, hi), "phi1", -6e-7, 6, 1e-8)
    x = np.random.default_rng(1234).standard_normal(g.n)
    p, mv = es.newton_apply(op, it, x, 0.0)
    spec = orc.StencilSpec(4096, 4096, 1, mode=orc.MODE_NEUMANN, coeff_kind=orc.COEFF_RADIAL)
    ref, _ = orc.newton_stencil(spec, orc.Interp(lo, hi, "phi1", -6e-7, it.xi, it.dd), x, 0.0)
    assert mv == 6 and p.tobytes() == ref.tobytes()


def test_large_3d_series_linearity_and_oracle():
    # 256^3 Dirichlet: oracle parity at fixed degree, and exact linearity
    # under power-of-two scaling (a size-independent property)
    g = es.Grid3D(256, 256, 256)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    lo, hi = es.gershgorin_bounds(op)
    it = es.make_interpolant(es.SpectralInterval(lo, hi), "exp", -1e-4, 5, 1e-8)
    x = torch.randn(g.n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    p, _ = es.newton_apply(op, it, x, 0.0)
    p4, _ = es.newton_apply(op, it, 4.0 * x, 0.0)
    assert torch.equal(p4, 4.0 * p)
    ref, _ = orc.newton_stencil(orc.StencilSpec(256, 256, 256), orc.Interp(lo, hi, "exp", -1e-4, it.xi, it.dd),
                                x.cpu().numpy(), 0.0)
    assert p.cpu().numpy().tobytes() == ref.tobytes()


def test_rosenbrock_fused_prologue_matches_generic_path():
    g = es.Grid3D(48, 40, 30)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    u0 = torch.from_numpy(1.0 + 0.1 * np.random.default_rng(12).random(g.n)).cuda()
    prob = es.SemilinearProblem(operator=op, nonlinearity=es.combustion_g, u0=u0)
    fused = es.RosenbrockStepper(prob, 1e-6)
    generic = es.RosenbrockStepper(prob, 1e-6)
    generic._fused = False
    fused._one_call = generic._one_call = False  # the Python-orchestrated steps (es_exprb_step: test_gpu_steps.py)
    f1, g1, lo1, hi1 = fused._prologue(u0, 0.0)
    f2, g2, lo2, hi2 = generic._prologue(u0, 0.0)
    assert fused._fused is True
    assert torch.equal(f1, f2) and torch.equal(g1, g2) and (lo1, hi1) == (lo2, hi2)
    u1, s1 = fused.step(u0, 0.0, 2e-4)
    u2, s2 = generic.step(u0, 0.0, 2e-4)
    assert s1.matvecs == s2.matvecs and torch.equal(u1, u2)


def test_rosenbrock_domain_error():
    g = es.Grid3D(16, 12, 10)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    u0 = np.full(g.n, 1.0)
    u0[77] = -0.5
    u0[200] = 0.0
    prob = es.SemilinearProblem(operator=op, nonlinearity=es.combustion_g, u0=u0)
    with pytest.raises(es.DomainError) as ei:
        es.exponential_rosenbrock_step(prob, u0, 1e-4, 1e-6)
    assert ei.value.index == 77


def _emulated_slab_series(op, it, v, tol, bounds):
    """Run the C ABI slab series for several slabs of one grid in one process
    (halo planes copied by hand, slices concatenated in z order)."""
    import ctypes

    from paper_1309_4616_b200 import _lib
    from paper_1309_4616_b200.device import ptr, stream_handle

    lib = _lib.load()
    g = op.grid
    plane = g.nx * g.ny
    slabs = []
    dd, xi = it.device_coeffs()
    vd = torch.from_numpy(v).cuda()
    for r, (lo, hi) in enumerate(bounds):
        d, keep = op.desc(z0=lo, lz=hi - lo)
        ws = torch.empty(int(lib.es_leja_stencil_workspace_bytes(ctypes.byref(d))), dtype=torch.uint8, device="cuda")
        hl = torch.zeros(plane, dtype=torch.float64, device="cuda") if lo > 0 else None
        hh = torch.zeros(plane, dtype=torch.float64, device="cuda") if hi < g.nz else None
        vs = vd[lo * plane: hi * plane].clone()
        p = torch.empty_like(vs)
        _lib.check(lib.es_leja_dist_begin(ctypes.byref(d), ptr(vs), ptr(p), ptr(dd), ptr(xi), dd.numel(),
                                          1.0 / it.interval.halfspan, it.interval.center / it.interval.halfspan, tol,
                                          None, ptr(hl), ptr(hh), ptr(ws), ws.numel(), stream_handle()))
        ns = ctypes.c_int32()
        _lib.check(lib.es_leja_dist_nslices(ptr(ws), ctypes.byref(ns)))
        slabs.append(dict(d=d, keep=keep, ws=ws, hl=hl, hh=hh, v=vs, p=p, n=vs.numel(),
                          sl=torch.empty(2 * ns.value, dtype=torch.float64, device="cuda")))

    def source(s, k):
        src = ctypes.c_void_p()
        _lib.check(lib.es_leja_dist_source(ptr(s["ws"]), k, ctypes.byref(src)))
        if src.value == s["v"].data_ptr():
            return s["v"]
        off = src.value - s["ws"].data_ptr()
        return s["ws"][off: off + 8 * s["n"]].view(torch.float64)

    for k in range(1, len(it.dd)):
        srcs = [source(s, k) for s in slabs]
        for r, s in enumerate(slabs):
            if s["hl"] is not None:
                s["hl"].copy_(srcs[r - 1][-plane:])
            if s["hh"] is not None:
                s["hh"].copy_(srcs[r + 1][:plane])
        for s in slabs:
            _lib.check(lib.es_leja_dist_node(ptr(s["ws"]), ptr(s["sl"]), stream_handle()))
        allsl = torch.cat([s["sl"] for s in slabs])
        for s in slabs:
            _lib.check(lib.es_leja_dist_decide(ptr(s["ws"]), ptr(allsl), allsl.numel() // 2, stream_handle()))
    outs, mvs = [], []
    for s in slabs:
        _lib.check(lib.es_leja_dist_end(ptr(s["ws"]), stream_handle()))
        res = _lib.SeriesResult()
        lib.es_leja_fetch(ptr(s["ws"]), ctypes.byref(res), stream_handle())
        outs.append(s["p"].cpu().numpy())
        mvs.append(res.matvecs)
    return np.concatenate(outs), mvs


@pytest.mark.parametrize("tol", [0.0, 1e-8])
def test_slab_series_kernels_match_single_domain(tol):
    # chunk-aligned slabs (multiples of 8 planes): bitwise, matvec counts equal
    g = es.Grid3D(64, 40, 48)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    it = es.make_interpolant(es.gershgorin_interval(op), "exp", -4e-4, 40, 1e-8)
    v = np.random.default_rng(21).standard_normal(g.n)
    ref, mv = es.newton_apply(op, it, v, tol)
    got, mvs = _emulated_slab_series(op, it, v, tol, [(0, 16), (16, 40), (40, 48)])
    assert mvs == [mv] * 3
    assert got.tobytes() == ref.tobytes()


def test_distributed_stencil_world1_nccl():
    import torch.distributed as dist

    from paper_1309_4616_b200.distributed import DistributedStencil

    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    g = es.Grid3D(64, 32, 24)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    dop = DistributedStencil(op)
    it = es.make_interpolant(es.gershgorin_interval(op), "phi1", -3e-4, 60, 1e-8)
    v = torch.from_numpy(np.random.default_rng(2).standard_normal(g.n)).cuda()
    ref, mv = es.newton_apply(op, it, v, 1e-8)
    got, mv2 = es.newton_apply(dop, it, v, 1e-8)
    assert mv2 == mv and torch.equal(got, ref)
    y = dop.fused_apply_flat(0.5, 2.0, v)
    assert torch.equal(y, op.fused_apply_flat(0.5, 2.0, v))
    u0 = 1.0 + 0.1 * torch.rand(g.n, dtype=torch.float64, device="cuda")
    p1 = es.SemilinearProblem(operator=op, nonlinearity=es.combustion_g, u0=u0)
    p2 = es.SemilinearProblem(operator=dop, nonlinearity=es.combustion_g, u0=u0)
    a, sa = es.RosenbrockStepper(p1, 1e-6).step(u0, 0.0, 2e-4)
    b, sb = es.RosenbrockStepper(p2, 1e-6).step(u0, 0.0, 2e-4)
    assert sa.matvecs == sb.matvecs and torch.equal(a, b)


def _orc_csr(a):
    return orc.Csr(a.nrows, a.row_ptr, a.col_idx.astype(np.int32), a.vals)


def _irregular_csr(n=3000, long_row=9000, seed=3):
    """Empty rows, a row longer than one staging round (4096 products), a
    ragged tail tile (n % 256 != 0)."""
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for r in range(n):
        if r % 7 == 3:
            continue  # empty row
        k = long_row if r == 1234 else int(rng.integers(1, 40))
        c = np.unique(rng.integers(0, n, size=min(k, n)))
        rows.append(np.full(len(c), r))
        cols.append(c)
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    vals = rng.standard_normal(len(rows))
    return es.CsrMatrix.from_coo(n, n, rows, cols, vals)


@pytest.mark.parametrize("n,long_row", [(3000, 2999), (20000, 20000)])
def test_csr_apply_irregular_rows_bitwise(n, long_row):
    a = _irregular_csr(n, long_row)
    x = np.random.default_rng(1).standard_normal(n)
    got = a.fused_apply_flat(0.3, -2.5, x)
    assert got.tobytes() == orc.csr_fused(_orc_csr(a), 0.3, -2.5, x).tobytes()
    got = es.spmv(a, x)
    assert got.tobytes() == orc.csr_fused(_orc_csr(a), 1.0, 0.0, x, use_beta=False).tobytes()


@pytest.mark.parametrize("graph", [True, False])
@pytest.mark.parametrize("tol", [0.0, 1e-8])
def test_csr_series_vs_oracle(graph, tol, monkeypatch):
    if not graph:
        monkeypatch.setenv("ES_NO_GRAPH", "1")
    from paper_1309_4616_b200.sparse import synthetic_symmetric

    a = synthetic_symmetric(300_001, 6, seed=11)
    oc = _orc_csr(a)
    lo, hi = oc.gershgorin()
    iv = es.gershgorin_interval(a)
    assert (iv.a, iv.b) == (lo, hi)
    it = es.make_interpolant(iv, "phi1", -1.0, 60, 1e-8)
    it_o = orc.Interp(lo, hi, "phi1", -1.0, it.xi, it.dd)
    v = np.random.default_rng(5).standard_normal(a.nrows)
    ref, mv_ref = orc.newton_csr(oc, it_o, v, tol)
    got, mv = es.newton_apply(a, it, v, tol)
    assert mv == mv_ref
    assert got.tobytes() == ref.tobytes()


def test_csr_series_irregular_rows_bitwise():
    a = _irregular_csr(20000, 20000, seed=8)
    oc = _orc_csr(a)
    lo, hi = oc.gershgorin()
    it = es.make_interpolant(es.gershgorin_interval(a), "exp", -1e-3, 60, 1e-8)
    it_o = orc.Interp(lo, hi, "exp", -1e-3, it.xi, it.dd)
    v = np.random.default_rng(6).standard_normal(a.nrows)
    ref, mv_ref = orc.newton_csr(oc, it_o, v, 1e-10)
    got, mv = es.newton_apply(a, it, v, 1e-10)
    assert mv == mv_ref and got.tobytes() == ref.tobytes()


def _emulated_row_series(a, it, v, tol, bounds):
    """The C ABI row-block series (es_leja_csr_dist_*) for several row blocks
    of one matrix in one process: the gathered vector is assembled by hand
    (global column indices address it directly), slices concatenated in
    block order."""
    import ctypes

    from paper_1309_4616_b200 import _lib
    from paper_1309_4616_b200.device import ptr, stream_handle

    lib = _lib.load()
    dd, xi = it.device_coeffs()
    xg = torch.zeros(a.nrows, dtype=torch.float64, device="cuda")
    blocks = []
    for lo, hi in bounds:
        k0, k1 = int(a.row_ptr[lo]), int(a.row_ptr[hi])
        rp = torch.from_numpy(a.row_ptr[lo: hi + 1] - k0).cuda()
        col = torch.from_numpy(a.col_idx[k0:k1].astype(np.int32)).cuda()
        vals = torch.from_numpy(a.vals[k0:k1].copy()).cuda()
        n = hi - lo
        vs = torch.from_numpy(v[lo:hi].copy()).cuda()
        p = torch.empty_like(vs)
        ws = torch.empty(int(lib.es_leja_csr_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
        _lib.check(lib.es_leja_csr_dist_begin(n, ptr(rp), ptr(col), ptr(vals), ptr(xg), xg.numel(), ptr(vs), ptr(p),
                                              ptr(dd),
                                              ptr(xi), dd.numel(), 1.0 / it.interval.halfspan,
                                              it.interval.center / it.interval.halfspan, tol, ptr(ws), ws.numel(),
                                              stream_handle()))
        ns = ctypes.c_int32()
        _lib.check(lib.es_leja_csr_dist_nslices(ptr(ws), ctypes.byref(ns)))
        blocks.append(dict(keep=(rp, col, vals), ws=ws, v=vs, p=p, n=n, lo=lo, hi=hi,
                           sl=torch.empty(2 * ns.value, dtype=torch.float64, device="cuda")))

    def source(b, k):
        src = ctypes.c_void_p()
        _lib.check(lib.es_leja_csr_dist_source(ptr(b["ws"]), k, ctypes.byref(src)))
        if src.value == b["v"].data_ptr():
            return b["v"]
        off = src.value - b["ws"].data_ptr()
        return b["ws"][off: off + 8 * b["n"]].view(torch.float64)

    for k in range(1, len(it.dd)):
        for b in blocks:
            xg[b["lo"]: b["hi"]].copy_(source(b, k))
        for b in blocks:
            _lib.check(lib.es_leja_csr_dist_node(ptr(b["ws"]), ptr(b["sl"]), stream_handle()))
        allsl = torch.cat([b["sl"] for b in blocks])
        for b in blocks:
            _lib.check(lib.es_leja_dist_decide(ptr(b["ws"]), ptr(allsl), allsl.numel() // 2, stream_handle()))
    outs, mvs = [], []
    for b in blocks:
        _lib.check(lib.es_leja_csr_dist_end(ptr(b["ws"]), stream_handle()))
        res = _lib.SeriesResult()
        lib.es_leja_fetch(ptr(b["ws"]), ctypes.byref(res), stream_handle())
        outs.append(b["p"].cpu().numpy())
        mvs.append(res.matvecs)
    return np.concatenate(outs), mvs


@pytest.mark.parametrize("tol", [0.0, 1e-8])
def test_row_block_series_kernels_match_single_matrix(tol):
    # blocks aligned to the 16384-row reduction chunks: bitwise, equal matvec counts
    from paper_1309_4616_b200.sparse import synthetic_symmetric

    n = 3 * 16384 + 777
    a = synthetic_symmetric(n, 5, seed=2)
    it = es.make_interpolant(es.gershgorin_interval(a), "phi1", -0.7, 50, 1e-8)
    v = np.random.default_rng(3).standard_normal(n)
    ref, mv = es.newton_apply(a, it, v, tol)
    got, mvs = _emulated_row_series(a, it, v, tol, [(0, 16384), (16384, 49152), (49152, n)])
    assert mvs == [mv] * 3
    assert got.tobytes() == ref.tobytes()


def test_distributed_csr_world1_nccl():
    import torch.distributed as dist

    from paper_1309_4616_b200.distributed import DistributedCsr
    from paper_1309_4616_b200.sparse import synthetic_symmetric

    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    a = synthetic_symmetric(70_000, 6, seed=4)
    dop = DistributedCsr(a)
    it = es.make_interpolant(es.gershgorin_interval(a), "phi1", -1.0, 80, 1e-8)
    v = torch.from_numpy(np.random.default_rng(2).standard_normal(a.nrows)).cuda()
    ref, mv = es.newton_apply(a, it, v, 1e-8)
    got, mv2 = es.newton_apply(dop, it, v, 1e-8)
    assert mv2 == mv and torch.equal(got, ref)
    y = dop.fused_apply_flat(0.5, 2.0, v)
    assert torch.equal(y, a.fused_apply_flat(0.5, 2.0, v))
    assert dop.ledger.last_scalars() == 0  # one rank: nothing crosses a link


# ---- the propagate path: complex CSR (golden: csr_complex) -----------------


def _zmat(d, name):
    n = len(d[f"{name}_row_ptr"]) - 1
    return es.CsrMatrix(n, n, d[f"{name}_row_ptr"], d[f"{name}_col"], d[f"{name}_vals"])


@pytest.mark.parametrize("name", ["real", "herm"])
def test_complex_csr_apply_bitwise(golden, name):
    d = golden("csr_complex")
    a = _zmat(d, name)
    assert a.fused_apply_flat(0.7 - 0.2j, -1.3, d["x"]).tobytes() == d[f"{name}_y"].tobytes()
    assert es.spmv(a, d["x"]).tobytes() == d[f"{name}_spmv"].tobytes()


@pytest.mark.parametrize("graph", [True, False])
@pytest.mark.parametrize("name", ["real", "herm"])
def test_complex_csr_series_bitwise(golden, name, graph, monkeypatch):
    if not graph:
        monkeypatch.setenv("ES_NO_GRAPH", "1")
    d = golden("csr_complex")
    a = _zmat(d, name)
    for k in range(int(d[f"{name}_nseries"])):
        key = f"{name}_s{k}"
        lo, hi, tol, mv_ref = d[key + "_meta"]
        iv = es.SpectralInterval(float(lo), float(hi), str(d[key + "_axis"]))
        xi, dd = d[key + "_xi"], d[key + "_dd"]
        it = es.LejaInterpolant(iv, str(d[key + "_target"]), complex(d[key + "_scale"]), len(dd) - 1, 1e-10,
                                iv.center + iv.halfspan * xi, xi, dd)
        p, mv = es.newton_apply(a, it, d["x"], float(tol))
        assert mv == int(mv_ref), key
        assert p.tobytes() == d[key + "_p"].tobytes(), key


@pytest.mark.parametrize("name", ["real", "herm"])
def test_propagate_with_halving_bitwise(golden, name):
    d = golden("csr_complex")
    a = _zmat(d, name)
    n = a.nrows
    psi0 = np.full(n, 1.0 / np.sqrt(n), dtype=np.complex128)
    psi, st = es.apply_matfunc(a, psi0, "exp", -3.0j, es.gershgorin_interval(a), tol=1e-8, max_degree=40)
    assert [st.matvecs, st.degree, st.halvings] == [int(v) for v in d[f"{name}_prop_stats"]]
    assert psi.tobytes() == d[f"{name}_psi"].tobytes()
    res = es.propagate(a, 3.0, tol=1e-8, max_degree=40)
    assert res.psi.tobytes() == psi.tobytes()
    assert res.norm_drift < 1e-6  # unitary evolution
    part = es.propagate(a, 3.0, tol=1e-8, max_degree=40, workers=3)
    assert part.psi.tobytes() == psi.tobytes()  # partitioned: identical, ledger counts (m-1) n per apply


def test_complex_series_large_vs_oracle():
    from paper_1309_4616_b200.sparse import synthetic_symmetric

    a = synthetic_symmetric(200_003, 6, seed=12)
    oc = orc.Csr(a.nrows, a.row_ptr, a.col_idx.astype(np.int32), a.vals)
    iv = es.gershgorin_interval(a)
    it = es.make_interpolant(iv, "exp", -0.2j, 80, 1e-10)
    v = np.random.default_rng(1).standard_normal(a.nrows) + 1j * np.random.default_rng(2).standard_normal(a.nrows)
    ref, mv_ref = orc.newton_csr_z(oc, it.dd, it.xi, iv.center, iv.halfspan, 1.0 / iv.halfspan, v, 1e-10)
    got, mv = es.newton_apply(a, it, v, 1e-10)
    assert mv == mv_ref and got.tobytes() == ref.tobytes()


# ---- peer-memory (NVLink P2P) slab series, emulated ranks on one device -----


def _p2p_ranks(op, bounds, timeout_ns=5_000_000_000, two=False):
    """Per-rank buffers and es_p2p_desc of an in-process emulation: every
    "peer" address is another emulated rank's local buffer.  two: two Leja
    nodes per pass (two-plane halos, halo_planes = 2)."""
    import ctypes

    from paper_1309_4616_b200 import _lib

    if two and os.environ.get("ES_TB", "1") == "0":
        pytest.skip("two-node passes disabled (ES_TB=0)")
    lib = _lib.load()
    g = op.grid
    plane = g.nx * g.ny
    m = len(bounds)
    counts = []
    for lo, hi in bounds:
        d, _ = op.desc(z0=lo, lz=hi - lo)
        ns = ctypes.c_int32()
        _lib.check(lib.es_leja_stencil_nslices(ctypes.byref(d), ctypes.byref(ns)))
        counts.append(ns.value)
    total = sum(counts)
    hp = 2 if two else 1
    ranks = []
    for r, (lo, hi) in enumerate(bounds):
        ranks.append(dict(lo=lo, hi=hi, halo=torch.zeros(4 * hp * plane, dtype=torch.float64, device="cuda"),
                          slices=torch.zeros(hp * 4 * total, dtype=torch.float64, device="cuda"),
                          ghalo=torch.zeros(2 * plane, dtype=torch.float64, device="cuda"),
                          arrive=torch.zeros(1, dtype=torch.int64, device="cuda"), off=sum(counts[:r]), two=two))
    rank_slices = torch.tensor([q["slices"].data_ptr() for q in ranks], dtype=torch.int64, device="cuda")
    rank_arrive = torch.tensor([q["arrive"].data_ptr() for q in ranks], dtype=torch.int64, device="cuda")
    for r, q in enumerate(ranks):
        x = _lib.P2PDesc()
        x.nranks, x.rank, x.slice_offset, x.total_slices = m, r, q["off"], total
        for par in range(2):
            if r > 0:
                x.halo_lo[par] = q["halo"].data_ptr() + 8 * par * hp * plane
                x.peer_lo[par] = ranks[r - 1]["halo"].data_ptr() + 8 * (2 + par) * hp * plane
            if r < m - 1:
                x.halo_hi[par] = q["halo"].data_ptr() + 8 * (2 + par) * hp * plane
                x.peer_hi[par] = ranks[r + 1]["halo"].data_ptr() + 8 * par * hp * plane
        x.halo_planes = hp
        if two:  # g' boundary planes of the neighbours (filled per run by _p2p_run)
            x.gdiag_lo = q["ghalo"].data_ptr() if r > 0 else None
            x.gdiag_hi = q["ghalo"].data_ptr() + 8 * plane if r < m - 1 else None
        x.rank_slices, x.rank_arrive, x.arrive_local = rank_slices.data_ptr(), rank_arrive.data_ptr(), \
            q["arrive"].data_ptr()
        x.timeout_ns = timeout_ns
        q["desc"] = x
        q["stream"] = fresh_stream()
        d, keep = op.desc(z0=q["lo"], lz=q["hi"] - q["lo"])
        q["d"], q["keep"] = d, keep
        q["ws"] = torch.empty(int(lib.es_leja_stencil_workspace_bytes(ctypes.byref(d))), dtype=torch.uint8,
                              device="cuda")
    it0 = es.make_interpolant(es.gershgorin_interval(op), "exp", -1e-4, 3, 1e-8)
    dd0, xi0 = it0.device_coeffs()
    v0 = torch.zeros(g.n, dtype=torch.float64, device="cuda")
    gd0 = torch.zeros(g.n, dtype=torch.float64, device="cuda")

    def launch(q, gd=None):
        sl = slice(q["lo"] * plane, q["hi"] * plane)
        q["p0"] = torch.empty(sl.stop - sl.start, dtype=torch.float64, device="cuda")
        with torch.cuda.stream(q["stream"]):
            lib.es_leja_p2p(ctypes.byref(q["d"]), ctypes.byref(q["desc"]), v0[sl].data_ptr(), q["p0"].data_ptr(),
                            dd0.data_ptr(), xi0.data_ptr(), 3, 1.0, 0.0, 0.0, None if gd is None else gd[sl].data_ptr(),
                            q["ws"].data_ptr(), q["ws"].numel(), q["stream"].cuda_stream)

    _p2p_warm(ranks, launch)
    _p2p_warm(ranks, lambda q: launch(q, gd0))  # the Rosenbrock (g') node variant too
    return ranks, (rank_slices, rank_arrive)


def _p2p_warm(ranks, launch):
    """Emulation only: build and upload every rank's series graph before the
    ranks run together.  On one device a graph instantiated while another
    emulated rank already spins can be held up behind it (in a real run each
    rank's graph is built in its own process, against its own GPU).  Each
    rank runs alone with a short timeout, then counters and tables are
    cleared."""
    import ctypes

    from paper_1309_4616_b200 import _lib
    from paper_1309_4616_b200.device import ptr

    lib = _lib.load()
    for q in ranks:
        keep = q["desc"].timeout_ns
        q["desc"].timeout_ns = 50_000_000
        q["desc"].base = 0
        launch(q)
        res = _lib.SeriesResult()
        lib.es_leja_fetch(ptr(q["ws"]), ctypes.byref(res), q["stream"].cuda_stream)
        q["desc"].timeout_ns = keep
        torch.cuda.synchronize()
        for r in ranks:
            r["arrive"].zero_()
            r["slices"].zero_()
    torch.cuda.synchronize()


def _p2p_run(op, ranks, it, v, tol, rounds, only=None, gdiag=None):
    import ctypes

    from paper_1309_4616_b200 import _lib
    from paper_1309_4616_b200.device import ptr

    lib = _lib.load()
    plane = op.grid.nx * op.grid.ny
    dd, xi = it.device_coeffs()
    vd = torch.from_numpy(v).cuda()
    gd = None if gdiag is None else torch.from_numpy(gdiag).cuda()
    launched = [q for r, q in enumerate(ranks) if only is None or r in only]
    nz = op.grid.nz
    for q in launched:  # all host-side preparation before any rank starts spinning
        q["v"] = vd[q["lo"] * plane: q["hi"] * plane].clone()
        q["g"] = None if gd is None else gd[q["lo"] * plane: q["hi"] * plane].clone()
        if gd is not None and q["two"]:
            if q["lo"] > 0:
                q["ghalo"][:plane] = gd[(q["lo"] - 1) * plane: q["lo"] * plane]
            if q["hi"] < nz:
                q["ghalo"][plane:] = gd[q["hi"] * plane: (q["hi"] + 1) * plane]
        q["p"] = torch.empty_like(q["v"])
        q["desc"].base = len(ranks) * rounds
    torch.cuda.synchronize()
    for q in launched:
        with torch.cuda.stream(q["stream"]):
            rc = lib.es_leja_p2p(ctypes.byref(q["d"]), ctypes.byref(q["desc"]), ptr(q["v"]), ptr(q["p"]), ptr(dd),
                                 ptr(xi), dd.numel(), 1.0 / it.interval.halfspan,
                                 it.interval.center / it.interval.halfspan, tol, ptr(q["g"]), ptr(q["ws"]),
                                 q["ws"].numel(), q["stream"].cuda_stream)
            _lib.check(rc, "es_leja_p2p")
    out = []
    for q in launched:
        res = _lib.SeriesResult()
        rc = lib.es_leja_fetch(ptr(q["ws"]), ctypes.byref(res), q["stream"].cuda_stream)
        out.append((rc, res.matvecs, q["p"].cpu().numpy(), res.passes))
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("two", [False, True])
@pytest.mark.parametrize("graph", [True, False])
def test_p2p_slab_series_emulated_ranks_bitwise(graph, two, monkeypatch):
    if not graph:
        monkeypatch.setenv("ES_NO_GRAPH", "1")
    g = es.Grid3D(64, 40, 48)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    bounds = [(0, 16), (16, 40), (40, 48)]  # chunk-aligned: decisions bitwise those of one domain
    ranks, keep = _p2p_ranks(op, bounds, two=two)
    rounds = 0
    for target, scale, tol in (("exp", -4e-4, 0.0), ("phi1", -3e-4, 1e-8), ("exp", -4e-4, 1e-8)):
        it = es.make_interpolant(es.gershgorin_interval(op), target, scale, 40, 1e-8)
        v = np.random.default_rng(21).standard_normal(g.n)
        ref, mv = es.newton_apply(op, it, v, tol)
        outs = _p2p_run(op, ranks, it, v, tol, rounds)
        assert [o[0] for o in outs] == [0, 0, 0]
        assert [o[1] for o in outs] == [mv] * 3
        assert np.concatenate([o[2] for o in outs]).tobytes() == ref.tobytes()
        # consecutive series continue the counters: round 0 + one per pass (a
        # two-node series may end with a one-node tail pass)
        assert len({o[3] for o in outs}) == 1
        rounds += outs[0][3] + 1


@pytest.mark.parametrize("two", [False, True])
def test_p2p_slab_series_rosenbrock_diag_and_neumann(two):
    g = es.Grid3D(32, 24, 40)
    op = es.StencilOperator(g, es.BoundaryCondition.neumann())
    bounds = [(0, 8), (8, 16), (16, 32), (32, 40)]
    ranks, keep = _p2p_ranks(op, bounds, two=two)
    it = es.make_interpolant(es.gershgorin_interval(op).widened(50.0), "phi1", -5e-4, 50, 1e-8)
    v = np.random.default_rng(5).standard_normal(g.n)
    gd = np.random.default_rng(6).random(g.n) * 30.0
    ref, mv = es.newton_apply(es.RosenbrockOperator(op, torch.from_numpy(gd).cuda()), it, v, 1e-10)
    outs = _p2p_run(op, ranks, it, v, 1e-10, 0, gdiag=gd)
    assert [o[1] for o in outs] == [mv] * 4
    assert np.concatenate([o[2] for o in outs]).tobytes() == np.asarray(ref).tobytes()


@pytest.mark.parametrize("bc", ["homogeneous", "neumann"])
def test_p2p_two_node_thin_slabs(bc):
    """Two-node peer slabs of 2 and 3 planes (the two-plane halos are a whole
    neighbour slab), ragged x/y tiles, with a g' diagonal: bitwise = one domain."""
    g = es.Grid3D(70, 21, 9)
    op = es.StencilOperator(g, BCS[bc])
    bounds = [(0, 2), (2, 5), (5, 7), (7, 9)]
    ranks, keep = _p2p_ranks(op, bounds, two=True)
    it = es.make_interpolant(es.gershgorin_interval(op).widened(20.0), "phi1", -5e-4, 31, 1e-8)
    v = np.random.default_rng(8).standard_normal(g.n)
    gd = np.random.default_rng(9).random(g.n) * 10.0
    for tol, gdiag in ((0.0, gd), (1e-9, None)):
        ref, mv = es.newton_apply(op if gdiag is None else es.RosenbrockOperator(op, torch.from_numpy(gdiag).cuda()),
                                  it, v, tol)
        rounds = 0 if tol == 0.0 else (31 + 1) // 2 + 1
        outs = _p2p_run(op, ranks, it, v, tol, rounds, gdiag=gdiag)
        assert [o[0] for o in outs] == [0] * 4
        assert [o[1] for o in outs] == [mv] * 4
        assert np.concatenate([o[2] for o in outs]).tobytes() == np.asarray(ref).tobytes()


def test_p2p_missing_peer_times_out_instead_of_hanging():
    from paper_1309_4616_b200 import _lib

    g = es.Grid3D(32, 16, 16)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    ranks, keep = _p2p_ranks(op, [(0, 8), (8, 16)], timeout_ns=200_000_000, two=True)
    it = es.make_interpolant(es.gershgorin_interval(op), "exp", -1e-3, 20, 1e-8)
    v = np.random.default_rng(1).standard_normal(g.n)
    (rc, mv, _, _), = _p2p_run(op, ranks, it, v, 0.0, 0, only=[0])
    assert rc == _lib.ES_ERR_CUDA and "peer" in _lib.last_error()


def test_distributed_stencil_p2p_world1():
    import torch.distributed as dist

    from paper_1309_4616_b200.distributed import DistributedStencil

    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    g = es.Grid3D(64, 32, 24)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    dop = DistributedStencil(op, exchange="p2p")
    assert dop.exchange == "p2p"
    v = torch.from_numpy(np.random.default_rng(2).standard_normal(g.n)).cuda()
    for tol in (1e-8, 0.0, 1e-8):
        it = es.make_interpolant(es.gershgorin_interval(op), "phi1", -3e-4, 60, 1e-8)
        ref, mv = es.newton_apply(op, it, v, tol)
        got, mv2 = es.newton_apply(dop, it, v, tol)
        assert mv2 == mv and torch.equal(got, ref)
    dop.peer.close()


def _emulated_csr_p2p(a, it, v, tol, bounds, timeout_ns=5_000_000_000, rounds=0, ranks=None):
    """es_leja_csr_p2p for several row blocks of one matrix, each on its own
    stream of this device; peers' gathered vectors are the other emulated
    ranks' local buffers.  Unpadded layout (row_offset = lo, npad = n)."""
    import ctypes

    from paper_1309_4616_b200 import _lib
    from paper_1309_4616_b200.device import ptr

    lib = _lib.load()
    n = a.nrows
    m = len(bounds)
    if ranks is None:
        counts = []
        for lo, hi in bounds:
            ns = ctypes.c_int32()
            _lib.check(lib.es_leja_csr_nslices(hi - lo, ctypes.byref(ns)))
            counts.append(ns.value)
        ranks = []
        for r, (lo, hi) in enumerate(bounds):
            k0, k1 = int(a.row_ptr[lo]), int(a.row_ptr[hi])
            ranks.append(dict(lo=lo, hi=hi, off=sum(counts[:r]),
                              rp=torch.from_numpy(a.row_ptr[lo: hi + 1] - k0).cuda(),
                              col=torch.from_numpy(a.col_idx[k0:k1].astype(np.int32)).cuda(),
                              vals=torch.from_numpy(a.vals[k0:k1].copy()).cuda(),
                              xg2=torch.zeros(2 * n, dtype=torch.float64, device="cuda"),
                              slices=torch.zeros(4 * sum(counts), dtype=torch.float64, device="cuda"),
                              arrive=torch.zeros(1, dtype=torch.int64, device="cuda"),
                              stream=fresh_stream(),
                              ws=torch.empty(int(lib.es_leja_csr_workspace_bytes(hi - lo)), dtype=torch.uint8,
                                             device="cuda")))
        tabs = {key: torch.tensor([q[key].data_ptr() for q in ranks], dtype=torch.int64, device="cuda")
                for key in ("xg2", "slices", "arrive")}
        for r, q in enumerate(ranks):
            x = _lib.P2PRowsDesc()
            x.nranks, x.rank, x.slice_offset, x.total_slices = m, r, q["off"], sum(counts)
            x.row_offset, x.npad = q["lo"], n
            x.xg_local[0], x.xg_local[1] = q["xg2"].data_ptr(), q["xg2"].data_ptr() + 8 * n
            x.rank_xg, x.rank_slices = tabs["xg2"].data_ptr(), tabs["slices"].data_ptr()
            x.rank_arrive, x.arrive_local = tabs["arrive"].data_ptr(), q["arrive"].data_ptr()
            x.timeout_ns = timeout_ns
            q["desc"], q["tabs"] = x, tabs
        v0 = torch.zeros(n, dtype=torch.float64, device="cuda")
        dd0, xi0 = es.make_interpolant(es.gershgorin_interval(a), "exp", -0.1, 3, 1e-8).device_coeffs()

        def launch(q):
            q["p0"] = torch.empty(q["hi"] - q["lo"], dtype=torch.float64, device="cuda")
            with torch.cuda.stream(q["stream"]):
                lib.es_leja_csr_p2p(q["hi"] - q["lo"], ptr(q["rp"]), ptr(q["col"]), ptr(q["vals"]),
                                    ctypes.byref(q["desc"]), v0[q["lo"]: q["hi"]].data_ptr(), ptr(q["p0"]),
                                    ptr(dd0), ptr(xi0), 3, 1.0, 0.0, 0.0, ptr(q["ws"]), q["ws"].numel(),
                                    q["stream"].cuda_stream)

        _p2p_warm(ranks, launch)
    dd, xi = it.device_coeffs()
    vd = torch.from_numpy(v).cuda()
    for q in ranks:  # all host-side preparation before any rank starts spinning
        q["v"] = vd[q["lo"]: q["hi"]].clone()
        q["p"] = torch.empty_like(q["v"])
        q["desc"].base = m * rounds
    torch.cuda.synchronize()
    for q in ranks:
        with torch.cuda.stream(q["stream"]):
            _lib.check(lib.es_leja_csr_p2p(q["hi"] - q["lo"], ptr(q["rp"]), ptr(q["col"]), ptr(q["vals"]),
                                           ctypes.byref(q["desc"]), ptr(q["v"]), ptr(q["p"]), ptr(dd), ptr(xi),
                                           dd.numel(), 1.0 / it.interval.halfspan,
                                           it.interval.center / it.interval.halfspan, tol, ptr(q["ws"]),
                                           q["ws"].numel(), q["stream"].cuda_stream), "es_leja_csr_p2p")
    outs = []
    for q in ranks:
        res = _lib.SeriesResult()
        rc = lib.es_leja_fetch(ptr(q["ws"]), ctypes.byref(res), q["stream"].cuda_stream)
        outs.append((rc, res.matvecs, q["p"].cpu().numpy()))
    torch.cuda.synchronize()
    return outs, ranks


@pytest.mark.parametrize("graph", [True, False])
def test_csr_p2p_row_blocks_emulated_bitwise(graph, monkeypatch):
    if not graph:
        monkeypatch.setenv("ES_NO_GRAPH", "1")
    from paper_1309_4616_b200.sparse import synthetic_symmetric

    n = 3 * 16384 + 777
    a = synthetic_symmetric(n, 5, seed=2)
    bounds = [(0, 16384), (16384, 49152), (49152, n)]
    ranks, rounds = None, 0
    for target, scale, tol in (("phi1", -0.7, 0.0), ("exp", -0.5, 1e-8), ("phi1", -0.7, 1e-8)):
        it = es.make_interpolant(es.gershgorin_interval(a), target, scale, 50, 1e-8)
        v = np.random.default_rng(3).standard_normal(n)
        ref, mv = es.newton_apply(a, it, v, tol)
        outs, ranks = _emulated_csr_p2p(a, it, v, tol, bounds, rounds=rounds, ranks=ranks)
        assert [o[0] for o in outs] == [0, 0, 0]
        assert [o[1] for o in outs] == [mv] * 3
        assert np.concatenate([o[2] for o in outs]).tobytes() == ref.tobytes()
        rounds += mv + 1


def test_distributed_csr_p2p_world1():
    import torch.distributed as dist

    from paper_1309_4616_b200.distributed import DistributedCsr
    from paper_1309_4616_b200.sparse import synthetic_symmetric

    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    a = synthetic_symmetric(70_000, 6, seed=4)
    dop = DistributedCsr(a, exchange="p2p")
    assert dop.exchange == "p2p"
    v = torch.from_numpy(np.random.default_rng(2).standard_normal(a.nrows)).cuda()
    for tol in (1e-8, 0.0, 1e-8):
        it = es.make_interpolant(es.gershgorin_interval(a), "phi1", -1.0, 80, 1e-8)
        ref, mv = es.newton_apply(a, it, v, tol)
        got, mv2 = es.newton_apply(dop, it, v, tol)
        assert mv2 == mv and torch.equal(got, ref)
    dop.peer.close()


# ---- edge cases (empty / degenerate / zero inputs), reference semantics ------


def test_zero_vector_series_stops_after_two_nodes():
    # |dd_k| ||w|| = 0 <= tol ||p|| = 0 holds at k = 1 and 2 (matfunc.py:302-311)
    g = es.Grid3D(32, 16, 8)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    it = es.make_interpolant(es.gershgorin_interval(op), "exp", -1e-3, 40, 1e-8)
    p, mv = es.newton_apply(op, it, np.zeros(g.n), 1e-8)
    assert mv == 2 and not p.any()
    from paper_1309_4616_b200.sparse import synthetic_symmetric

    a = synthetic_symmetric(1000, 3, seed=1)
    it = es.make_interpolant(es.gershgorin_interval(a), "phi1", -0.5, 40, 1e-8)
    p, mv = es.newton_apply(a, it, np.zeros(1000), 1e-8)
    assert mv == 2 and not p.any()
    pz, mvz = es.newton_apply(a, it, np.zeros(1000, dtype=np.complex128), 1e-8)
    assert mvz == 2 and not pz.any()


def test_degenerate_intervals_return_dd0_v():
    # a == b: one node, dd_0 v, zero matvecs (matfunc.py:285-286)
    g = es.Grid3D(1, 1, 1)
    op = es.StencilOperator(g, es.BoundaryCondition.neumann())
    iv = es.gershgorin_interval(op)
    assert iv.a == iv.b == 0.0
    it = es.make_interpolant(iv, "phi1", -0.3, 20, 1e-8)
    p, mv = es.newton_apply(op, it, np.array([2.5]), 1e-8)
    assert mv == 0 and p.tobytes() == (it.dd[0] * np.array([2.5])).tobytes()
    empty = es.CsrMatrix(0, 0, np.zeros(1, dtype=np.int64), np.zeros(0, dtype=np.int32), np.zeros(0))
    it = es.make_interpolant(es.gershgorin_interval(empty), "exp", -1.0, 20, 1e-8)
    p, mv = es.newton_apply(empty, it, np.zeros(0), 1e-8)
    assert mv == 0 and p.shape == (0,)
    diag = es.CsrMatrix.from_dense(np.diag([3.0, 3.0, 3.0]))
    it = es.make_interpolant(es.gershgorin_interval(diag), "exp", -0.5j, 20, 1e-8)  # complex dd_0
    v = np.array([1.0, -2.0, 0.5])
    p, mv = es.newton_apply(diag, it, v, 1e-8)
    assert mv == 0 and p.tobytes() == (it.dd[0] * v).tobytes()


def test_convergence_error_carries_residual_and_degree():
    g = es.Grid3D(24, 24, 24)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    it = es.make_interpolant(es.gershgorin_interval(op), "exp", -5e-3, 6, 1e-12)  # far too few nodes
    v = np.random.default_rng(0).standard_normal(g.n)
    with pytest.raises(es.ConvergenceError) as ei:
        es.newton_apply(op, it, v, 1e-12)
    spec = orc.StencilSpec(24, 24, 24)
    lo, hi = spec.gershgorin()
    with pytest.raises(orc.OracleConvergenceError) as eo:
        orc.newton_stencil(spec, orc.Interp(lo, hi, "exp", -5e-3, it.xi, it.dd), v, 1e-12)
    assert ei.value.degree == eo.value.degree == 6
    assert ei.value.residual == pytest.approx(eo.value.residual, rel=1e-12)


# ---- single precision plain applies (the reference's float kernels) --------


def test_f32_stencil_applies_bitwise(golden):
    d = golden("f32")
    for i in range(int(d["ncases"])):
        g = es.Grid3D(*(int(v) for v in d[f"c{i}_dims"]))
        bc = str(d[f"c{i}_bc"])
        bco = (es.BoundaryCondition.function(lambda x, y, z: z * (1 - z) * x * y, "poly") if bc == "poly"
               else BCS[bc])
        op = es.StencilOperator(g, bco, coeff=coeff_d if bool(d[f"c{i}_coeff"]) else None)
        x = d[f"c{i}_x"]
        if bc == "poly":
            got = es.apply(op, es.Field(g, x)).values
        else:
            a, b = d[f"c{i}_ab"]
            got = op.fused_apply_flat(float(a), float(b), x)
        assert got.dtype == np.float32
        assert got.tobytes() == d[f"c{i}_y"].tobytes(), (i, tuple(d[f"c{i}_dims"]), bc)


def test_f32_slab_with_halos_and_coefficient_bitwise(golden):
    d = golden("f32")
    g = es.Grid3D(11, 9, 12)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous(), coeff=coeff_d)
    x3 = torch.from_numpy(d["slab_x"]).cuda().view(g.shape)
    out = torch.empty((4, g.ny, g.nx), dtype=torch.float32, device="cuda")
    es.fused_slab(op, 1.5, -0.25, x3[5:9].contiguous(), out, halo_lo=x3[4].contiguous(), halo_hi=x3[9].contiguous(),
                  z0=5)
    assert out.cpu().numpy().reshape(-1).tobytes() == d["slab_y"].tobytes()


def test_f32_combustion_and_f32_csr(golden):
    d = golden("f32")
    g = es.combustion_g(d["comb_u"])
    assert g.dtype == np.float32
    # CUDA expf vs libm expf: <= 2 ulp (and a few ulp of float subnormals)
    np.testing.assert_allclose(g, d["comb_g"], rtol=4e-7, atol=1e-43)
    with pytest.raises(es.DomainError) as ei:
        es.combustion_g(np.array([1.0, 0.5, -1.0], dtype=np.float32))
    assert ei.value.index == 2
    n = len(d["csr_row_ptr"]) - 1
    a = es.CsrMatrix(n, n, d["csr_row_ptr"], d["csr_col"], d["csr_vals"])
    y = es.fused_spmv(a, 0.7, -1.3, d["csr_x"])
    # the reference promotes to f64 and, with no compiled f32/f64 combo, falls
    # back to its numpy twin, whose np.add.reduce sums rows pairwise; the
    # device sums in storage order like every other CSR path (1e-14)
    assert y.dtype == np.float64
    np.testing.assert_allclose(y, d["csr_y"], rtol=1e-13, atol=1e-13 * np.max(np.abs(d["csr_y"])))


# ---- two Leja nodes per pass (stencil_tb.cuh, opt-in ES_TB=1) ---------------


@pytest.mark.parametrize("graph,march", [(True, "0"), (False, "0"), (True, "1"), (False, "1")])
def test_two_node_pass_bitwise(graph, march, monkeypatch):
    """Temporal blocking: same p, same matvec counts as one node per pass,
    for Dirichlet / Neumann, coefficient kinds, a g' diagonal, odd and even
    node counts, ragged tiles and chunks; march "1": the plane-marching
    kernel (stencil_tb3m.cuh) where it applies (coefficient none)."""
    monkeypatch.setenv("ES_TB3M", march)
    if not graph:
        monkeypatch.setenv("ES_NO_GRAPH", "1")
    cases = [((64, 40, 48), "homogeneous", None, False, 1e-8), ((70, 18, 21), "neumann", None, True, 1e-10),
             ((66, 24, 17), "homogeneous", coeff_d, True, 0.0), ((128, 16, 9), "neumann", "radial", False, 1e-8)]
    for dims, bc, coeff, gd, tol in cases:
        g = es.Grid3D(*dims)
        op = es.StencilOperator(g, BCS[bc], coeff=es.radial_coeff if coeff == "radial" else coeff)
        iv = es.gershgorin_interval(op)
        it = es.make_interpolant(iv.widened(40.0) if gd else iv, "phi1", -4e-4, 41, 1e-8)
        v = torch.from_numpy(np.random.default_rng(3).standard_normal(g.n)).cuda()
        gdiag = torch.from_numpy(np.random.default_rng(4).random(g.n) * 20.0).cuda() if gd else None
        monkeypatch.setenv("ES_TB", "0")
        ref, mv = es.newton_apply(op, it, v, tol, gdiag=gdiag)
        monkeypatch.setenv("ES_TB", "1")
        got, mv2 = es.newton_apply(op, it, v, tol, gdiag=gdiag)
        monkeypatch.delenv("ES_TB")
        assert mv2 == mv, (dims, bc)
        assert torch.equal(got, ref), (dims, bc)


@pytest.mark.parametrize("dims,bc,chunk", [((512, 512, 256), "homogeneous", None), ((256, 128, 300), "neumann", "128")])
def test_two_node_long_chunks_bitwise(dims, bc, chunk, monkeypatch):
    """The plane-marching pass picks longer z chunks on large grids
    (csrc/stencil.cu prepare_series: 64 planes for the first grid; the
    second forces 128 with a ragged last chunk): p and matvec counts equal
    the one-node series bit for bit, with g' and tol > 0."""
    if chunk:
        monkeypatch.setenv("ES_TBCHUNK", chunk)
    g = es.Grid3D(*dims)
    op = es.StencilOperator(g, BCS[bc])
    iv = es.gershgorin_interval(op).widened(30.0)
    rng = np.random.default_rng(sum(dims))
    v = torch.from_numpy(rng.standard_normal(g.n)).cuda()
    gdiag = torch.from_numpy(rng.random(g.n) * 30.0).cuda()
    it = es.make_interpolant(iv, "phi1", -1e-5, 60, 1e-8)
    out = {}
    for tb in ("0", "1"):
        monkeypatch.setenv("ES_TB", tb)
        out[tb] = es.newton_apply(op, it, v, 1e-9, gdiag=gdiag)
    monkeypatch.delenv("ES_TB")
    (ref, m0), (got, m1) = out["0"], out["1"]
    assert m1 == m0 and m0 > 4, (m0, m1)
    assert torch.equal(got, ref)


@pytest.mark.parametrize("dims,bc,nodes", [((6, 4, 2), "homogeneous", 7), ((10, 9, 3), "neumann", 8),
                                           ((130, 17, 33), "homogeneous", 9), ((64, 8, 64), "neumann", 2),
                                           ((66, 10, 35), "homogeneous", 3), ((2, 2, 5), "neumann", 6)])
@pytest.mark.parametrize("march", ["0", "1"])
def test_two_node_pass_edges_vs_oracle(dims, bc, nodes, march, monkeypatch):
    """Two-node passes on tiny / ragged grids (tiles cut by the domain in x, y
    and z, one- and two-plane slabs, odd and even node counts, g' diagonal)
    against the oracle, bitwise, at fixed degree (both 3D two-node kernels)."""
    monkeypatch.setenv("ES_TB3M", march)
    g = es.Grid3D(*dims)
    op = es.StencilOperator(g, BCS[bc])
    lo, hi = es.gershgorin_bounds(op)
    it = es.make_interpolant(es.SpectralInterval(lo, hi), "phi1", -2e-4, nodes, 1e-8)
    rng = np.random.default_rng(sum(dims))
    v = rng.standard_normal(g.n)
    gd = rng.random(g.n) * 5.0
    p, mv = es.newton_apply(es.RosenbrockOperator(op, torch.from_numpy(gd).cuda()), it, v, 0.0)
    spec = orc.StencilSpec(*dims, mode=ORC_MODE[bc])
    ref, _ = orc.newton_stencil(spec, orc.Interp(lo, hi, "phi1", -2e-4, it.xi, it.dd), v, 0.0, gdiag=gd)
    assert mv == nodes
    assert np.asarray(p).tobytes() == ref.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("graph,march", [(True, "0"), (False, "0"), (True, "1")])
def test_two_node_tail_pass_bitwise(graph, march, monkeypatch):
    """A two-node series runs node k alone when node k-1 met the term test
    for the first time (the series then usually stops at k).  Over a sweep
    of tolerances -- stops at odd and even k, and first hits that do not
    stop (the pass pairing then shifts by one) -- p and the matvec counts
    equal the plain two-node and the one-node series bit for bit, and the
    pass count never exceeds the plain pairing's."""
    from paper_1309_4616_b200 import timing

    monkeypatch.setenv("ES_TB3M", march)
    if not graph:
        monkeypatch.setenv("ES_NO_GRAPH", "1")
    g = es.Grid3D(72, 40, 44)
    op = es.StencilOperator(g, BCS["homogeneous"])
    iv = es.gershgorin_interval(op).widened(30.0)
    rng = np.random.default_rng(12)
    v = torch.from_numpy(rng.standard_normal(g.n)).cuda()
    gdiag = torch.from_numpy(rng.random(g.n) * 30.0).cuda()
    it = es.make_interpolant(iv, "phi1", -3e-4, 60, 1e-8)
    stops = set()
    for tol in np.logspace(-13, -3, 31):
        runs = {}
        for tb, tail in (("0", "1"), ("1", "0"), ("1", "1")):
            monkeypatch.setenv("ES_TB", tb)
            monkeypatch.setenv("ES_TB_TAIL", tail)
            with timing.SeriesTimer() as tm:
                p, mv = es.newton_apply(op, it, v, float(tol), gdiag=gdiag)
            runs[(tb, tail)] = (p, mv, tm.passes())
        p0, m0, _ = runs[("0", "1")]
        for key in (("1", "0"), ("1", "1")):
            p, m, _ = runs[key]
            assert m == m0, (tol, key, m, m0)
            assert torch.equal(p, p0), (tol, key)
        plain, tail = runs[("1", "0")][2], runs[("1", "1")][2]
        assert plain == (m0 + 1) // 2, (tol, plain, m0)
        assert tail <= plain + 1 and 2 * tail >= m0, (tol, tail, plain, m0)
        stops.add(m0 & 1)
    monkeypatch.delenv("ES_TB")
    monkeypatch.delenv("ES_TB_TAIL")
    assert stops == {0, 1}, stops


SMALL_CASES = [((256, 256), "homogeneous", None, False, 1e-8), ((128, 96), "neumann", "radial", False, 1e-10),
               ((64, 70), "none", None, True, 1e-9), ((250, 33), "homogeneous", coeff_d, True, 0.0),
               ((512, 40), "neumann", coeff_d, False, 1e-12), ((2, 3), "homogeneous", None, False, 1e-8)]


@pytest.mark.gpu
@pytest.mark.parametrize("dims,bc,coeff,gd,tol", SMALL_CASES)
def test_small_series_bitwise(dims, bc, coeff, gd, tol, monkeypatch):
    """The persistent small-grid series (one cooperative launch, grid barrier
    per node; series_small.cu) equals the graph path (ES_SMALL=0) bit for
    bit -- p, matvec counts, last term and |p| -- for every ghost mode,
    coefficient kind, with and without a g' diagonal, tol > 0 and fixed
    degree, and the oracle too."""
    nx, ny = dims
    g = es.Grid3D(nx, ny, 1)
    op = es.StencilOperator(g, BCS[bc], coeff=es.radial_coeff if coeff == "radial" else coeff)
    iv = es.gershgorin_interval(op)
    iv = iv.widened(25.0) if gd else iv
    it = es.make_interpolant(iv, "phi1", -12.0 / max(abs(iv.a), abs(iv.b)), 70, 1e-8)
    rng = np.random.default_rng(nx * 7 + ny)
    v = torch.from_numpy(rng.standard_normal(g.n)).cuda()
    gdiag = torch.from_numpy(rng.random(g.n) * 25.0).cuda() if gd else None
    out = {}
    for small in ("0", "1"):
        monkeypatch.setenv("ES_SMALL", small)
        out[small] = es.newton_apply(op, it, v, tol, gdiag=gdiag)
    monkeypatch.delenv("ES_SMALL")
    (ref, mv), (got, mv2) = out["0"], out["1"]
    assert mv2 == mv, (dims, bc, mv, mv2)
    assert torch.equal(got, ref), (dims, bc)


@pytest.mark.gpu
def test_small_series_convergence_error_matches(monkeypatch):
    """Degree exhausted with tol > 0: both paths raise ConvergenceError with
    the same residual and degree."""
    g = es.Grid3D(96, 64, 1)
    op = es.StencilOperator(g, BCS["homogeneous"])
    it = es.make_interpolant(es.gershgorin_interval(op), "phi1", -5e-2, 6, 1e-8)
    v = torch.from_numpy(np.random.default_rng(5).standard_normal(g.n)).cuda()
    msgs = []
    for small in ("0", "1"):
        monkeypatch.setenv("ES_SMALL", small)
        with pytest.raises(es.ConvergenceError) as ei:
            es.newton_apply(op, it, v, 1e-14)
        msgs.append((ei.value.residual, ei.value.degree))
    monkeypatch.delenv("ES_SMALL")
    assert msgs[0] == msgs[1], msgs


@pytest.mark.gpu
@pytest.mark.parametrize("source", [False, True])
def test_small_expeuler_step_bitwise(source, monkeypatch):
    """The fused small-grid exponential-Euler step (both series, g(u) - b in
    the kernel, u + h z) equals the two-graph step bit for bit, and a point
    outside the combustion domain still raises DomainError with its index."""
    g = es.Grid3D(256, 256, 1)
    op = es.StencilOperator(g, BCS["homogeneous"])
    rng = np.random.default_rng(21)
    u0 = 1.0 + 0.1 * rng.random(g.n)
    b = 0.01 * rng.standard_normal(g.n) if source else None
    prob = es.SemilinearProblem(operator=op, nonlinearity=es.combustion_g, u0=u0, boundary_source=b)
    res = {}
    for small in ("0", "1"):
        monkeypatch.setenv("ES_SMALL", small)
        res[small] = es.exponential_euler_step(prob, u0, 2e-3, 1e-4)
    u_ref, st_ref = res["0"]
    u_got, st_got = res["1"]
    assert (st_got.matvecs_exp, st_got.matvecs_phi1) == (st_ref.matvecs_exp, st_ref.matvecs_phi1)
    assert np.array_equal(u_got, u_ref)
    bad = u0.copy()
    bad[777] = -1.0
    for small in ("0", "1"):
        monkeypatch.setenv("ES_SMALL", small)
        with pytest.raises(es.DomainError) as ei:
            es.exponential_euler_step(es.SemilinearProblem(operator=op, nonlinearity=es.combustion_g, u0=bad),
                                      bad, 2e-3, 1e-4)
        assert "777" in str(ei.value)
    monkeypatch.delenv("ES_SMALL")


@pytest.mark.gpu
@pytest.mark.parametrize("graph,rows,march", [(True, "0", "0"), (False, "0", "0"), (True, "1", "0"),
                                               (True, "0", "1"), (False, "0", "1")])
def test_two_node_2d_bitwise(graph, rows, march, monkeypatch):
    """Two Leja nodes per pass on single-plane grids (stencil_tb2d.cuh) equal
    the one-node series bit for bit -- p and matvec counts -- for Dirichlet
    and Neumann, no coefficient and the staged sampled D, odd and even node
    counts, tiles cut by the domain (nx not a multiple of 256), row chunks cut
    by ny, fixed degree and tol > 0 (small-grid persistent path off)."""
    monkeypatch.setenv("ES_SMALL", "0")
    monkeypatch.setenv("ES_TB2R", rows)  # "1": the R-row-stage variant where nx % 8 == 0 (stencil_tb2r.cuh)
    monkeypatch.setenv("ES_TB2M", march)  # "1": the row-marching variant (stencil_tb2m.cuh)
    if not graph:
        monkeypatch.setenv("ES_NO_GRAPH", "1")
    cases = [((1000, 77), "neumann", "radial", 1e-10), ((512, 64), "homogeneous", None, 0.0),
             ((770, 130), "homogeneous", coeff_d, 1e-8), ((258, 33), "neumann", None, 1e-12),
             ((2048, 40), "neumann", "radial", 0.0)]
    for (nx, ny), bc, coeff, tol in cases:
        g = es.Grid3D(nx, ny, 1)
        op = es.StencilOperator(g, BCS[bc], coeff=es.radial_coeff if coeff == "radial" else coeff)
        iv = es.gershgorin_interval(op)
        for nodes in (37, 40):
            it = es.make_interpolant(iv, "phi1", -9.0 / max(abs(iv.a), abs(iv.b)), nodes, 1e-8)
            v = torch.from_numpy(np.random.default_rng(nx + ny).standard_normal(g.n)).cuda()
            out = {}
            for tb in ("0", "1"):
                monkeypatch.setenv("ES_TB2D", tb)
                try:
                    out[tb] = es.newton_apply(op, it, v, tol)
                except es.ConvergenceError as e:
                    out[tb] = (e.residual, e.degree)
            monkeypatch.delenv("ES_TB2D")
            a, b = out["0"], out["1"]
            assert b[1] == a[1], ((nx, ny), bc, nodes)
            if isinstance(a[0], torch.Tensor):
                assert torch.equal(b[0], a[0]), ((nx, ny), bc, nodes)
            else:
                assert a == b


@pytest.mark.parametrize("tol", [0.0, 1e-8])
def test_partitioned_stencil_series_runs_on_slabs(tol):
    """PartitionedStencil's series runs slab by slab (es_leja_dist_* per slab,
    seam planes exchanged per node): bitwise the one-domain series for
    chunk-aligned slabs incl. matvec counts, one ledger entry per node of
    2 (m-1) nx ny scalars; a non-aligned partition keeps p bitwise at fixed
    degree."""
    g = es.Grid3D(64, 40, 48)
    op = es.StencilOperator(g, es.BoundaryCondition.homogeneous())
    it = es.make_interpolant(es.gershgorin_interval(op), "phi1", -4e-4, 40, 1e-8)
    v = np.random.default_rng(31).standard_normal(g.n)
    ref, mv = es.newton_apply(op, it, v, tol)
    for m in (2, 3):
        w = es.PartitionedStencil(op, es.make_partition(g, m))  # 24/24, 16/16/16: 8-plane aligned
        got, mv2 = es.newton_apply(w, it, v, tol)
        assert mv2 == mv and got.tobytes() == ref.tobytes(), m
        assert w.ledger.apply_count == mv and w.ledger.last_scalars() == 2 * (m - 1) * 64 * 40
    if tol == 0.0:
        g5 = es.Grid3D(64, 40, 45)
        op5 = es.StencilOperator(g5, es.BoundaryCondition.neumann())
        it5 = es.make_interpolant(es.gershgorin_interval(op5), "exp", -4e-4, 25, 1e-8)
        v5 = np.random.default_rng(32).standard_normal(g5.n)
        ref5, _ = es.newton_apply(op5, it5, v5, 0.0)
        got5, _ = es.newton_apply(es.PartitionedStencil(op5, es.make_partition(g5, 4)), it5, v5, 0.0)
        assert got5.tobytes() == ref5.tobytes()
