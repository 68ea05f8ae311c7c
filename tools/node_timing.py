"""µs per fused Leja node (fixed-degree series, tol = 0, CUDA events) for
stencil configurations given as nx,ny,nz[:bc[:coeff[:gd]]]; prints
algorithmic GB/s.  Not part of the product."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1309_4616_b200 as es  # noqa: E402

specs = sys.argv[1:] or ["4096,4096,1:neumann:radial", "4096,4096,1:neumann", "4096,4096,1:homogeneous",
                         "512,512,512:homogeneous::gd", "512,512,512:homogeneous"]
for spec in specs:
    parts = spec.split(":") + ["", "", ""]
    nx, ny, nz = (int(v) for v in parts[0].split(","))
    bc = {"neumann": es.BoundaryCondition.neumann(), "homogeneous": es.BoundaryCondition.homogeneous(),
          "none": es.BoundaryCondition.none()}[parts[1] or "homogeneous"]
    g = es.Grid3D(nx, ny, nz)
    op = es.StencilOperator(g, bc, coeff=es.radial_coeff if parts[2] in ("radial", "array") else None)
    if parts[2] == "array":  # the same D, staged as a sampled array (ES_COEFF_ARRAY)
        from paper_1309_4616_b200 import _lib

        op._coeff_kind = _lib.ES_COEFF_ARRAY
    nodes = 24
    it = es.make_interpolant(es.gershgorin_interval(op), "phi1", -1e-7, nodes, 1e-8)
    v = torch.randn(g.n, dtype=torch.float64, device="cuda")
    gd = torch.rand(g.n, dtype=torch.float64, device="cuda") if parts[3] == "gd" else None
    for _ in range(2):
        es.newton_apply(op, it, v, 0.0, gdiag=gd)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p, mv = es.newton_apply(op, it, v, 0.0, gdiag=gd)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3 / mv)
    bpp = 40 if gd is not None else 32
    print(f"{spec:36s} node {best * 1e6:8.1f} us  {bpp * g.n / best / 1e9:7.0f} GB/s algorithmic", flush=True)
