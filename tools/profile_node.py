"""Run a few fused Leja nodes of one config with plain launches (ncu cannot
profile kernels inside conditional CUDA graphs) -- the target for
`ncu --set full -k regex:k_node`.  Not part of the product."""

import argparse
import os
import sys

os.environ["ES_NO_GRAPH"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1309_4616_b200 as es  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--nodes", type=int, default=6)
a = ap.parse_args()
if a.config == "C5":
    from paper_1309_4616_b200.sparse import synthetic_symmetric

    m = synthetic_symmetric(2**22, 6, seed=1234)
    it = es.make_interpolant(es.gershgorin_interval(m), "phi1", -1.0, a.nodes, 1e-8)
    v = torch.rand(m.nrows, dtype=torch.float64, device="cuda")
    for _ in range(2):
        p, mv = es.newton_apply(m, it, v, 0.0)
    torch.cuda.synchronize()
    print("nodes", mv)
    sys.exit(0)
dims = {"C3": (512, 512, 512), "C2": (4096, 4096, 1), "C4": (1024, 1024, 1024), "C1": (256, 256, 1)}[a.config]
g = es.Grid3D(*dims)
bc = es.BoundaryCondition.neumann() if a.config == "C2" else es.BoundaryCondition.homogeneous()
op = es.StencilOperator(g, bc, coeff=es.radial_coeff if a.config == "C2" else None)
lo, hi = es.gershgorin_bounds(op)
it = es.make_interpolant(es.SpectralInterval(lo, hi), "phi1", -2.5e-5, a.nodes, 1e-8)
v = torch.rand(g.n, dtype=torch.float64, device="cuda")
gd = torch.rand(g.n, dtype=torch.float64, device="cuda") if a.config in ("C3", "C4") else None
for _ in range(2):
    p, mv = es.newton_apply(op, it, v, 0.0, gdiag=gd)
torch.cuda.synchronize()
print("nodes", mv)
