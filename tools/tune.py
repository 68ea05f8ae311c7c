"""Chunk-length sweep of the fused node kernel (device-timed series).
Not part of the product; used to pick defaults."""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1309_4616_b200 as es  # noqa: E402
from paper_1309_4616_b200 import timing  # noqa: E402


def run(cfg, env, nodes=20, reps=3):
    for k in ("ES_TCHUNK3D", "ES_TCHUNK2D", "ES_KERNEL"):
        os.environ.pop(k, None)
    os.environ.update(env)
    dims, bc, coeff, gd, bpp = cfg
    g = es.Grid3D(*dims)
    op = es.StencilOperator(g, bc, coeff=coeff)
    lo, hi = es.gershgorin_bounds(op)
    it = es.make_interpolant(es.SpectralInterval(lo, hi), "phi1", -2.5e-5, nodes, 1e-8)
    v = torch.rand(g.n, dtype=torch.float64, device="cuda")
    gdv = torch.rand(g.n, dtype=torch.float64, device="cuda") if gd else None
    es.newton_apply(op, it, v, 0.0, gdiag=gdv)
    with timing.SeriesTimer() as tm:
        for _ in range(reps):
            es.newton_apply(op, it, v, 0.0, gdiag=gdv)
    s, mv = tm.totals()
    node = s / mv
    return {"env": env, "node_us": node * 1e6, "GBs": bpp * g.n / node / 1e9}


C3 = ((512, 512, 512), es.BoundaryCondition.homogeneous(), None, True, 40)
C3e = ((512, 512, 512), es.BoundaryCondition.homogeneous(), None, False, 32)
C2 = ((4096, 4096, 1), es.BoundaryCondition.neumann(), es.radial_coeff, False, 32)
C2p = ((4096, 4096, 1), es.BoundaryCondition.homogeneous(), None, False, 32)
C4 = ((1024, 1024, 1024), es.BoundaryCondition.homogeneous(), None, True, 40)
out = []
for ch in ("4", "8", "12", "16", "32"):
    out.append(("C3", run(C3, {"ES_TCHUNK3D": ch})))
out.append(("C3-euler", run(C3e, {})))
out.append(("C3-v1", run(C3, {"ES_KERNEL": "v1"})))
for ch in (None, "16", "32"):
    out.append(("C2", run(C2, {} if ch is None else {"ES_TCHUNK2D": ch})))
out.append(("C2-plain", run(C2p, {})))
out.append(("C4", run(C4, {})))
for name, r in out:
    print(name, json.dumps(r), flush=True)
